"""SpMV on the config-3 power-law matrix (10M rows, ~100M nnz, SURVEY A.8
generator): the plan's warp-block kernel with and without its L2 policy
(LAPIS_B200_SPMV_WB_POLICY), timed and checked against each other."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if len(sys.argv) > 1:  # worker: one mode per process (the policy switch is read once)
    import torch
    sys.path.insert(0, str(ROOT))
    import paper_2509_25605_b200 as lb  # noqa: E402
    import synth_inputs as S  # noqa: E402
    spec = S.PowerLawSpec(10_000_000, seed=1)
    rp, ci = S.powerlaw_structure_device(spec)
    n = rp.numel() - 1
    nnz = int(rp[-1].item())
    v = torch.from_numpy(S.powerlaw_values(spec, nnz)).cuda()
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    work = nnz * 12 + (n + 1) * 8 + 2 * n * 8
    plan = lb.CsrPlan(rp)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        plan.spmv(ci, v, x, y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        plan.spmv(ci, v, x, y)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 20 / 1e3
    torch.save(y.cpu(), f"/tmp/spmv_pl_{sys.argv[1]}.pt")
    print(sys.argv[1], plan.info()["kernel"], f"{t * 1e3:.3f} ms  {work / t / 1e9:.0f} GB/s", flush=True)
else:
    for pol in ("1", "0"):
        subprocess.run([sys.executable, __file__, pol], env={**os.environ, "LAPIS_B200_SPMV_WB_POLICY": pol},
                       check=True)
    import torch
    d = (torch.load("/tmp/spmv_pl_1.pt") - torch.load("/tmp/spmv_pl_0.pt")).abs().max().item()
    print("max |diff| policy vs plain:", d)
