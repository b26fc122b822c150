"""Per-CTA start/end of the C5 exact row-stream launches (LAPIS_B200_RS_TIMES)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
path = "gpurun_out/rs_times.txt"
os.environ["LAPIS_B200_RS_TIMES"] = path
if os.path.exists(path):
    os.remove(path)
import paper_2509_25605_b200 as lb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 585
rp, ci, v = lb.synth_stencil(27, n)
N = rp.numel() - 1
x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, N)).cuda()
y = torch.empty(N, dtype=torch.float64, device="cuda")
plan = lb.CsrPlan(rp, exact=True)
for _ in range(12):
    plan.spmv(ci, v, x, y)
torch.cuda.synchronize()
blocks = open(path).read().split("launch ")[1:]
for blk in blocks:
    lines = blk.strip().splitlines()
    a = np.array([[int(t) for t in l.split()] for l in lines[1:]], dtype=np.float64)
    t0 = a[:, 0].min()
    st, en, sm = (a[:, 0] - t0) / 1e6, (a[:, 1] - t0) / 1e6, a[:, 2].astype(int)
    per_sm = np.bincount(sm)
    # end time by SM
    sm_end = np.zeros(sm.max() + 1)
    np.maximum.at(sm_end, sm, en)
    print(f"grid {len(a)}: span {en.max():.2f} ms; start max {st.max():.3f}; end min/p10/p50/p90/max "
          f"{en.min():.2f} {np.percentile(en, 10):.2f} {np.median(en):.2f} {np.percentile(en, 90):.2f} "
          f"{en.max():.2f}; CTAs/SM {per_sm.min()}-{per_sm.max()}; slowest SMs "
          f"{np.argsort(sm_end)[-6:].tolist()} fastest {np.argsort(sm_end)[:6].tolist()}")
