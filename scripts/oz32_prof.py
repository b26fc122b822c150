import sys
import torch
sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb  # noqa: E402
A = torch.rand(4096, 4096, device="cuda")
B = torch.rand(4096, 4096, device="cuda")
for _ in range(2):
    C = lb.gemm(A, B)
torch.cuda.synchronize()
