import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2509_25605_b200 as lb
n = 256
A = np.eye(n, dtype=np.float32)
B = (np.arange(n * n) % 1000).reshape(n, n).astype(np.float32)
C = lb.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), mode="tf32x3").cpu().numpy()
print("identity ok:", np.array_equal(C, B))
bad = np.argwhere(C != B)
print("bad count", len(bad), bad[:10])
# where does C[i, j] come from? locate values
for (i, j) in [(0, 0), (0, 1), (0, 32), (1, 0), (8, 0), (0, 255), (3, 40)]:
    v = C[i, j]
    src = np.argwhere(B == v)
    print((i, j), v, "B has it at", src[:4].tolist())
