"""One gated-residual GEMM launch at the 240p proj shape (for ncu captures)."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
M, N, K = 2 * 6075, 1152, int(sys.argv[1]) if len(sys.argv) > 1 else 1152
a = torch.randn(M, K, device=dev).bfloat16()
w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
bias = torch.zeros(N, device=dev)
x = torch.randn(M, N, device=dev)
gate = torch.randn(2, N, device=dev)
o2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2, out2=o2, bn=192)
torch.cuda.synchronize()
print("done")
