"""One tcgen05 FMHA launch at a spatial shape (for ncu captures): python scripts/fmha_one.py S T."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import kernels

S = int(sys.argv[1]) if len(sys.argv) > 1 else 3600
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
H, C, B = 16, 1152, 2
qkv = torch.randn(B * T * S, 3 * C, device=dev).bfloat16()
o = torch.empty(B * T * S, C, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * T, Lq=S, Lk=S,
                      q_map=(1, S, 0, 1), kv_map=(1, S, 0, 1), tc=True)
torch.cuda.synchronize()
print("done")
