"""Timeline of CTA 0 of the temporal-attention kernel (DDIT_TA_TRACE build):
python scripts/build_variant.py tatrace attention_temporal.cu -DDDIT_TA_TRACE
DDIT_LIB=paper_2506_13497_b200/libddit_tatrace.so python scripts/ta_trace.py T S"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import kernels
from paper_2506_13497_b200._lib import lib

T, S = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
H, C, B = 16, 1152, 2
M = B * T * S
qkv = torch.randn(M, 3 * C, device=dev).bfloat16()
o = torch.empty(M, C, device=dev, dtype=torch.bfloat16)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
mp = (S, T * S, 1, S)
for _ in range(3):
    flush.zero_()
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * S, Lq=T, Lk=T,
                      q_map=mp, kv_map=mp, temporal=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
lib().ddit_ta_trace(buf, 1024)
t0 = buf[1023]
names = ["issued", "landed", "QK", "S_read", "P_st", "PV", "epi_done"]
print("unit " + " ".join(f"{n:>9s}" for n in names))
for u in range(0, 40):
    row = [buf[8 * u + k] for k in range(7)]
    if all(v == 0 for v in row):
        break
    print(f"{u:4d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in row))
