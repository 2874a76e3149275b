"""Timeline of CTA 0 in one gated-residual GEMM (proj shape, 2-CTA BN 192) from the
DDIT_EPI_TRACE build: MMA issuer (tmem-empty wait, first / last k-block) and epilogue warp 0
(tmem-full wait, per sub-tile residual-load wait and store issue), in microseconds from the
first event. Usage: DDIT_LIB=paper_2506_13497_b200/libddit_trace.so python scripts/epi_trace.py [K] [copy]"""
import ctypes
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
copy = len(sys.argv) > 2 and sys.argv[2] == "1"
qkv = len(sys.argv) > 2 and sys.argv[2] == "qkv"  # QKV shape + epilogue: MMA-side events only
fc1 = len(sys.argv) > 2 and sys.argv[2] == "fc1"  # fc1 shape + GELU epilogue: MMA-side events only
M, N = 2 * 6075, (3456 if qkv else 4608 if fc1 else 1152)
a = torch.randn(M, K, device=dev).bfloat16()
w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
bias = torch.zeros(N, device=dev)
x = torch.randn(M, N, device=dev)
gate = torch.randn(2, N, device=dev)
o2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16) if copy else None
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
L = _lib.lib()
L.ddit_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
for it in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    if fc1:
        kernels.gemm(a, w, epi=_lib.EPI_GELU_BF16, bias=bias)
    elif qkv:
        qw = torch.ones(72, device=dev)
        tab = torch.randn(15, 36, 2, device=dev)
        kernels.gemm(a, w, epi=_lib.EPI_QKV, bias=bias, qnorm_w=qw, knorm_w=qw, hidden=1152, rope_tab=tab,
                     rope_T=15, rope_S=405, bn=144)
    else:
        kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2, out2=o2)
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 1024)()
L.ddit_debug_trace(buf, 1024)
t = list(buf)
clk = 1.7e3  # cycles per us (approx; sm clock under load)
base = min(v for v in t if v)
us = lambda v: (v - base) / clk if v else float("nan")
print("events:", us(t[0]), us(t[1]), us(t[64]), us(t[65]), us(t[128]), us(t[129]))
ntiles = sum(1 for i in range(32) if t[2 * i])
if qkv or fc1:
    for i in range(ntiles):
        print(f"tile {i}: mma wait-empty {us(t[2*i]):7.2f} -> {us(t[2*i+1]):7.2f} (waited {us(t[2*i+1]) - us(t[2*i]):5.2f})"
              f"  kb0 {us(t[64+2*i]):7.2f} kblast {us(t[64+2*i+1]):7.2f}")
    sys.exit(0)
for i in range(ntiles):
    print(f"tile {i}: mma wait-empty {us(t[2*i]):7.2f} -> {us(t[2*i+1]):7.2f}  kb0 {us(t[64+2*i]):7.2f} kblast {us(t[64+2*i+1]):7.2f} | "
          f"epi wait-full {us(t[128+2*i]):7.2f} -> {us(t[128+2*i+1]):7.2f}")
    subs = []
    for s in range(6):
        subs.append(f"[wr {us(t[384+16*i+s]):6.2f} go {us(t[256+16*i+2*s]):6.2f} ld {us(t[256+16*i+2*s+1]):6.2f} "
                    f"tm {us(t[512+16*i+s]):6.2f} cp {us(t[768+16*i+s]):6.2f} st {us(t[640+16*i+s]):6.2f}]")
    print("\n".join("      " + x for x in subs if "nan" not in x))
