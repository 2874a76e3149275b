"""Time the gated-residual GEMMs at the 240p shapes (proj / cross-proj with bf16 copy / fc2) with
rotating buffers larger than L2, for the library named by DDIT_LIB (A/B of build variants).
Usage: DDIT_LIB=... python scripts/resid_ab.py"""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
M, N, SETS = 2 * 6075, 1152, 4


def t_of(fs, it=24):
    for f in fs:
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for i in range(it):
        fs[i % len(fs)]()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


res = []
for K, copy in [(1152, False), (1152, True), (4608, False)]:
    fs = []
    for _ in range(SETS):
        a = torch.randn(M, K, device=dev).bfloat16()
        w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
        bias = torch.zeros(N, device=dev)
        x = torch.randn(M, N, device=dev)
        gate = torch.randn(2, N, device=dev)
        o2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16) if copy else None
        fs.append(lambda a=a, w=w, bias=bias, x=x, gate=gate, o2=o2: kernels.gemm(
            a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2, out2=o2))
    res.append(f"K={K} copy={int(copy)}: {t_of(fs):6.1f} us")
print(os.path.basename(str(_lib.LIB_PATH)), " | ".join(res), flush=True)
