"""Sweep BN x {1-CTA, 2-CTA} for the gated-residual GEMMs at the 240p shapes."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
M, N = 2 * 6075, 1152


def t_of(f, it=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


for K, copy in [(1152, True), (1152, False), (4608, False)]:
    a = torch.randn(M, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
    bias = torch.zeros(N, device=dev)
    x = torch.randn(M, N, device=dev)
    gate = torch.randn(2, N, device=dev)
    o2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16) if copy else None
    for two in (1, 0):
        _lib.lib().ddit_set_gemm_2cta(two)
        for bn in (96, 128, 192):
            f = lambda: kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2,
                                     out2=o2, bn=bn)
            t = t_of(f)
            g = lambda: kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, bn=bn)
            tp = t_of(g)
            print(f"K={K} copy={int(copy)} 2cta={two} bn={bn}: resid {t:6.1f} us  plain {tp:6.1f} us", flush=True)
    _lib.lib().ddit_set_gemm_2cta(1)

# QKV epilogue (bias + per-head RMSNorm + RoPE) at the 240p shape, vs the plain bf16 epilogue
K, N = 1152, 3456
a = torch.randn(M, K, device=dev).bfloat16()
w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
bias = torch.zeros(N, device=dev)
qw = torch.ones(72, device=dev)
tab = torch.randn(15, 36, 2, device=dev)
for two in (1, 0):
    _lib.lib().ddit_set_gemm_2cta(two)
    f = lambda: kernels.gemm(a, w, epi=_lib.EPI_QKV, bias=bias, qnorm_w=qw, knorm_w=qw, hidden=1152,
                             rope_tab=tab, rope_T=15, rope_S=1, bn=144)
    g = lambda: kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, bn=192)
    print(f"qkv 2cta={two}: qkv-epilogue {t_of(f):6.1f} us  plain(bn192) {t_of(g):6.1f} us", flush=True)
_lib.lib().ddit_set_gemm_2cta(1)
