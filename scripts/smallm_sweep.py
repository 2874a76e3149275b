"""GEMM tile choices at the small per-rank M of DoP 4/8 (calibrates gemm_pick_tile)."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")


def t_of(f, it=40):
    """Device time per launch from a CUDA graph of `it` launches (the host-side plan building of
    kernels.gemm -- tensor-map encoding -- would otherwise dominate at these sizes)."""
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            f()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


for M in (1620, 3060, 6120):
    for (N, K, epi) in ((1152, 1152, _lib.EPI_BF16), (1152, 4608, _lib.EPI_RESID), (4608, 1152, _lib.EPI_GELU_BF16)):
        a = torch.randn(M, K, device=dev).bfloat16()
        w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
        bias = torch.zeros(N, device=dev)
        x = torch.randn(M, N, device=dev)
        res = []
        for two in (1, 0):
            _lib.lib().ddit_set_gemm_2cta(two)
            for bn in (96, 128, 192, 256):
                if N % bn:
                    continue
                if epi == _lib.EPI_RESID:
                    f = lambda: kernels.gemm(a, w, epi=epi, bias=bias, resid=x, rows_per_b=M, bn=bn)
                else:
                    f = lambda: kernels.gemm(a, w, epi=epi, bias=bias, bn=bn)
                res.append((t_of(f), f"{'2cta' if two else '1cta'}-{bn}"))
        _lib.lib().ddit_set_gemm_2cta(1)
        res.sort()
        print(f"M={M} N={N} K={K} epi={epi}: " + "  ".join(f"{n} {t:.1f}" for t, n in res), flush=True)
