"""QKV GEMM (M = 12150, N = 3456, K = 1152) at the 240p step shape: plain bf16 epilogue at
BN 128 / 144 / 192 vs the fused RMSNorm (+RoPE) epilogue at BN 144, graph-timed."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")


def gtime(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(it):
                fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(3):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (3 * it)


M, N, K = 12150, 3456, 1152
a = torch.randn(M, K, device=dev).bfloat16()
w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
bias = torch.zeros(N, device=dev)
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
fl = 2 * M * N * K
for bn in (128, 192):
    t = gtime(lambda: kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, out=out, bn=bn,
                                   stream=torch.cuda.current_stream()))
    print(f"plain bn={bn}: {t*1e3:7.1f} us {fl/t/1e9:7.1f} TF/s", flush=True)
qw = torch.ones(72, device=dev)
tab = torch.randn(15, 36, 2, device=dev)
for rope in (False, True):
    t = gtime(lambda: kernels.gemm(a, w, epi=_lib.EPI_QKV, bias=bias, out=out, qnorm_w=qw, knorm_w=qw, hidden=1152,
                                   rope_tab=tab if rope else None, rope_T=15, rope_S=405, bn=144,
                                   stream=torch.cuda.current_stream()))
    print(f"qkv epilogue bn=144 rope={rope}: {t*1e3:7.1f} us {fl/t/1e9:7.1f} TF/s", flush=True)
# per-head padded weights (80-row slots): the 256 x 240 tile
wp = torch.zeros(48 * 80, K, device=dev, dtype=torch.bfloat16)
bp = torch.zeros(48 * 80, device=dev)
for h in range(48):
    wp[h * 80:h * 80 + 72] = w[h * 72:(h + 1) * 72]
for rope in (False, True):
    t = gtime(lambda: kernels.gemm(a, wp, epi=_lib.EPI_QKV, bias=bp, out=out, qnorm_w=qw, knorm_w=qw, hidden=1152,
                                   rope_tab=tab if rope else None, rope_T=15, rope_S=405, bn=240,
                                   stream=torch.cuda.current_stream()))
    print(f"qkv epilogue padded bn=240 rope={rope}: {t*1e3:7.1f} us {fl/t/1e9:7.1f} TF/s (algorithmic)", flush=True)
