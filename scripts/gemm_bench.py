"""Time the STDiT3-XL/2 240p GEMM shapes on tcgen05 (ours) vs torch.matmul (cuBLAS)."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
M = 2 * 6075


def gtime(fn, it=20):
    """Device time per call of fn, replayed from a CUDA graph of `it` calls (the per-call host
    work -- plan / tensor-map encode -- happens once, at capture)."""
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
shapes = [("qkv", 3456, 1152, 192, _lib.EPI_BF16), ("proj", 1152, 1152, 128, _lib.EPI_BF16),
          ("fc1", 4608, 1152, 256, _lib.EPI_GELU_BF16), ("fc2", 1152, 4608, 128, _lib.EPI_BF16),
          ("fc1_192", 4608, 1152, 192, _lib.EPI_GELU_BF16), ("proj192", 1152, 1152, 192, _lib.EPI_BF16),
          ("big", 8192, 8192, 256, _lib.EPI_BF16)]
for name, N, K, bn, epi in shapes:
    m = M if name != "big" else 8192
    a = torch.randn(m, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
    bias = torch.zeros(N, device=dev)
    out = torch.empty(m, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        kernels.gemm(a, w, epi=epi, bias=bias, out=out, bn=bn)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    it = 20
    s.record()
    for _ in range(it):
        kernels.gemm(a, w, epi=epi, bias=bias, out=out, bn=bn)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / it
    for _ in range(3):
        torch.matmul(a, w.T)
    s.record()
    for _ in range(it):
        torch.matmul(a, w.T)
    e.record(); torch.cuda.synchronize()
    tc = s.elapsed_time(e) / it
    fl = 2 * m * N * K
    print(f"{name:8s} M={m} N={N} K={K} bn={bn}: ours {t*1e3:8.1f} us {fl/t/1e9:7.1f} TF/s | cublas {tc*1e3:8.1f} us {fl/tc/1e9:7.1f} TF/s", flush=True)

# fp32 residual epilogue (proj / cproj / fc2): resid[m, n] += gate[b, n] * (a @ w.T + bias), with
# and without the bf16 copy; reported against HBM bytes as well as FLOPs
for name, N, K, bn, copy in [("proj_resid", 1152, 1152, 192, True), ("cproj_resid", 1152, 1152, 192, False),
                             ("fc2_resid", 1152, 4608, 192, False), ("proj_r128", 1152, 1152, 128, True)]:
    m = M
    a = torch.randn(m, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
    bias = torch.zeros(N, device=dev)
    x = torch.randn(m, N, device=dev)
    gate = torch.randn(2, N, device=dev)
    o2 = torch.empty(m, N, device=dev, dtype=torch.bfloat16) if copy else None
    f = lambda: kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=m // 2,
                             out2=o2, bn=bn)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    it = 20
    s.record()
    for _ in range(it):
        f()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / it
    fl = 2 * m * N * K
    byt = m * K * 2 + N * K * 2 + m * N * 8 + (m * N * 2 if copy else 0)
    print(f"{name:11s} M={m} N={N} K={K} bn={bn}: {t*1e3:8.1f} us {fl/t/1e9:7.1f} TF/s "
          f"{byt/t/1e6:7.1f} GB/s (compulsory {byt/1e6:.0f} MB)", flush=True)

# reduce-add vs load / update / store residual epilogue (no copy), same shapes
L = _lib.lib()
for name, N, K, bn in [("cproj", 1152, 1152, 192), ("fc2", 1152, 4608, 192), ("cproj128", 1152, 1152, 128)]:
    m = M
    a = torch.randn(m, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) / math.sqrt(K)).bfloat16()
    bias = torch.zeros(N, device=dev)
    x = torch.randn(m, N, device=dev)
    gate = torch.randn(2, N, device=dev)
    for red in (1, 0):
        L.ddit_set_resid_reduce(red)
        f = lambda: kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=m // 2,
                                 bn=bn, stream=torch.cuda.current_stream())
        t = gtime(f)
        print(f"{name:9s} red={red}: {t*1e3:8.1f} us {2*m*N*K/t/1e9:7.1f} TF/s (graph)", flush=True)
    # and the same with the bf16 copy (proj)
    o2 = torch.empty(m, N, device=dev, dtype=torch.bfloat16)
    f = lambda: kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=m // 2,
                             out2=o2, bn=bn, stream=torch.cuda.current_stream())
    t = gtime(f)
    print(f"{name:9s} copy : {t*1e3:8.1f} us {2*m*N*K/t/1e9:7.1f} TF/s (graph)", flush=True)
    out = torch.empty(m, N, device=dev, dtype=torch.bfloat16)
    f = lambda: kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, out=out, bn=bn, stream=torch.cuda.current_stream())
    t = gtime(f)
    print(f"{name:9s} plain: {t*1e3:8.1f} us {2*m*N*K/t/1e9:7.1f} TF/s (graph)", flush=True)
    L.ddit_set_resid_reduce(1)
