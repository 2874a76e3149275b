"""Temporal attention (tcgen05 kernel) at the step shapes: 240p (T=15, S=405), 480p / 720p x 102
(T=30, S=1620 / 3600), B=2, XL/2 heads. Cold (L2 flushed before every launch) and hot times,
HBM GB/s of the compulsory traffic (q, k, v read once + o written once)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import kernels

dev = torch.device("cuda:0")
H, D, C, B = 16, 72, 1152, 2
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(T, S, it=10):
    M = B * T * S
    qkv = torch.randn(M, 3 * C, device=dev).bfloat16()
    o = torch.empty(M, C, device=dev, dtype=torch.bfloat16)
    mp = (S, T * S, 1, S)
    fn = lambda: kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H,  # noqa: E731
                                   num_seqs=B * S, Lq=T, Lk=T, q_map=mp, kv_map=mp, temporal=True)
    for _ in range(3):
        fn()
    cold = []
    for _ in range(it):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        cold.append(s.elapsed_time(e) * 1e3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(it):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    hot = s.elapsed_time(e) * 1e3 / it
    cold.sort()
    c = cold[len(cold) // 2]
    byts = M * 4 * C * 2
    print(f"temporal T={T:2d} S={S:4d}: cold {c:7.1f} us ({byts / c / 1e3:6.0f} GB/s)  "
          f"hot(graph) {hot:7.1f} us ({byts / hot / 1e3:6.0f} GB/s)  {byts / 1e6:.0f} MB", flush=True)


for T, S in ((15, 405), (30, 1620), (30, 3600)):
    run(T, S)
