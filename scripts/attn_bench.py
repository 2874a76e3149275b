"""Microbenchmark the attention kernels at the 240p XL/2 shapes (spatial, cross, temporal)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import kernels

dev = torch.device("cuda:0")
H, D, C = 16, 72, 1152
B, T, S, Ly = 2, 15, 405, 300
M = B * T * S
qkv = torch.randn(M, 3 * C, device=dev).bfloat16()
o = torch.empty(M, C, device=dev, dtype=torch.bfloat16)
q = torch.randn(M, C, device=dev).bfloat16()
kv = torch.randn(B * Ly, 2 * C, device=dev).bfloat16()


def timeit(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3


fl_sp = 4 * B * T * S * S * C
fl_cr = 4 * M * Ly * C
for tc in (True,):
    t = timeit(lambda: kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * T,
                                         Lq=S, Lk=S, q_map=(1, S, 0, 1), kv_map=(1, S, 0, 1), tc=tc))
    print(f"spatial tc={tc}: {t:7.1f} us  {fl_sp / t / 1e6:6.1f} TF/s", flush=True)
    t = timeit(lambda: kernels.attention(q, kv[:, :C], kv[:, C:], o, heads=H, num_seqs=B, Lq=T * S, Lk=Ly,
                                         q_map=(1, T * S, 0, 1), kv_map=(1, Ly, 0, 1), tc=tc))
    print(f"cross   tc={tc}: {t:7.1f} us  {fl_cr / t / 1e6:6.1f} TF/s", flush=True)
mp = (S, T * S, 1, S)
t = timeit(lambda: kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * S,
                                     Lq=T, Lk=T, q_map=mp, kv_map=mp, temporal=True))
print(f"temporal fast: {t:7.1f} us  {M * 4 * C * 2 / t / 1e3:6.1f} GB/s (q,k,v read + o write)", flush=True)
# long-sequence regime (720p spatial: S=3600)
S2, T2 = 3600, 2
qkv2 = torch.randn(B * T2 * S2, 3 * C, device=dev).bfloat16()
o2 = torch.empty(B * T2 * S2, C, device=dev, dtype=torch.bfloat16)
fl2 = 4 * B * T2 * S2 * S2 * C
for tc in (True,):
    t = timeit(lambda: kernels.attention(qkv2[:, :C], qkv2[:, C:2 * C], qkv2[:, 2 * C:], o2, heads=H, num_seqs=B * T2,
                                         Lq=S2, Lk=S2, q_map=(1, S2, 0, 1), kv_map=(1, S2, 0, 1), tc=tc), it=5)
    print(f"spatial720 tc={tc}: {t:7.1f} us  {fl2 / t / 1e6:6.1f} TF/s", flush=True)
# temporal attention in the long-clip regime (480p/720p x 102 frames: T = 30)
for (T3, S3) in ((30, 1620), (30, 3600)):
    M3 = B * T3 * S3
    qkv3 = torch.randn(M3, 3 * C, device=dev).bfloat16()
    o3 = torch.empty(M3, C, device=dev, dtype=torch.bfloat16)
    mp3 = (S3, T3 * S3, 1, S3)
    t = timeit(lambda: kernels.attention(qkv3[:, :C], qkv3[:, C:2 * C], qkv3[:, 2 * C:], o3, heads=H,
                                         num_seqs=B * S3, Lq=T3, Lk=T3, q_map=mp3, kv_map=mp3, temporal=True), it=5)
    print(f"temporal T={T3} S={S3}: {t:7.1f} us  {M3 * 4 * C * 2 / t / 1e3:6.1f} GB/s "
          f"{4 * B * S3 * T3 * T3 * C / t / 1e6:6.1f} TF/s", flush=True)
    del qkv3, o3
