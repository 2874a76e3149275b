"""Timeline of CTA 0 in one tcgen05 FMHA launch from the DDIT_FMHA_TRACE build (per softmax group
and tile: S ready, MUFU token, exps done, P buffer free, P stored; per unit: O ready, O stored;
MMA warps: QK / PV issue), in cycles from the first event.
Usage: DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so python scripts/fmha_trace.py cross|spatial|720"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
mode = sys.argv[1] if len(sys.argv) > 1 else "cross"
H, D, C = 16, 72, 1152
L = _lib.lib()
L.ddit_fmha_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
g = torch.Generator(device=dev).manual_seed(0)
if mode == "cross":
    B, N, Ly = 2, 6075, 300
    q = torch.randn(B * N, C, device=dev, generator=g).bfloat16()
    kv = torch.randn(B * Ly, 2 * C, device=dev, generator=g).bfloat16()
    o = torch.empty(B * N, C, device=dev, dtype=torch.bfloat16)

    def run():
        kernels.attention(q, kv[:, :C], kv[:, C:], o, heads=H, num_seqs=B, Lq=N, Lk=Ly,
                          q_map=(1, N, 0, 1), kv_map=(1, Ly, 0, 1), tc=True)
else:
    S, T = (405, 30) if mode == "spatial" else (3600, 60)
    qkv = torch.randn(T * S, 3 * C, device=dev, generator=g).bfloat16()
    o = torch.empty(T * S, C, device=dev, dtype=torch.bfloat16)

    def run():
        kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=T,
                          Lq=S, Lk=S, q_map=(1, S, 0, 1), kv_map=(1, S, 0, 1), tc=True)
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(f"{mode}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per launch")
buf = (ctypes.c_ulonglong * 2048)()
L.ddit_fmha_trace(buf, 2048)
v = list(buf)
t0 = min(x for x in v if x) if any(v) else 0


def rel(x):
    return (x - t0) if x else -1


names = ["S_wait", "S_rdy", "tok", "exps", "Pfree", "Pst", "O_rdy", "O_st"]
for grp in (0, 1):
    print(f"softmax group {grp}: tile: " + " ".join(f"{n:>7}" for n in names) + "   QKiss   PViss")
    for n in range(64):
        row = [rel(v[grp * 512 + n * 8 + 7])] + [rel(v[grp * 512 + n * 8 + k]) for k in range(7)]
        mm = [rel(v[1024 + grp * 256 + n * 2 + k]) for k in range(2)]
        if row[0] < 0 and mm[0] < 0:
            continue
        print(f"  {n:3d}: " + " ".join(f"{x:7d}" for x in row) + "  " + " ".join(f"{x:7d}" for x in mm))

print("MMA warps per unit: q_wait_start  q_full  k_full(t0)  s_free(t0)")
for grp in (0, 1):
    for u in range(32):
        row = [rel(v[1536 + grp * 128 + u * 4 + k]) for k in range(4)]
        if row[0] < 0:
            continue
        print(f"  g{grp} unit {u:2d}: " + " ".join(f"{x:7d}" for x in row))
print("producer per unit: start  Q_issued  K(t0)_issued  V(last)_issued")
for u in range(64):
    row = [rel(v[1792 + u * 4 + k]) for k in range(4)]
    if row[0] < 0:
        continue
    print(f"  unit {u:2d}: " + " ".join(f"{x:7d}" for x in row))
