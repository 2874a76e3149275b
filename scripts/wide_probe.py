"""2-CTA GEMM with 256 x 2BN tiles (DDIT_GEMM_WIDE=1) vs 256 x BN at the N = 1152 step shapes
(fc2 / cross-proj reduce-add epilogue, cross-q plain bf16): graph-timed, and the outputs of both
tilings compared bit for bit (saved to / checked against /tmp/wide_probe_ref.pt)."""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, kernels

dev = torch.device("cuda:0")
wide = os.environ.get("DDIT_GEMM_WIDE", "0") == "1"


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


M = 12150
g = torch.Generator(device=dev).manual_seed(0)
outs = {}
for name, N, K, red in [("fc2", 1152, 4608, True), ("cproj", 1152, 1152, True), ("crossq", 1152, 1152, False)]:
    a = torch.randn(M, K, device=dev, generator=g).bfloat16()
    w = (torch.randn(N, K, device=dev, generator=g) / math.sqrt(K)).bfloat16()
    bias = torch.randn(N, device=dev, generator=g)
    gate = torch.randn(2, N, device=dev, generator=g)
    if red:
        x0 = torch.randn(M, N, device=dev, generator=g)
        x = x0.clone()
        f = lambda: kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2,  # noqa
                                 bn=192, stream=torch.cuda.current_stream())
        x.copy_(x0)
        f()
        torch.cuda.synchronize()
        outs[name] = x.clone()
    else:
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        f = lambda: kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, out=out, bn=192,  # noqa
                                 stream=torch.cuda.current_stream())
        f()
        torch.cuda.synchronize()
        outs[name] = out.clone()
    t = gtime(f)
    print(f"{name:7s} wide={int(wide)}: {t*1e3:7.1f} us {2*M*N*K/t/1e9:7.1f} TF/s", flush=True)
ref = "/tmp/wide_probe_ref.pt"
if not wide:
    torch.save({k: v.cpu() for k, v in outs.items()}, ref)
elif os.path.exists(ref):
    r = torch.load(ref)
    for k, v in outs.items():
        print(k, "bit-exact vs 256 x BN tiles:", torch.equal(v.cpu(), r[k]))
