"""A/B timing of the XL/2 step (DoP 1, device-resident z, eager launches + one graph pass) under
runtime switches that take effect at request open: ddit_set_resid_reduce (reduce-add vs load /
update / store residual epilogue).  Env switches (DDIT_LN, DDIT_FMHA_POLY, ...) need one process
each.  Usage: python scripts/ab_step.py 240p [label]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, shapes, weights
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

res = sys.argv[1] if len(sys.argv) > 1 else "240p"
label = sys.argv[2] if len(sys.argv) > 2 else ""
dev = torch.device("cuda:0")
cfg = weights.XL2
W = weights.init_weights(cfg, seed=3, device=dev)
model = STDiTModel(cfg, W, dev)
del W
sh = shapes.shape_of(res)
z0, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
L = _lib.lib()
outs = {}
for red in (1, 0, 1):
    L.ddit_set_resid_reduce(red)
    req = StepRequest(model, sh, y)
    z = z0.clone().contiguous()
    for i in range(3):
        req.step(z, i)
    torch.cuda.synchronize()
    zt = z0.clone().contiguous()
    req.step(zt, 5)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 8
    s.record()
    for i in range(n):
        req.step(z, 3 + i)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    outs.setdefault(red, zt)
    print(f"{res} {label} resid_reduce={red}: {ms:.3f} ms/step (eager)", flush=True)
    req.close()
L.ddit_set_resid_reduce(1)
print(f"{res} {label} reduce vs load/update/store step output bit-exact: {torch.equal(outs[0], outs[1])}")
