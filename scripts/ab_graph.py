"""Graph-replayed A/B of the XL/2 step under a runtime switch that takes effect at request open
(ddit_set_<name>(0|1)), interleaved A B A B ... so clock drift hits both arms alike; the step
output is checked bit-identical between arms. Only for switches whose effect is per request:
a switch that changes device state (an L2 persisting carve-out, persisting lines) leaks into the
other arm, which then measures the leftovers -- A/B those in separate processes.
Usage: python scripts/ab_graph.py <switch, e.g. fmha_l2pf[:0,1,2]> [res=240p] [rounds=4] [steps=20]"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import _lib, shapes, weights
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

name, _, vals = sys.argv[1].partition(":")
arms = [int(v) for v in vals.split(",")] if vals else [0, 1]
res = sys.argv[2] if len(sys.argv) > 2 else "240p"
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
dev = torch.device("cuda:0")
cfg = weights.XL2
W = weights.init_weights(cfg, seed=3, device=dev)
model = STDiTModel(cfg, W, dev)
del W
sh = shapes.shape_of(res)
z0, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
setter = getattr(_lib.lib(), "ddit_set_" + name)
reqs, outs = {}, {}
for on in arms:
    setter(on)
    req = StepRequest(model, sh, y)
    z = z0.clone().contiguous()
    req.graph_step(z, 5)
    torch.cuda.synchronize()
    outs[on] = z.clone()
    reqs[on] = (req, z)
setter(1)
times = {a: [] for a in arms}
for r in range(rounds):
    for on in arms if r % 2 == 0 else arms[::-1]:
        req, z = reqs[on]
        for i in range(3):
            req.graph_step(z, i)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for i in range(steps):
            req.graph_step(z, 3 + i % 20)
        e.record()
        torch.cuda.synchronize()
        times[on].append(s.elapsed_time(e) / steps)
for on in arms:
    t = times[on]
    print(f"{res} {name}={on}: median {statistics.median(t):.3f} ms/step  all "
          + " ".join(f"{x:.3f}" for x in t), flush=True)
same = all(torch.equal(outs[arms[0]], outs[a]) for a in arms)
print(f"{res} {name}: step output bit-identical between arms: {same}")
for on in arms:
    reqs[on][0].close()
