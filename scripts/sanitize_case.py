"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one tiny STDiT3 step at DoP 1 (every step kernel: embeddings, LN, tcgen05 GEMMs with all
epilogues, FMHA, temporal attention, final layer), the same step as a DoP-2 virtual group with the
exchange fused into fc2 (peer stores + flag protocol), the staged (NCCL-arm) pack/unpack, a
re-shard and a tiny VAE decode.  Usage: compute-sanitizer --tool X python scripts/sanitize_case.py"""
import dataclasses
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, vae_weights as vw, weights
from paper_2506_13497_b200.executor import reshard
from paper_2506_13497_b200.stdit import STDiTModel, StagedVirtualGroup, StepRequest, VirtualGroup
from paper_2506_13497_b200.vae import VAEDecoder

dev = torch.device("cuda:0")
cfg = dataclasses.replace(weights.TINY, depth=1)
W = weights.init_weights(cfg, seed=3)
sh = shapes.shape_of("144p-16f")
z, y = weights.synthetic_inputs(cfg, sh.latent)
model = STDiTModel(cfg, W, dev)
r1 = StepRequest(model, sh, y.to(dev))
z1 = z.to(dev).contiguous()
r1.step(z1, 0)
grp = VirtualGroup(model, sh, y.to(dev), 2)
parts = grp.split(z.to(dev))
grp.step(parts, 0)
sg = StagedVirtualGroup(model, sh, y.to(dev), 2)
sparts = sg.split(z.to(dev))
sg.step(sparts, 0)
g4 = VirtualGroup(model, sh, y.to(dev), 4)
p4 = [torch.empty_like(p) for p in g4.split(z.to(dev))]
reshard(g4.ranks, p4, grp.ranks, parts)
torch.cuda.synchronize()
ok = torch.equal(torch.cat(parts, 2), z1) and torch.equal(torch.cat(sparts, 2), z1) \
    and torch.equal(torch.cat(p4, 2), z1)
dec = VAEDecoder(vw.TINY_VAE, vw.init_vae_weights(vw.TINY_VAE), dev)
v = dec.decode(z1, sh.frames, sh.height, sh.width)
torch.cuda.synchronize()
print("sanitize case done, dop2/staged/reshard bit-exact:", ok, "video", tuple(v.shape))
