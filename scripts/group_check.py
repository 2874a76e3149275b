"""Multi-process DoP-P check: P processes (torchrun), IPC-mapped exchange buffers, flag
barrier; the gathered z' must equal the single-process DoP-1 step bit for bit.
All ranks may share one GPU (the 1-GPU test box) or use one GPU each."""
import dataclasses
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.distributed as dist

from paper_2506_13497_b200 import shapes, weights
from paper_2506_13497_b200.dist import GroupStep
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
ngpu = torch.cuda.device_count()
dev = torch.device("cuda", rank % ngpu)
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
label = sys.argv[1] if len(sys.argv) > 1 else "144p"
cfg = dataclasses.replace(weights.TINY, depth=2)
W = weights.init_weights(cfg, seed=3)
sh = shapes.shape_of(label)
z, y = weights.synthetic_inputs(cfg, sh.latent)
model = STDiTModel(cfg, W, dev)
g = GroupStep(model, sh, y.to(dev))
zl = z[:, :, g.shard.t_lo:g.shard.t_hi].to(dev).contiguous()
for step in (0, 1):
    g.step(zl, step)
for step in (2, 3):  # CUDA-graph replays: the device-side exchange epoch must advance
    g.req.graph_step(zl, step)
torch.cuda.synchronize()
parts = [None] * world
dist.all_gather_object(parts, zl.cpu())
ok = True
if rank == 0:
    z1 = z.to(dev).contiguous()
    req = StepRequest(model, sh, y.to(dev))
    for step in (0, 1, 2, 3):
        req.step(z1, step)
    torch.cuda.synchronize()
    zp = torch.cat(parts, dim=2)
    diff = (zp - z1.cpu()).abs().max().item()
    ok = torch.equal(zp, z1.cpu())
    print(f"GROUP dop={world} label={label} max|diff|={diff} {'PASS' if ok else 'FAIL'}", flush=True)
dist.barrier()
g.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
