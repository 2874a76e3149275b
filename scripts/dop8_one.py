"""One 240p XL/2 step as a DoP-8 virtual group on one GPU (for ncu launch lists of the small-M
per-rank kernels): python scripts/dop8_one.py [label] [dop]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, weights
from paper_2506_13497_b200.stdit import STDiTModel, VirtualGroup

label = sys.argv[1] if len(sys.argv) > 1 else "240p"
dop = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda:0")
cfg = weights.XL2
W = weights.init_weights(cfg, seed=3, device=dev)
model = STDiTModel(cfg, W, dev)
del W
sh = shapes.shape_of(label)
z, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
grp = VirtualGroup(model, sh, y, dop)
parts = grp.split(z)
for i in range(2):
    grp.step(parts, i)
torch.cuda.synchronize()
print("done")
