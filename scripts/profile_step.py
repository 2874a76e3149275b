"""Run 2 XL/2 steps (for ncu launch lists / captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, weights
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

label = sys.argv[1] if len(sys.argv) > 1 else "240p"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
cfg = weights.XL2
W = weights.init_weights(cfg, seed=3, device=dev)
model = STDiTModel(cfg, W, dev)
del W
sh = shapes.shape_of(label)
z, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
req = StepRequest(model, sh, y)
z = z.contiguous()
for i in range(nsteps):
    req.step(z, i)
torch.cuda.synchronize()
print("done")
