"""First timing of the XL/2 step at DoP 1 (device-resident inputs, CUDA events)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, weights
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

label = sys.argv[1] if len(sys.argv) > 1 else "240p"
dev = torch.device("cuda:0")
cfg = weights.XL2
t0 = time.time()
W = weights.init_weights(cfg, seed=3, device=dev)
print(f"init weights {time.time()-t0:.1f}s", flush=True)
model = STDiTModel(cfg, W, dev)
del W
sh = shapes.shape_of(label)
z, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
req = StepRequest(model, sh, y)
zd = z.contiguous()
for i in range(3):
    req.step(zd, i)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
n = 5
s.record()
for i in range(n):
    req.step(zd, 3 + i)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
T, S = sh.T, sh.S
C, L, Ly = 1152, 28, 300
N = T * S
F = 2 * (L * (2 * 28 * N * C * C + 2 * 4 * Ly * C * C + 4 * T * S * S * C + 4 * S * T * T * C + 2 * 4 * N * Ly * C) + 64 * N * C)
print(f"{label}: {ms:.2f} ms/step  {F/ms/1e9:.1f} TFLOP/s  (F={F/1e12:.2f} TF)  finite={torch.isfinite(zd).all().item()}", flush=True)
