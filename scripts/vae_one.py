"""One OpenSora VAE decode of a latent (for ncu launch lists): python scripts/vae_one.py 240p."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, vae_weights as vw
from paper_2506_13497_b200.vae import VAEDecoder

sh = shapes.shape_of(sys.argv[1] if len(sys.argv) > 1 else "240p")
cfg = vw.OPENSORA_VAE
dev = torch.device("cuda:0")
dec = VAEDecoder(cfg, vw.init_vae_weights(cfg, device=dev), dev)
z = torch.randn(1, 4, *sh.latent, device=dev)
dec.decode(z, sh.frames, sh.height, sh.width)
torch.cuda.synchronize()
print("launches per decode", dec.launches // 1)
