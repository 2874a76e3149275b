"""Golden vectors of the fp32 STDiT3 oracle (tiny config, 144p x 16 frames) -- the build's own
fixtures (the reference has no model code: parity for latents is unpinned by it).

    python tests/golden/make_stdit_golden.py
writes stdit_tiny_golden.pt: seeded inputs' checksums and z' after steps 0, 17, 29.
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import stdit3  # noqa: E402
from paper_2506_13497_b200 import shapes, weights  # noqa: E402


def main():
    cfg = weights.TINY
    W = weights.init_weights(cfg, seed=3)
    sh = shapes.shape_of("144p-16f")
    z, y = weights.synthetic_inputs(cfg, sh.latent)
    y2 = stdit3.prepare_text(W, y)
    out = {"z": z, "y_sum": y.double().sum().item(), "w_sum": sum(v.double().sum().item() for v in W.values())}
    for step in (0, 17, 29):
        out[f"z_{step}"] = stdit3.denoise_step(W, cfg, z, y2, step, sh.height, sh.width)
    torch.save(out, Path(__file__).with_name("stdit_tiny_golden.pt"))
    print("wrote stdit_tiny_golden.pt")


if __name__ == "__main__":
    main()
