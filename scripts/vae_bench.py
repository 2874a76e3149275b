"""Time the full OpenSora VAE decode of a 240p x 51 latent on one B200."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, vae_weights as vw
from paper_2506_13497_b200.vae import VAEDecoder, vae_flops

label = sys.argv[1] if len(sys.argv) > 1 else "240p"
sh = shapes.shape_of(label)
cfg = vw.OPENSORA_VAE
dev = torch.device("cuda:0")
dec = VAEDecoder(cfg, vw.init_vae_weights(cfg, device=dev), dev, graphs=1 if sh.height <= 240 else 0)
z = torch.randn(1, 4, *sh.latent, device=dev)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
fl = vae_flops(cfg, sh.frames, sh.T, *sh.latent[1:])
for mode in ("eager", "graph") if dec.max_graphs else ("eager",):
    fn = dec.decode_eager if mode == "eager" else dec.decode
    for _ in range(2):
        out = fn(z, sh.frames, sh.height, sh.width)
    torch.cuda.synchronize()
    n0 = dec.launches
    s.record()
    out = fn(z, sh.frames, sh.height, sh.width)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"VAE decode {label}x{sh.frames} ({mode}): {ms:.1f} ms, {fl / 1e12:.1f} TFLOP -> "
          f"{fl / ms / 1e9:.0f} TFLOP/s, launches {dec.launches - n0}, out {tuple(out.shape)} "
          f"finite={torch.isfinite(out).all().item()}")
# VAE DoP q: each rank decodes its block of frames (vae.vae_shard); the DoP-q
# decode latency is the slowest rank's (ranks run one after another on this GPU)
from paper_2506_13497_b200.vae import vae_shard  # noqa: E402

for q in (2, 4):
    per = []
    for r in range(q):
        t_lo, t_hi, f_lo, f_hi = vae_shard(cfg, sh.T, sh.frames, q, r)
        if f_hi <= f_lo:
            continue
        zp = z[:, :, t_lo:t_hi].contiguous()
        f0 = t_lo // cfg.micro_z * cfg.micro_frame_size
        nf = min(-(-(t_hi - t_lo) // cfg.micro_z) * cfg.micro_frame_size, sh.frames - f0)
        dec.decode_eager(zp, nf, sh.height, sh.width, frames=(f_lo - f0, f_hi - f0))
        s.record()
        dec.decode_eager(zp, nf, sh.height, sh.width, frames=(f_lo - f0, f_hi - f0))
        e.record()
        torch.cuda.synchronize()
        per.append(s.elapsed_time(e))
    print(f"VAE decode {label}x{sh.frames} at VAE DoP {q}: per-rank ms {[round(x, 1) for x in per]} "
          f"-> {max(per):.1f} ms")
