"""OpenSora-1.2 VAE decoder configuration and seeded random-init weights.

The paper decodes with OpenSoraVAE: ``VideoAutoencoderPipeline`` = a causal
temporal VAE (``VAE_Temporal_SD``: filters 128, multipliers (1,2,2,4), 4 res blocks, temporal
upsampling in the two top levels) applied per 17-frame micro-batch (5 latent frames), followed
by the SDXL spatial VAE decoder (``AutoencoderKL``: blocks (128,256,512,512), 2 layers + 1,
single-head mid attention) per frame, after ``z * scale + shift`` ([EXT] public definitions;
the reference only looks the VAE time up, profiles.py:78-85). No checkpoints exist here:
weights are random (fan-in scaled) so outputs are non-trivial.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class VAEConfig:
    latent_channels: int = 4
    # spatial (SDXL VAE decoder)
    block_out: tuple[int, ...] = (128, 256, 512, 512)
    layers_per_block: int = 2
    groups: int = 32
    sd_eps: float = 1e-6
    scaling_factor: float = 0.13025
    # temporal (OpenSora VAE_Temporal_SD decoder)
    t_filters: int = 128
    t_mults: tuple[int, ...] = (1, 2, 2, 4)
    t_res_blocks: int = 4
    t_downsample: tuple[bool, ...] = (False, True, True)
    t_eps: float = 1e-5
    micro_frame_size: int = 17
    scale: tuple[float, ...] = (3.85, 2.32, 2.33, 3.06)
    shift: tuple[float, ...] = (0.0, 0.22, 0.19, 0.17)

    @property
    def time_factor(self) -> int:
        return 2 ** sum(self.t_downsample)

    @property
    def micro_z(self) -> int:
        t = self.micro_frame_size
        pad = 0 if t % self.time_factor == 0 else self.time_factor - t % self.time_factor
        return (t + pad) // self.time_factor


OPENSORA_VAE = VAEConfig()
# reduced widths for CPU-oracle parity tests (tensor-core convs need multiples of 64 channels,
# the single-head mid attention GEMMs 128)
TINY_VAE = VAEConfig(block_out=(64, 64, 128, 128), layers_per_block=1, t_filters=64,
                     t_mults=(1, 1, 1, 2), t_res_blocks=1)


def vae_param_shapes(cfg: VAEConfig) -> list[tuple[str, tuple[int, ...], str]]:
    """(name, shape, kind). Conv weights are [Cout, kt, kh, kw, Cin] (channels-last K)."""
    L = cfg.latent_channels
    out: list[tuple[str, tuple[int, ...], str]] = []

    def conv(name, cin, cout, k, bias=True):
        out.append((name + ".weight", (cout, *k, cin), "conv"))
        if bias:
            out.append((name + ".bias", (cout,), "bias"))

    def norm(name, c):
        out.append((name + ".weight", (c,), "gamma"))
        out.append((name + ".bias", (c,), "beta"))

    # ---- temporal decoder
    top = cfg.t_filters * cfg.t_mults[-1]
    conv("t.post_quant_conv", L, L, (1, 1, 1))
    conv("t.conv1", L, top, (3, 3, 3))

    def t_res(name, cin, cout):
        norm(name + ".norm1", cin)
        conv(name + ".conv1", cin, cout, (3, 3, 3), bias=False)
        norm(name + ".norm2", cout)
        conv(name + ".conv2", cout, cout, (3, 3, 3), bias=False)
        if cin != cout:
            conv(name + ".conv3", cin, cout, (1, 1, 1), bias=False)

    for i in range(cfg.t_res_blocks):
        t_res(f"t.res_blocks.{i}", top, top)
    prev = top
    for i in reversed(range(len(cfg.t_mults))):
        f = cfg.t_filters * cfg.t_mults[i]
        for j in range(cfg.t_res_blocks):
            t_res(f"t.block_res_blocks.{i}.{j}", prev, f)
            prev = f
        if i > 0 and cfg.t_downsample[i - 1]:
            conv(f"t.conv_blocks.{i - 1}", prev, prev * 2, (3, 3, 3))
    norm("t.norm1", prev)
    conv("t.conv_out", prev, L, (3, 3, 3))
    # ---- spatial decoder (2-D convs stored with kt = 1)
    rev = list(reversed(cfg.block_out))
    conv("s.post_quant_conv", L, L, (1, 1, 1))
    conv("s.conv_in", L, rev[0], (1, 3, 3))

    def s_res(name, cin, cout):
        norm(name + ".norm1", cin)
        conv(name + ".conv1", cin, cout, (1, 3, 3))
        norm(name + ".norm2", cout)
        conv(name + ".conv2", cout, cout, (1, 3, 3))
        if cin != cout:
            conv(name + ".conv_shortcut", cin, cout, (1, 1, 1))

    s_res("s.mid.resnets.0", rev[0], rev[0])
    norm("s.mid.attn.group_norm", rev[0])
    for nm in ("to_q", "to_k", "to_v", "to_out"):
        out.append((f"s.mid.attn.{nm}.weight", (rev[0], rev[0]), "linear"))
        out.append((f"s.mid.attn.{nm}.bias", (rev[0],), "bias"))
    s_res("s.mid.resnets.1", rev[0], rev[0])
    prev = rev[0]
    for i, ch in enumerate(rev):
        for j in range(cfg.layers_per_block + 1):
            s_res(f"s.up.{i}.resnets.{j}", prev, ch)
            prev = ch
        if i < len(rev) - 1:
            conv(f"s.up.{i}.upsample", ch, ch, (1, 3, 3))
    norm("s.norm_out", prev)
    conv("s.conv_out", prev, 3, (1, 3, 3))
    return out


def init_vae_weights(cfg: VAEConfig, seed: int = 7, device="cpu") -> dict[str, torch.Tensor]:
    g = torch.Generator(device=device).manual_seed(seed)
    W: dict[str, torch.Tensor] = {}
    for name, shape, kind in vae_param_shapes(cfg):
        if kind == "conv":
            fan_in = math.prod(shape[1:])
            t = torch.randn(shape, generator=g, device=device) / math.sqrt(fan_in)
        elif kind == "linear":
            t = torch.randn(shape, generator=g, device=device) / math.sqrt(shape[1])
        elif kind == "bias":
            t = 0.02 * torch.randn(shape, generator=g, device=device)
        elif kind == "gamma":
            t = 1.0 + 0.1 * torch.randn(shape, generator=g, device=device)
        else:  # beta
            t = 0.1 * torch.randn(shape, generator=g, device=device)
        W[name] = t.float()
    return W
