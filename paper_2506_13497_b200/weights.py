"""STDiT3 configuration and seeded random-init weights.

There are no checkpoints (no network); weights are random-initialised from a seed with a
non-degenerate scheme (SURVEY.md §8(d) "Weight init for parity"): STDiT's zero-init of the
gates / final projection would make every output trivially equal, so instead

* every Linear / patch-embed weight: xavier_uniform,
* every bias: N(0, 0.02),
* per-block ``scale_shift_table`` [6, C] and the final [2, C] table: N(0, 1) / sqrt(C),
* qk RMSNorm weights: 1 + 0.1 N(0, 1),
* the null caption embedding ``y_embedding`` [300, 4096]: N(0, 1) / sqrt(4096).

Parameter names follow the public OpenSora-1.2 STDiT3 state dict ([EXT]; the paper names
the model at PAPER.md:548). The same dict feeds the fp32 CPU oracle (tests only) and the
device copies used by libddit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class STDiTConfig:
    depth: int = 28
    hidden: int = 1152
    heads: int = 16
    mlp_ratio: float = 4.0
    in_channels: int = 4
    pred_sigma: bool = True
    caption_channels: int = 4096
    text_tokens: int = 300
    freq_dim: int = 256
    input_sq_size: int = 512
    eps: float = 1e-6

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def mlp_hidden(self) -> int:
        return int(self.hidden * self.mlp_ratio)

    @property
    def out_channels(self) -> int:
        return self.in_channels * 2 if self.pred_sigma else self.in_channels

    @property
    def patch_out(self) -> int:
        return self.out_channels * 4  # patch (1, 2, 2)


XL2 = STDiTConfig()  # OpenSora STDiT3-XL/2: 28 layers, hidden 1152, 16 heads x 72
TINY = STDiTConfig(depth=2, hidden=288, heads=4)  # same head_dim 72


def config_by_name(name: str) -> STDiTConfig:
    return {"xl2": XL2, "tiny": TINY}[name]


def param_shapes(cfg: STDiTConfig) -> list[tuple[str, tuple[int, ...], str]]:
    """(name, shape, init-kind) in a fixed order (the RNG stream order)."""
    C, F, Y = cfg.hidden, cfg.freq_dim, cfg.caption_channels
    out: list[tuple[str, tuple[int, ...], str]] = [
        ("x_embedder.proj.weight", (C, cfg.in_channels, 1, 2, 2), "xavier"),
        ("x_embedder.proj.bias", (C,), "bias"),
        ("t_embedder.mlp.0.weight", (C, F), "xavier"),
        ("t_embedder.mlp.0.bias", (C,), "bias"),
        ("t_embedder.mlp.2.weight", (C, C), "xavier"),
        ("t_embedder.mlp.2.bias", (C,), "bias"),
        ("fps_embedder.mlp.0.weight", (C, F), "xavier"),
        ("fps_embedder.mlp.0.bias", (C,), "bias"),
        ("fps_embedder.mlp.2.weight", (C, C), "xavier"),
        ("fps_embedder.mlp.2.bias", (C,), "bias"),
        ("t_block.1.weight", (6 * C, C), "xavier"),
        ("t_block.1.bias", (6 * C,), "bias"),
        ("y_embedder.y_proj.fc1.weight", (C, Y), "xavier"),
        ("y_embedder.y_proj.fc1.bias", (C,), "bias"),
        ("y_embedder.y_proj.fc2.weight", (C, C), "xavier"),
        ("y_embedder.y_proj.fc2.bias", (C,), "bias"),
        ("y_embedder.y_embedding", (cfg.text_tokens, Y), "null"),
    ]
    for kind in ("spatial", "temporal"):
        for i in range(cfg.depth):
            p = f"{kind}_blocks.{i}."
            out += [
                (p + "scale_shift_table", (6, C), "table"),
                (p + "attn.qkv.weight", (3 * C, C), "xavier"),
                (p + "attn.qkv.bias", (3 * C,), "bias"),
                (p + "attn.q_norm.weight", (cfg.head_dim,), "norm"),
                (p + "attn.k_norm.weight", (cfg.head_dim,), "norm"),
                (p + "attn.proj.weight", (C, C), "xavier"),
                (p + "attn.proj.bias", (C,), "bias"),
                (p + "cross_attn.q_linear.weight", (C, C), "xavier"),
                (p + "cross_attn.q_linear.bias", (C,), "bias"),
                (p + "cross_attn.kv_linear.weight", (2 * C, C), "xavier"),
                (p + "cross_attn.kv_linear.bias", (2 * C,), "bias"),
                (p + "cross_attn.proj.weight", (C, C), "xavier"),
                (p + "cross_attn.proj.bias", (C,), "bias"),
                (p + "mlp.fc1.weight", (cfg.mlp_hidden, C), "xavier"),
                (p + "mlp.fc1.bias", (cfg.mlp_hidden,), "bias"),
                (p + "mlp.fc2.weight", (C, cfg.mlp_hidden), "xavier"),
                (p + "mlp.fc2.bias", (C,), "bias"),
            ]
    out += [
        ("final_layer.scale_shift_table", (2, C), "table"),
        ("final_layer.linear.weight", (cfg.patch_out, C), "xavier"),
        ("final_layer.linear.bias", (cfg.patch_out,), "bias"),
    ]
    return out


def init_weights(cfg: STDiTConfig, seed: int = 3, device="cpu") -> dict[str, torch.Tensor]:
    """Seeded fp32 weights. CPU and CUDA generators give different streams: parity tests
    always initialise on the CPU and copy."""
    g = torch.Generator(device=device).manual_seed(seed)
    W: dict[str, torch.Tensor] = {}
    for name, shape, kind in param_shapes(cfg):
        if kind == "xavier":
            fan_out = shape[0]
            fan_in = int(math.prod(shape[1:]))
            bound = math.sqrt(6.0 / (fan_in + fan_out))
            t = (torch.rand(shape, generator=g, device=device) * 2 - 1) * bound
        elif kind == "bias":
            t = torch.randn(shape, generator=g, device=device) * 0.02
        elif kind == "table":
            t = torch.randn(shape, generator=g, device=device) / math.sqrt(cfg.hidden)
        elif kind == "norm":
            t = 1.0 + 0.1 * torch.randn(shape, generator=g, device=device)
        elif kind == "null":
            t = torch.randn(shape, generator=g, device=device) / math.sqrt(shape[-1])
        else:  # pragma: no cover
            raise ValueError(kind)
        W[name] = t.float()
    return W


def synthetic_inputs(cfg: STDiTConfig, latent: tuple[int, int, int], seed_z: int = 0,
                     seed_y: int = 1, device="cpu"):
    """z ~ N(0,1) [1, 4, T, Hl, Wl] and caption embedding y ~ N(0,1) [1, 300, 4096]."""
    gz = torch.Generator(device=device).manual_seed(seed_z)
    gy = torch.Generator(device=device).manual_seed(seed_y)
    T, H, W = latent
    z = torch.randn((1, cfg.in_channels, T, H, W), generator=gz, device=device)
    y = torch.randn((1, cfg.text_tokens, cfg.caption_channels), generator=gy, device=device)
    return z, y
