"""ORACLE (test infrastructure only) -- fp32 CPU restatement of the OpenSora-1.2 VAE decode.

Parity status: unpinned by the reference (it has no model code: the VAE is the lookup
``ProfileTable.vae``, reference pkg/src/ditsim/profiles.py:78-85). Restates the public
definitions ([EXT]; PAPER.md:550 names OpenSoraVAE):

* ``VideoAutoencoderPipeline.decode``: ``z * scale + shift``; the temporal VAE decodes each
  micro-batch of ``micro_z`` latent frames into ``min(17, remaining)`` frames; the spatial VAE
  decodes every frame;
* OpenSora ``VAE_Temporal`` decoder: CausalConv3d (zero front padding of kt-1 frames, "same"
  spatial padding), ResBlocks GN(32, eps 1e-5) -> SiLU -> conv -> GN -> SiLU -> conv (+ 1x1x1
  shortcut when channels change), temporal upsampling conv f -> 2f then
  "B (C ts) T H W -> B C (T ts) H W", final GN -> SiLU -> conv, drop the front time padding;
* diffusers ``AutoencoderKL`` decoder: z / scaling_factor -> post_quant_conv -> conv_in ->
  mid (ResnetBlock2D, single-head Attention with GroupNorm and residual, ResnetBlock2D) ->
  up blocks (layers_per_block + 1 ResnetBlock2D, nearest x2 + conv except the last) ->
  GN(eps 1e-6) -> SiLU -> conv_out.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def _w(W, name):  # [Cout, kt, kh, kw, Cin] -> torch conv3d weight [Cout, Cin, kt, kh, kw]
    return W[name + ".weight"].permute(0, 4, 1, 2, 3)


def causal_conv3d(W, name, x, bias=True):
    w = _w(W, name)
    kt, kh, kw = w.shape[2:]
    x = F.pad(x, (kw // 2, kw // 2, kh // 2, kh // 2, kt - 1, 0))
    return F.conv3d(x, w, W.get(name + ".bias") if bias else None)


def conv2d(W, name, x):
    w = _w(W, name)[:, :, 0]
    return F.conv2d(x, w, W[name + ".bias"], padding=w.shape[-1] // 2)


def gn(W, name, x, groups, eps):
    return F.group_norm(x, groups, W[name + ".weight"], W[name + ".bias"], eps)


# ------------------------------------------------------------------ temporal VAE decoder
def t_resblock(W, cfg, name, x):
    h = F.silu(gn(W, name + ".norm1", x, cfg.groups, cfg.t_eps))
    h = causal_conv3d(W, name + ".conv1", h, bias=False)
    h = F.silu(gn(W, name + ".norm2", h, cfg.groups, cfg.t_eps))
    h = causal_conv3d(W, name + ".conv2", h, bias=False)
    if (name + ".conv3.weight") in W:
        x = causal_conv3d(W, name + ".conv3", x, bias=False)
    return x + h


def temporal_decode(W, cfg, z, num_frames: int):
    """z [B, 4, t, h, w] -> [B, 4, num_frames, h, w]."""
    tf = cfg.time_factor
    time_padding = 0 if num_frames % tf == 0 else tf - num_frames % tf
    x = causal_conv3d(W, "t.post_quant_conv", z)
    x = causal_conv3d(W, "t.conv1", x)
    for i in range(cfg.t_res_blocks):
        x = t_resblock(W, cfg, f"t.res_blocks.{i}", x)
    for i in reversed(range(len(cfg.t_mults))):
        for j in range(cfg.t_res_blocks):
            x = t_resblock(W, cfg, f"t.block_res_blocks.{i}.{j}", x)
        if i > 0 and cfg.t_downsample[i - 1]:
            x = causal_conv3d(W, f"t.conv_blocks.{i - 1}", x)
            B, C2, T, H, Wd = x.shape
            x = x.view(B, C2 // 2, 2, T, H, Wd).permute(0, 1, 3, 2, 4, 5).reshape(B, C2 // 2, 2 * T, H, Wd)
    x = F.silu(gn(W, "t.norm1", x, cfg.groups, cfg.t_eps))
    x = causal_conv3d(W, "t.conv_out", x)
    return x[:, :, time_padding:]


# ------------------------------------------------------------------ spatial VAE decoder
def s_resblock(W, cfg, name, x):
    h = F.silu(gn(W, name + ".norm1", x, cfg.groups, cfg.sd_eps))
    h = conv2d(W, name + ".conv1", h)
    h = F.silu(gn(W, name + ".norm2", h, cfg.groups, cfg.sd_eps))
    h = conv2d(W, name + ".conv2", h)
    if (name + ".conv_shortcut.weight") in W:
        x = conv2d(W, name + ".conv_shortcut", x)
    return x + h


def mid_attention(W, cfg, x):
    B, C, H, Wd = x.shape
    h = gn(W, "s.mid.attn.group_norm", x, cfg.groups, cfg.sd_eps)
    h = h.view(B, C, H * Wd).transpose(1, 2)
    p = "s.mid.attn."
    q = F.linear(h, W[p + "to_q.weight"], W[p + "to_q.bias"])
    k = F.linear(h, W[p + "to_k.weight"], W[p + "to_k.bias"])
    v = F.linear(h, W[p + "to_v.weight"], W[p + "to_v.bias"])
    a = torch.softmax(q @ k.transpose(1, 2) / C**0.5, dim=-1) @ v
    o = F.linear(a, W[p + "to_out.weight"], W[p + "to_out.bias"])
    return x + o.transpose(1, 2).reshape(B, C, H, Wd)


def spatial_decode(W, cfg, z):
    """z [N, 4, h, w] -> frames [N, 3, 8h, 8w]."""
    x = conv2d(W, "s.post_quant_conv", z / cfg.scaling_factor)
    x = conv2d(W, "s.conv_in", x)
    x = s_resblock(W, cfg, "s.mid.resnets.0", x)
    x = mid_attention(W, cfg, x)
    x = s_resblock(W, cfg, "s.mid.resnets.1", x)
    n = len(cfg.block_out)
    for i in range(n):
        for j in range(cfg.layers_per_block + 1):
            x = s_resblock(W, cfg, f"s.up.{i}.resnets.{j}", x)
        if i < n - 1:
            x = F.interpolate(x, scale_factor=2.0, mode="nearest")
            x = conv2d(W, f"s.up.{i}.upsample", x)
    x = F.silu(gn(W, "s.norm_out", x, cfg.groups, cfg.sd_eps))
    return conv2d(W, "s.conv_out", x)


def vae_decode(W, cfg, z, num_frames: int, height: int, width: int):
    """VideoAutoencoderPipeline.decode: z [B, 4, T, h, w] -> video [B, 3, num_frames, H, W]."""
    sc = torch.tensor(cfg.scale).view(1, -1, 1, 1, 1)
    sh = torch.tensor(cfg.shift).view(1, -1, 1, 1, 1)
    z = z * sc + sh
    chunks = []
    left = num_frames
    for i in range(0, z.shape[2], cfg.micro_z):
        chunks.append(temporal_decode(W, cfg, z[:, :, i:i + cfg.micro_z], min(cfg.micro_frame_size, left)))
        left -= cfg.micro_frame_size
    x = torch.cat(chunks, dim=2)  # [B, 4, F, h, w]
    B, C, Fr, h, w = x.shape
    frames = spatial_decode(W, cfg, x.permute(0, 2, 1, 3, 4).reshape(B * Fr, C, h, w))
    frames = frames.view(B, Fr, 3, 8 * h, 8 * w).permute(0, 2, 1, 3, 4)
    return frames[:, :, :, :height, :width]
