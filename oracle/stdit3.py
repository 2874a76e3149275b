"""ORACLE (test infrastructure only) -- fp32 CPU restatement of one STDiT3 denoise step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this module, and only as the checker / the timed CPU baseline -- never as the product path.

Parity status: **unpinned by the reference.** The reference (arxiv 2506.13497 ``ditsim``)
contains no model code: the denoise step is the lookup ``ProfileTable.dit_step``
(reference pkg/src/ditsim/profiles.py:69-76) and real execution is out of scope
(reference SPEC.md:16). This file restates the public OpenSora-1.2 STDiT3 + RFLOW sampler
([EXT]; the paper names them at PAPER.md:546-557) so the CUDA path has a numeric oracle;
golden vectors under tests/golden are generated from it by tests/golden/make_stdit_golden.py.

Conventions pinned here (the CUDA path must follow them):
* blocks: adaLN ``x*(1+scale)+shift`` after a non-affine LayerNorm(eps 1e-6); self-attention
  with qkv bias, per-head LlamaRMSNorm on q,k, interleaved RoPE (rotary-embedding-torch
  "lang" frequencies, theta 10000, dim 72) on q,k in temporal blocks only, scale 1/sqrt(72);
  gated residual; cross-attention (no norm) of each sample's tokens onto its own 300 text
  tokens; tanh-GELU MLP; gated residual.
* spatial blocks attend within a frame (S tokens), temporal blocks across frames (T tokens).
* t embedding: 256-d sinusoid (cos, sin) -> Linear, SiLU, Linear; + fps embedding (same
  form); t_block = SiLU -> Linear(C, 6C); final layer uses t (not t_block).
* RFLOW: 30 steps, timesteps (1 - i/30) * 1000, timestep transform with ratio =
  sqrt(H*W / 512^2) * sqrt(T_latent), CFG guidance 7.0 with ``u + g (c - u)`` on the first
  4 of 8 output channels, Euler ``z += v * dt / 1000``. (OpenSora uses num_frames//17*5 for
  the temporal ratio; that equals T_latent for 51/102 frames and would collapse the 16-frame
  tiny config to t = 0, so T_latent is used.)
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

NUM_TIMESTEPS = 1000


# ------------------------------------------------------------------ embeddings
def timestep_embedding(t: torch.Tensor, dim: int = 256, max_period: float = 10000.0) -> torch.Tensor:
    half = dim // 2
    freqs = torch.exp(-math.log(max_period) * torch.arange(half, dtype=torch.float32) / half)
    args = t[:, None].float() * freqs[None]
    return torch.cat([torch.cos(args), torch.sin(args)], dim=-1)


def _mlp2(W, p, x, act):
    x = F.linear(x, W[p + "0.weight"], W[p + "0.bias"])
    x = act(x)
    return F.linear(x, W[p + "2.weight"], W[p + "2.bias"])


def t_embed(W, cfg, timestep: torch.Tensor, fps: float) -> torch.Tensor:
    B = timestep.shape[0]
    t = _mlp2(W, "t_embedder.mlp.", timestep_embedding(timestep, cfg.freq_dim), F.silu)
    f = torch.full((B,), float(fps))
    t = t + _mlp2(W, "fps_embedder.mlp.", timestep_embedding(f, cfg.freq_dim), F.silu)
    return t


def t_block(W, t):
    return F.linear(F.silu(t), W["t_block.1.weight"], W["t_block.1.bias"])


def y_embed(W, y: torch.Tensor) -> torch.Tensor:
    h = F.linear(y, W["y_embedder.y_proj.fc1.weight"], W["y_embedder.y_proj.fc1.bias"])
    h = F.gelu(h, approximate="tanh")
    return F.linear(h, W["y_embedder.y_proj.fc2.weight"], W["y_embedder.y_proj.fc2.bias"])


def pos_embed_2d(C: int, h: int, w: int, scale: float, base_size: int) -> torch.Tensor:
    """[h*w, C] sin-cos embedding ([EXT] OpenSora PositionEmbedding2D, w-major meshgrid)."""
    half = C // 2
    inv_freq = 1.0 / (10000 ** (torch.arange(0, half, 2).float() / half))
    gh = torch.arange(h, dtype=torch.float32) / scale * (base_size / h)
    gw = torch.arange(w, dtype=torch.float32) / scale * (base_size / w)
    # token s = i*w + j sits at row gh[i], column gw[j]. OpenSora builds the grid with
    # meshgrid(grid_w, grid_h) ("w goes first"), so the FIRST half of the embedding encodes
    # the column coordinate and the second half the row coordinate.
    row = gh[:, None].expand(h, w).reshape(-1)
    col = gw[None, :].expand(h, w).reshape(-1)

    def sincos(p):
        out = p[:, None] * inv_freq[None]
        return torch.cat([torch.sin(out), torch.cos(out)], dim=-1)

    return torch.cat([sincos(col), sincos(row)], dim=-1)


def patch_embed(W, x: torch.Tensor) -> torch.Tensor:
    """[B, 4, T, Hl, Wl] -> [B, T*S, C] (zero-pads odd Hl/Wl like PatchEmbed3D)."""
    _, _, T, H, Wd = x.shape
    if Wd % 2:
        x = F.pad(x, (0, 1))
    if H % 2:
        x = F.pad(x, (0, 0, 0, 1))
    y = F.conv3d(x, W["x_embedder.proj.weight"], W["x_embedder.proj.bias"], stride=(1, 2, 2))
    return y.flatten(2).transpose(1, 2)


# ------------------------------------------------------------------ attention pieces
def rms_norm(x, w, eps=1e-6):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def rope_interleaved(x: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """x [..., L, D]; rotate pairs (2i, 2i+1) by pos * theta_i, theta_i = 10000^(-2i/D)."""
    D = x.shape[-1]
    theta = 1.0 / (10000 ** (torch.arange(0, D, 2)[: D // 2].float() / D))
    ang = pos.float()[:, None] * theta[None]  # [L, D/2]
    c, s = torch.cos(ang), torch.sin(ang)
    x2 = x.unflatten(-1, (D // 2, 2))
    a, b = x2[..., 0], x2[..., 1]
    return torch.stack([a * c - b * s, b * c + a * s], dim=-1).flatten(-2)


def self_attention(W, p, cfg, x, rope: bool):
    """x [Bq, L, C] (sequences) -> [Bq, L, C]."""
    Bq, L, C = x.shape
    H, D = cfg.heads, cfg.head_dim
    qkv = F.linear(x, W[p + "attn.qkv.weight"], W[p + "attn.qkv.bias"])
    q, k, v = qkv.view(Bq, L, 3, H, D).permute(2, 0, 3, 1, 4).unbind(0)
    q = rms_norm(q, W[p + "attn.q_norm.weight"], cfg.eps)
    k = rms_norm(k, W[p + "attn.k_norm.weight"], cfg.eps)
    if rope:
        pos = torch.arange(L)
        q = rope_interleaved(q, pos)
        k = rope_interleaved(k, pos)
    # sequences in chunks so the fp32 score matrix stays <= ~1 GB (720p: L = 3600 tokens)
    step = max(1, (1 << 28) // (H * L * L))
    o = torch.cat([((q[i:i + step] * D**-0.5) @ k[i:i + step].transpose(-2, -1)).softmax(-1)
                   @ v[i:i + step] for i in range(0, Bq, step)], 0)
    o = o.transpose(1, 2).reshape(Bq, L, C)
    return F.linear(o, W[p + "attn.proj.weight"], W[p + "attn.proj.bias"])


def cross_attention(W, p, cfg, x, y):
    """x [B, N, C] attends to its own sample's text y [B, Ly, C] (block-diagonal mask)."""
    B, N, C = x.shape
    H, D = cfg.heads, cfg.head_dim
    q = F.linear(x, W[p + "cross_attn.q_linear.weight"], W[p + "cross_attn.q_linear.bias"])
    kv = F.linear(y, W[p + "cross_attn.kv_linear.weight"], W[p + "cross_attn.kv_linear.bias"])
    q = q.view(B, N, H, D).transpose(1, 2)
    k, v = kv.view(B, -1, 2, H, D).permute(2, 0, 3, 1, 4).unbind(0)
    o = ((q * D**-0.5) @ k.transpose(-2, -1)).softmax(-1) @ v
    o = o.transpose(1, 2).reshape(B, N, C)
    return F.linear(o, W[p + "cross_attn.proj.weight"], W[p + "cross_attn.proj.bias"])


def layer_norm(x, eps=1e-6):
    return F.layer_norm(x, (x.shape[-1],), eps=eps)


def block(W, cfg, kind: str, i: int, x, y, t_mlp, T: int, S: int):
    """One STDiT3 block. x [B, T*S, C] in (t, s) token order."""
    p = f"{kind}_blocks.{i}."
    B, N, C = x.shape
    mod = W[p + "scale_shift_table"][None] + t_mlp.view(B, 6, C)
    shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp = mod.unbind(1)
    xm = layer_norm(x, cfg.eps) * (1 + scale_msa[:, None]) + shift_msa[:, None]
    if kind == "temporal":
        xs = xm.view(B, T, S, C).transpose(1, 2).reshape(B * S, T, C)
        o = self_attention(W, p, cfg, xs, rope=True)
        o = o.view(B, S, T, C).transpose(1, 2).reshape(B, N, C)
    else:
        xs = xm.view(B * T, S, C)
        o = self_attention(W, p, cfg, xs, rope=False).view(B, N, C)
    x = x + gate_msa[:, None] * o
    x = x + cross_attention(W, p, cfg, x, y)
    xm = layer_norm(x, cfg.eps) * (1 + scale_mlp[:, None]) + shift_mlp[:, None]
    h = F.gelu(F.linear(xm, W[p + "mlp.fc1.weight"], W[p + "mlp.fc1.bias"]), approximate="tanh")
    h = F.linear(h, W[p + "mlp.fc2.weight"], W[p + "mlp.fc2.bias"])
    return x + gate_mlp[:, None] * h


# ------------------------------------------------------------------ model + sampler
def forward(W, cfg, x, timestep, y_emb, height: int, width: int, fps: float = 24.0,
            depth: int | None = None):
    """STDiT3 forward. x [B, 4, T, Hl, Wl]; y_emb [B, Ly, C] (already y-embedded).
    Returns [B, out_channels, T, Hl, Wl]."""
    B, _, T, Hl, Wl = x.shape
    h, w = (Hl + 1) // 2, (Wl + 1) // 2
    S = h * w
    C = cfg.hidden
    base_size = round(S**0.5)
    scale = math.sqrt(height * width) / cfg.input_sq_size
    pos = pos_embed_2d(C, h, w, scale, base_size)
    t = t_embed(W, cfg, timestep, fps)
    t_mlp = t_block(W, t)
    xt = patch_embed(W, x).view(B, T, S, C) + pos[None, None]
    xt = xt.reshape(B, T * S, C)
    nd = cfg.depth if depth is None else depth
    for i in range(nd):
        xt = block(W, cfg, "spatial", i, xt, y_emb, t_mlp, T, S)
        xt = block(W, cfg, "temporal", i, xt, y_emb, t_mlp, T, S)
    # final layer
    sst = W["final_layer.scale_shift_table"][None] + t[:, None]
    shift, scale_ = sst.unbind(1)
    xt = layer_norm(xt, cfg.eps) * (1 + scale_[:, None]) + shift[:, None]
    xt = F.linear(xt, W["final_layer.linear.weight"], W["final_layer.linear.bias"])
    # unpatchify: features ordered (hp, wp, c)
    oc = cfg.out_channels
    xt = xt.view(B, T, h, w, 2, 2, oc).permute(0, 6, 1, 2, 4, 3, 5).reshape(B, oc, T, 2 * h, 2 * w)
    return xt[:, :, :, :Hl, :Wl]


def sampling_timesteps(num_steps: int, height: int, width: int, t_latent: int) -> list[float]:
    ts = [(1.0 - i / num_steps) * NUM_TIMESTEPS for i in range(num_steps)]
    ratio = math.sqrt(height * width / (512 * 512)) * math.sqrt(t_latent)
    out = []
    for t in ts:
        u = t / NUM_TIMESTEPS
        out.append(ratio * u / (1 + (ratio - 1) * u) * NUM_TIMESTEPS)
    return out


def prepare_text(W, y_cond: torch.Tensor) -> torch.Tensor:
    """CFG text batch [y; y_null] through the y-embedder -> [2, Ly, C]."""
    y_null = W["y_embedder.y_embedding"][None]
    return y_embed(W, torch.cat([y_cond, y_null], 0))


def denoise_step(W, cfg, z: torch.Tensor, y_emb2: torch.Tensor, step: int, height: int,
                 width: int, num_steps: int = 30, guidance: float = 7.0, fps: float = 24.0,
                 depth: int | None = None) -> torch.Tensor:
    """One RFLOW Euler step with classifier-free guidance. z [1, 4, T, Hl, Wl] fp32."""
    T = z.shape[2]
    ts = sampling_timesteps(num_steps, height, width, T)
    t = torch.tensor([ts[step]] * 2, dtype=torch.float32)
    pred = forward(W, cfg, torch.cat([z, z], 0), t, y_emb2, height, width, fps, depth)
    pred = pred[:, : cfg.in_channels]
    cond, uncond = pred.chunk(2, dim=0)
    v = uncond + guidance * (cond - uncond)
    dt = (ts[step] - ts[step + 1]) if step < num_steps - 1 else ts[step]
    return z + v * (dt / NUM_TIMESTEPS)
