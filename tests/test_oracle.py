"""CPU tests of the fp32 STDiT3 oracle: building blocks against independent formulations,
and the committed golden vectors (regression pin)."""
import math
from pathlib import Path

import torch
import torch.nn.functional as F

from oracle import stdit3
from paper_2506_13497_b200 import shapes, weights

GOLD = Path(__file__).parent / "golden" / "stdit_tiny_golden.pt"


def test_rope_matches_complex_rotation():
    torch.manual_seed(0)
    x = torch.randn(3, 5, 72)
    pos = torch.arange(5)
    got = stdit3.rope_interleaved(x, pos)
    theta = 1.0 / (10000 ** (torch.arange(0, 72, 2).float() / 72))
    ang = pos[:, None].float() * theta[None]
    xc = torch.view_as_complex(x.reshape(3, 5, 36, 2).contiguous())
    ref = torch.view_as_real(xc * torch.polar(torch.ones_like(ang), ang)).reshape(3, 5, 72)
    assert torch.allclose(got, ref, atol=1e-5)


def test_pos_embed_matches_literal_opensora_meshgrid():
    """Literal transcription of OpenSora PositionEmbedding2D._get_cached_emb ([EXT])."""
    C, h, w, scale, base = 64, 5, 7, 0.6, 6
    half = C // 2
    inv_freq = 1.0 / (10000 ** (torch.arange(0, half, 2).float() / half))
    grid_h = torch.arange(h) / scale * (base / h)
    grid_w = torch.arange(w) / scale * (base / w)
    grid_h, grid_w = torch.meshgrid(grid_w, grid_h, indexing="ij")
    grid_h = grid_h.t().reshape(-1)
    grid_w = grid_w.t().reshape(-1)

    def sc(t):
        o = torch.einsum("i,d->id", t, inv_freq)
        return torch.cat((torch.sin(o), torch.cos(o)), dim=-1)

    ref = torch.cat([sc(grid_h), sc(grid_w)], dim=-1)
    assert torch.allclose(stdit3.pos_embed_2d(C, h, w, scale, base), ref, atol=1e-6)


def test_self_attention_matches_sdpa():
    cfg = weights.STDiTConfig(depth=1, hidden=144, heads=2)
    W = weights.init_weights(cfg, seed=1)
    x = torch.randn(3, 11, 144)
    p = "spatial_blocks.0."
    got = stdit3.self_attention(W, p, cfg, x, rope=False)
    qkv = F.linear(x, W[p + "attn.qkv.weight"], W[p + "attn.qkv.bias"]).view(3, 11, 3, 2, 72)
    q, k, v = qkv.permute(2, 0, 3, 1, 4)
    q = stdit3.rms_norm(q, W[p + "attn.q_norm.weight"])
    k = stdit3.rms_norm(k, W[p + "attn.k_norm.weight"])
    o = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(3, 11, 144)
    ref = F.linear(o, W[p + "attn.proj.weight"], W[p + "attn.proj.bias"])
    assert torch.allclose(got, ref, atol=1e-5)


def test_timestep_transform_matches_opensora_formula_for_51_frames():
    h, w, T = 240, 426, 15
    ts = stdit3.sampling_timesteps(30, h, w, T)
    nf = 51 // 17 * 5  # OpenSora's num_frames // 17 * 5
    ratio = math.sqrt(h * w / 512 ** 2) * math.sqrt(nf)
    for i, t in enumerate(ts):
        u = 1 - i / 30
        assert abs(t - ratio * u / (1 + (ratio - 1) * u) * 1000) < 1e-9
    assert ts[0] == 1000.0


def test_unpatchify_inverts_patch_order():
    """Feature f = (hp*2 + wp)*C_out + c of token (t, i, j) lands at [c, t, 2i+hp, 2j+wp]."""
    cfg = weights.STDiTConfig(depth=0, hidden=144, heads=2)
    B, T, h, w = 1, 2, 3, 4
    oc = cfg.out_channels
    feats = torch.arange(B * T * h * w * 4 * oc, dtype=torch.float32).view(B, T, h, w, 2, 2, oc)
    out = feats.permute(0, 6, 1, 2, 4, 3, 5).reshape(B, oc, T, 2 * h, 2 * w)
    assert out[0, 3, 1, 2 * 2 + 1, 2 * 3 + 0] == feats[0, 1, 2, 3, 1, 0, 3]


def test_golden_vectors_reproduce():
    g = torch.load(GOLD)
    cfg = weights.TINY
    W = weights.init_weights(cfg, seed=3)
    sh = shapes.shape_of("144p-16f")
    z, y = weights.synthetic_inputs(cfg, sh.latent)
    assert torch.equal(z, g["z"])
    assert abs(y.double().sum().item() - g["y_sum"]) < 1e-6
    y2 = stdit3.prepare_text(W, y)
    z1 = stdit3.denoise_step(W, cfg, z, y2, 17, sh.height, sh.width)
    assert torch.allclose(z1, g["z_17"], rtol=1e-5, atol=1e-6)
