"""tcgen05 implicit-GEMM convolution vs torch fp32 conv (same op, same bf16-rounded inputs)."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return (torch.linalg.vector_norm(a.float() - b.float()) / torch.linalg.vector_norm(b.float())).item()


def ref_conv(x, w, bias, residual, causal):
    # x [B,T,H,W,C] -> torch NCTHW
    xt = x.float().permute(0, 4, 1, 2, 3)
    wt = w.float().permute(0, 4, 1, 2, 3)
    kt, kh, kw = w.shape[1:4]
    pt = (kt - 1, 0) if causal else (kt // 2, kt // 2)
    xt = F.pad(xt, (kw // 2, kw // 2, kh // 2, kh // 2, *pt))
    y = F.conv3d(xt, wt, bias.float() if bias is not None else None)
    y = y.permute(0, 2, 3, 4, 1)
    if residual is not None:
        y = y + residual.float()
    return y


@pytest.mark.parametrize("B,T,H,W,Cin,Cout,k", [
    (2, 1, 30, 54, 128, 256, (1, 3, 3)),     # 2-D, narrow frame (2 rows per tile)
    (1, 1, 60, 107, 64, 128, (1, 3, 3)),     # odd width
    (1, 1, 24, 300, 128, 64, (1, 3, 3)),     # wide frame (3 column tiles)
    (1, 5, 12, 20, 128, 128, (3, 3, 3)),     # causal 3-D
    (2, 3, 8, 16, 64, 256, (1, 1, 1)),       # 1x1 shortcut
    (1, 4, 10, 10, 256, 512, (3, 3, 3)),
])
@pytest.mark.parametrize("with_res", [False, True])
def test_conv_matches_torch(cuda, B, T, H, W, Cin, Cout, k, with_res):
    from paper_2506_13497_b200 import kernels

    g = torch.Generator().manual_seed(0)
    x = torch.randn(B, T, H, W, Cin, generator=g).to(cuda, torch.bfloat16)
    w = (torch.randn(Cout, *k, Cin, generator=g) / (Cin * k[0] * k[1] * k[2]) ** 0.5).to(cuda, torch.bfloat16)
    bias = (0.1 * torch.randn(Cout, generator=g)).to(cuda)
    res = torch.randn(B, T, H, W, Cout, generator=g).to(cuda, torch.bfloat16) if with_res else None
    y = kernels.conv(x, w, bias=bias, residual=res, causal_time=True)
    ref = ref_conv(x, w, bias, res, True)
    torch.cuda.synchronize()
    assert rel_l2(y, ref) < 1e-2


@pytest.mark.parametrize("B,T,H,W,Cin,Cout,k", [
    (1, 3, 61, 107, 128, 256, (1, 3, 3)),    # 183 pixel tiles: the last pair has a lone tile
    (1, 4, 30, 54, 256, 128, (3, 3, 3)),     # causal 3-D, 2 rows per tile
    (2, 2, 45, 80, 64, 64, (1, 3, 3)),       # BN 64: 32 weight rows per CTA
])
@pytest.mark.parametrize("with_res", [False, True])
def test_conv_cta_pairs_bit_identical(cuda, B, T, H, W, Cin, Cout, k, with_res):
    """cta_group::2 conv tiles (pairs of 128-pixel tiles, half the weight rows per CTA) against
    the 1-CTA kernel, bit for bit, and against torch fp32."""
    from paper_2506_13497_b200 import _lib, kernels

    g = torch.Generator().manual_seed(1)
    x = torch.randn(B, T, H, W, Cin, generator=g).to(cuda, torch.bfloat16)
    w = (torch.randn(Cout, *k, Cin, generator=g) / (Cin * k[0] * k[1] * k[2]) ** 0.5).to(cuda, torch.bfloat16)
    bias = (0.1 * torch.randn(Cout, generator=g)).to(cuda)
    res = torch.randn(B, T, H, W, Cout, generator=g).to(cuda, torch.bfloat16) if with_res else None
    ys = []
    for pair in (1, 0):
        _lib.lib().ddit_set_conv_2cta(pair)
        try:
            ys.append(kernels.conv(x, w, bias=bias, residual=res, causal_time=True))
        finally:
            _lib.lib().ddit_set_conv_2cta(1)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1])
    assert rel_l2(ys[0], ref_conv(x, w, bias, res, True)) < 1e-2


@pytest.mark.parametrize("H,W,Cin,Cout", [(24, 432, 128, 128), (30, 216, 64, 256), (12, 108, 256, 64)])
def test_conv_tile_shapes_bit_identical(cuda, H, W, Cin, Cout):
    """Per-layer pixel-tile shapes (16 x 8, 32 x 4, ... chosen for the fewest tiles) against the
    128-pixel-row tiles, bit for bit."""
    from paper_2506_13497_b200 import _lib, kernels

    g = torch.Generator().manual_seed(2)
    x = torch.randn(2, 1, H, W, Cin, generator=g).to(cuda, torch.bfloat16)
    w = (torch.randn(Cout, 1, 3, 3, Cin, generator=g) / (Cin * 9) ** 0.5).to(cuda, torch.bfloat16)
    bias = (0.1 * torch.randn(Cout, generator=g)).to(cuda)
    ys = []
    for search in (1, 0):
        _lib.lib().ddit_set_conv_tile_search(search)
        try:
            ys.append(kernels.conv(x, w, bias=bias, causal_time=False))
        finally:
            _lib.lib().ddit_set_conv_tile_search(1)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1])
    assert rel_l2(ys[0], ref_conv(x, w, bias, None, False)) < 1e-2


@pytest.mark.parametrize("B,T,H,W,Cin,Cout,with_res,per_sample", [
    (2, 1, 30, 54, 128, 256, False, False),   # 2 rows per tile, 108 of 128 tile rows used
    (1, 3, 61, 107, 128, 256, True, False),   # ragged tiles, lone last pair tile, residual
    (2, 2, 45, 80, 64, 64, False, False),     # 2 channels per group
    (1, 2, 120, 216, 128, 128, True, False),  # 16 x 8 tiles, 4 channels per group
    (1, 1, 20, 30, 128, 512, False, False),   # 16 channels per group
    (2, 5, 12, 20, 128, 256, True, True),     # causal 3-D, statistics per sample over T frames
])
def test_conv_groupnorm_statistics(cuda, B, T, H, W, Cin, Cout, with_res, per_sample):
    """GroupNorm statistics from the conv epilogue (per pixel tile, in-frame pixels only; per
    frame, or per sample over all frames): the same partials from the CTA-pair and the 1-CTA
    kernel bit for bit, totals equal to the sums over the output, and the GroupNorm from them
    equal to the statistics-pass GroupNorm to fp32 rounding."""
    from paper_2506_13497_b200 import _lib, kernels
    from paper_2506_13497_b200._lib import ptr

    L = _lib.lib()
    G = 32
    N, P = (B, T * H * W) if per_sample else (B * T, H * W)
    kt = 3 if per_sample else 1
    g = torch.Generator().manual_seed(3)
    x = torch.randn(B, T, H, W, Cin, generator=g).to(cuda, torch.bfloat16)
    w = (torch.randn(Cout, kt, 3, 3, Cin, generator=g) / (Cin * 9 * kt) ** 0.5).to(cuda, torch.bfloat16)
    bias = (0.3 + 0.1 * torch.randn(Cout, generator=g)).to(cuda)
    res = torch.randn(B, T, H, W, Cout, generator=g).to(cuda, torch.bfloat16) if with_res else None
    nblk = L.ddit_conv_frame_tiles(H, W) * (T if per_sample else 1)
    parts, ys = [], []
    for pair in (1, 0):
        L.ddit_set_conv_2cta(pair)
        try:
            part = torch.full((N * G * nblk * 2,), float("nan"), device=cuda)
            ys.append(kernels.conv(x, w, bias=bias, residual=res, causal_time=per_sample, gn_part=part,
                                   gn_groups=G, gn_per_sample=per_sample))
            parts.append(part)
        finally:
            L.ddit_set_conv_2cta(1)
    torch.cuda.synchronize()
    assert torch.equal(ys[0], ys[1])
    assert torch.equal(parts[0], parts[1])  # every slot written (NaN-filled before)
    y = ys[0]
    tot = parts[0].view(N, G, nblk, 2).double().sum(2)
    yg = y.double().view(N, P, G, Cout // G)
    ref = torch.stack([yg.sum((1, 3)), (yg * yg).sum((1, 3))], -1)
    assert torch.allclose(tot, ref, rtol=1e-5, atol=1e-5 * P * (Cout // G))
    gamma = (1 + 0.1 * torch.randn(Cout, generator=g)).to(cuda)
    beta = (0.1 * torch.randn(Cout, generator=g)).to(cuda)
    out_a = torch.empty_like(y)
    out_b = torch.empty_like(y)
    coef = torch.empty(N * Cout * 2, device=cuda)
    stats = torch.empty(N * G * 2 + N * 512 * G + N * Cout, dtype=torch.float64, device=cuda)
    _lib.check(L.ddit_groupnorm_partials(ptr(y), ptr(out_a), ptr(parts[0]), nblk, ptr(coef), ptr(gamma),
                                         ptr(beta), N, P, Cout, G, 1e-6, 1, None))
    _lib.check(L.ddit_groupnorm(ptr(y), ptr(out_b), ptr(stats), ptr(gamma), ptr(beta), N, P, Cout,
                                G, 1e-6, 1, None))
    torch.cuda.synchronize()
    assert rel_l2(out_a, out_b) < 1e-3
    assert (out_a.float() - out_b.float()).abs().max().item() < 0.05
