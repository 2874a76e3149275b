"""The VAE's memory-bound / small-channel kernels one at a time against torch fp32 references:
GroupNorm (+SiLU) over channels-last [N][P][C] (per-frame and whole-clip statistics, grouping
with fewer than 8 channels per group, a partition that does not depend on N), the
small-channel direct conv ([kt][kh][kw][Cin][Cout] weights, strided fp32 input) and the
frames-out crop."""
import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return (torch.linalg.vector_norm(a.float() - b.float()) / torch.linalg.vector_norm(b.float())).item()


def _gn(x, gamma, beta, G, eps, silu):
    from paper_2506_13497_b200._lib import check, lib, ptr, stream_ptr

    N, P, C = x.shape
    stats = torch.empty(N * G * 2 + N * 512 * G + N * C, dtype=torch.float64, device=x.device)
    y = torch.empty_like(x)
    check(lib().ddit_groupnorm(ptr(x), ptr(y), ptr(stats), ptr(gamma), ptr(beta), N, P, C, G, eps,
                               1 if silu else 0, stream_ptr()))
    return y


@pytest.mark.parametrize("N,P,C,G,silu", [(1, 8100, 512, 32, True), (5, 1620, 128, 32, True),
                                          (3, 4000, 256, 32, False), (2, 777, 64, 32, True)])
def test_groupnorm_matches_torch(cuda, N, P, C, G, silu):
    g = torch.Generator(device=cuda).manual_seed(N * 1000 + C)
    x = (torch.randn(N, P, C, device=cuda, generator=g) * 3 + 1.5).bfloat16()
    gamma = torch.randn(C, device=cuda, generator=g)
    beta = torch.randn(C, device=cuda, generator=g)
    y = _gn(x, gamma, beta, G, 1e-6, silu)
    ref = torch.nn.functional.group_norm(x.float().permute(0, 2, 1), G, gamma, beta, 1e-6).permute(0, 2, 1)
    if silu:
        ref = torch.nn.functional.silu(ref)
    torch.cuda.synchronize()
    assert rel_l2(y, ref) < 1e-2


def test_groupnorm_frame_stats_do_not_depend_on_batch(cuda):
    """VAE DoP decodes frame ranges: frame f's output must not change with the other frames in
    the call (the statistics partition depends on P and C only)."""
    g = torch.Generator(device=cuda).manual_seed(7)
    x = torch.randn(6, 2048, 128, device=cuda, generator=g).bfloat16()
    gamma = torch.randn(128, device=cuda, generator=g)
    beta = torch.randn(128, device=cuda, generator=g)
    whole = _gn(x, gamma, beta, 32, 1e-6, True)
    part = _gn(x[2:5].contiguous(), gamma, beta, 32, 1e-6, True)
    torch.cuda.synchronize()
    assert torch.equal(whole[2:5], part)


def test_conv_small_matches_torch(cuda):
    """Cin = 4 -> Cout = 256, 3x3x3 causal-in-time conv from a strided fp32 channels-first input
    (the temporal VAE's first conv) and a 4 -> 4 1x1 conv; weights in [kt][kh][kw][Cin][Cout]."""
    from paper_2506_13497_b200._lib import check, lib, ptr, stream_ptr
    from paper_2506_13497_b200.vae import _small

    g = torch.Generator(device=cuda).manual_seed(3)
    B, Cin, T, H, W, Cout = 1, 4, 5, 9, 13, 256
    x = torch.randn(B, Cin, T, H, W, device=cuda, generator=g)  # channels-first fp32
    w = torch.randn(Cout, 3, 3, 3, Cin, device=cuda, generator=g) * 0.2  # [Cout][kt][kh][kw][Cin]
    b = torch.randn(Cout, device=cuda, generator=g)
    y = torch.empty(B, T, H, W, Cout, device=cuda, dtype=torch.bfloat16)
    st = (ctypes.c_longlong * 5)(*x.stride())  # b, c, t, h, w
    check(lib().ddit_conv_small(ptr(x), 1, st, ptr(_small(w)), ptr(b), ptr(y), B, T, H, W, Cin, Cout, 3, 3, 3,
                                1, 0, 0, 0, stream_ptr()))
    # causal in time: pad 2 frames before, none after; 1 pixel each side spatially
    xp = torch.nn.functional.pad(x, (1, 1, 1, 1, 2, 0))
    ref = torch.nn.functional.conv3d(xp, w.permute(0, 4, 1, 2, 3), b).permute(0, 2, 3, 4, 1)
    torch.cuda.synchronize()
    assert rel_l2(y, ref) < 1e-2


def test_frames_out_crops_channels_first(cuda):
    from paper_2506_13497_b200._lib import check, lib, ptr, stream_ptr

    g = torch.Generator(device=cuda).manual_seed(5)
    N, H, W, ld = 4, 24, 40, 64
    y = torch.randn(N, H, W, ld, device=cuda, generator=g).bfloat16()
    out = torch.empty(1, 3, N, 21, 35, device=cuda)
    check(lib().ddit_frames_out(ptr(y), ptr(out), N, H, W, ld, 3, 21, 35, stream_ptr()))
    ref = y[:, :21, :35, :3].float().permute(3, 0, 1, 2).unsqueeze(0)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
