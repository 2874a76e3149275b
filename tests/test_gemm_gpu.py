"""tcgen05 GEMM + fused epilogues vs a plain torch fp32 reference of the same op."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 0], ids=["2cta", "1cta"], autouse=True)
def gemm_mode(request, cuda):
    from paper_2506_13497_b200 import _lib

    _lib.lib().ddit_set_gemm_2cta(request.param)
    yield request.param
    _lib.lib().ddit_set_gemm_2cta(1)


def rel_l2(a, b):
    a = a.float()
    b = b.float()
    return (torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b).clamp_min(1e-30)).item()


def _inputs(M, N, K, dev, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.randn(M, K, generator=g).to(dev, torch.bfloat16)
    w = (torch.randn(N, K, generator=g) / math.sqrt(K)).to(dev, torch.bfloat16)
    bias = (0.1 * torch.randn(N, generator=g)).to(dev)
    return a, w, bias


@pytest.mark.parametrize("bn", [96, 128, 192, 256])
@pytest.mark.parametrize("M,N,K", [(128, 1152, 64), (300, 2304, 1152), (1000, 4608, 1152),
                                   (777, 1152, 4608), (200, 288, 288), (5, 576, 104)])
def test_gemm_bias_bf16(cuda, bn, M, N, K):
    from paper_2506_13497_b200 import kernels, _lib

    if N % bn:
        pytest.skip("N not a multiple of BN")
    a, w, bias = _inputs(M, N, K, cuda)
    out = kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, bn=bn)
    ref = a.float() @ w.float().T + bias
    torch.cuda.synchronize()
    assert rel_l2(out, ref) < 5e-3


def test_gemm_f32_and_gelu(cuda):
    from paper_2506_13497_b200 import kernels, _lib

    a, w, bias = _inputs(513, 4608, 1152, cuda, seed=1)
    ref = a.float() @ w.float().T + bias
    out = kernels.gemm(a, w, epi=_lib.EPI_F32, bias=bias, bn=256)
    assert rel_l2(out, ref) < 1e-5
    out = kernels.gemm(a, w, epi=_lib.EPI_GELU_BF16, bias=bias, bn=256)
    assert rel_l2(out, torch.nn.functional.gelu(ref, approximate="tanh")) < 5e-3


@pytest.mark.parametrize("bn,N,K", [(128, 1152, 1152), (192, 1152, 4608), (96, 288, 1152), (256, 2304, 288)])
def test_gemm_resid_gate(cuda, bn, N, K):
    from paper_2506_13497_b200 import kernels, _lib

    M = 2 * 607
    a, w, bias = _inputs(M, N, K, cuda, seed=2)
    x = torch.randn(M, N, device=cuda)
    gate = torch.randn(2, N, device=cuda)
    x0 = x.clone()
    out2 = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2, out2=out2, bn=bn)
    b = torch.arange(M, device=cuda) // (M // 2)
    ref = x0 + gate[b] * (a.float() @ w.float().T + bias)
    assert rel_l2(x, ref) < 1e-5
    assert rel_l2(out2, ref) < 5e-3
    # no gate, no bf16 copy
    x1 = x0.clone()
    kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x1, bn=bn)
    assert rel_l2(x1, x0 + a.float() @ w.float().T + bias) < 1e-5


@pytest.mark.parametrize("bn", [96, 128, 192, 256])
def test_gemm_resid_reduce_matches_load_update_store(cuda, bn):
    """The reduce-add residual epilogue (TMA reduce into x, nothing loaded) and the TMA load /
    update / store epilogue give bit-identical x (both round acc + b, g * (.), x + (.) in turn),
    which is what keeps DoP-P (whose fc2 exchanges rows) bit-exact with DoP 1."""
    from paper_2506_13497_b200 import kernels, _lib

    L = _lib.lib()
    M, N, K = 2 * 1013, 2304, 1152
    a, w, bias = _inputs(M, N, K, cuda, seed=5)
    x0 = torch.randn(M, N, device=cuda)
    gate = torch.randn(2, N, device=cuda)
    outs = []
    try:
        for red in (0, 1):
            L.ddit_set_resid_reduce(red)
            x = x0.clone()
            kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=M // 2, bn=bn)
            outs.append(x)
    finally:
        L.ddit_set_resid_reduce(1)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    b = torch.arange(M, device=cuda) // (M // 2)
    assert rel_l2(outs[1], x0 + gate[b] * (a.float() @ w.float().T + bias)) < 1e-5


@pytest.mark.parametrize("rope", [False, True])
def test_gemm_qkv_epilogue(cuda, rope):
    from paper_2506_13497_b200 import kernels, _lib

    C, H, D = 1152, 16, 72
    T, S = 5, 37
    M = 2 * T * S
    a, w, bias = _inputs(M, 3 * C, C, cuda, seed=3)
    qw = 1 + 0.1 * torch.randn(D, device=cuda)
    kw = 1 + 0.1 * torch.randn(D, device=cuda)
    freqs = 1.0 / (10000 ** (torch.arange(0, D, 2, dtype=torch.float64)[: D // 2] / D))
    ang = torch.arange(T, dtype=torch.float64)[:, None] * freqs[None]
    tab = torch.stack([ang.cos(), ang.sin()], -1).float().to(cuda).contiguous()
    out = kernels.gemm(a, w, epi=_lib.EPI_QKV, bias=bias, qnorm_w=qw, knorm_w=kw, hidden=C,
                       rope_tab=tab if rope else None, rope_T=T, rope_S=S, bn=144)
    ref = (a.float() @ w.float().T + bias).view(M, 3, H, D)
    q, k, v = ref.unbind(1)

    def rms(x, wt):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-6) * wt

    q, k = rms(q, qw), rms(k, kw)
    if rope:
        pos = (torch.arange(M, device=cuda) // S) % T
        cs = tab[pos]  # [M, 36, 2]
        def rot(x):
            x2 = x.view(M, H, D // 2, 2)
            c = cs[:, None, :, 0]
            s = cs[:, None, :, 1]
            a0, a1 = x2[..., 0], x2[..., 1]
            return torch.stack([a0 * c - a1 * s, a1 * c + a0 * s], -1).view(M, H, D)
        q, k = rot(q), rot(k)
    ref = torch.stack([q, k, v], 1).view(M, 3 * C)
    assert rel_l2(out, ref) < 5e-3
    # per-head padded weights (80-row slots, 256 x 240 / 128 x 240 tiles of three whole heads):
    # the same output bit for bit
    wp = torch.zeros(3 * H * 80, C, device=cuda, dtype=torch.bfloat16)
    bp = torch.zeros(3 * H * 80, device=cuda)
    for h in range(3 * H):
        wp[h * 80:h * 80 + 72] = w[h * 72:(h + 1) * 72]
        bp[h * 80:h * 80 + 72] = bias[h * 72:(h + 1) * 72]
    out_p = torch.empty_like(out)
    kernels.gemm(a, wp, epi=_lib.EPI_QKV, bias=bp, out=out_p, qnorm_w=qw, knorm_w=kw, hidden=C,
                 rope_tab=tab if rope else None, rope_T=T, rope_S=S, bn=240)
    torch.cuda.synchronize()
    assert torch.equal(out_p, out)


@pytest.mark.parametrize("nb,N", [(4, 576), (4, 1152), (3, 1152)])
def test_gemm_resid_gate_many_batches(cuda, nb, N):
    """Gate rows for more than two samples: staged in shared memory when (1 + nb) * N floats fit
    (nb = 4, N = 576), read from global memory otherwise (N = 1152); ragged last sample (nb = 3)."""
    from paper_2506_13497_b200 import kernels, _lib

    M, K = 1300, 1152
    rows_per_b = -(-M // nb)
    a, w, bias = _inputs(M, N, K, cuda, seed=9)
    x = torch.randn(M, N, device=cuda)
    gate = torch.randn(nb, N, device=cuda)
    x0 = x.clone()
    kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate, rows_per_b=rows_per_b, bn=192)
    b = torch.arange(M, device=cuda) // rows_per_b
    assert rel_l2(x, x0 + gate[b] * (a.float() @ w.float().T + bias)) < 1e-5


@pytest.mark.parametrize("M", [12150, 1000, 300])
@pytest.mark.parametrize("red", [True, False], ids=["reduce-add", "bf16"])
def test_gemm_wide_tiles_bit_identical(cuda, gemm_mode, M, red):
    """The 256 x 384 tiles (two BN = 192 accumulator halves, fc2's K = 4608) reproduce the
    256 x 192 tiles bit for bit, with the reduce-add residual and the plain bf16 epilogue; the
    1-CTA parametrisation runs the regular kernel on both sides."""
    from paper_2506_13497_b200 import _lib, kernels

    N, K = 1152, 4608
    a, w, bias = _inputs(M, N, K, cuda, seed=7)
    gate = torch.randn(2, N, device=cuda)
    x0 = torch.randn(M, N, device=cuda)
    outs = []
    for wide in (1, 0):
        _lib.lib().ddit_set_gemm_wide(wide)
        try:
            if red:
                x = x0.clone()
                kernels.gemm(a, w, epi=_lib.EPI_RESID, bias=bias, resid=x, gate=gate,
                             rows_per_b=(M + 1) // 2, bn=192)
                outs.append(x)
            else:
                out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
                kernels.gemm(a, w, epi=_lib.EPI_BF16, bias=bias, out=out, bn=192)
                outs.append(out)
        finally:
            _lib.lib().ddit_set_gemm_wide(1)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    ref = a.float() @ w.float().T + bias
    if red:
        b = torch.arange(M, device=cuda) // ((M + 1) // 2)
        ref = x0 + gate[b] * ref
    assert rel_l2(outs[0], ref) < 1e-2
