"""Thin Python wrappers over the kernel-level C-ABI entry points (tests / profiling).

Every wrapper takes torch CUDA tensors (PyTorch is plumbing: memory and streams) and
passes raw pointers to libddit.so. Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import Attn, Epi, check, lib, ptr, stream_ptr


def _c(x) -> int | None:
    return ptr(x) if isinstance(x, torch.Tensor) else x


def gemm(
    a: torch.Tensor,
    w: torch.Tensor,
    *,
    epi: int = _lib.EPI_BF16,
    bias: torch.Tensor | None = None,
    out: torch.Tensor | None = None,
    resid: torch.Tensor | None = None,
    gate: torch.Tensor | None = None,
    rows_per_b: int = 0,
    out2: torch.Tensor | None = None,
    qnorm_w: torch.Tensor | None = None,
    knorm_w: torch.Tensor | None = None,
    hidden: int = 0,
    rope_tab: torch.Tensor | None = None,
    rope_T: int = 1,
    rope_S: int = 1,
    eps: float = 1e-6,
    bn: int = 128,
    stream=None,
) -> torch.Tensor | None:
    """``epi(a @ w.T + bias)`` on tcgen05. a: [M,K] bf16, w: [N,K] bf16."""
    assert a.dtype == torch.bfloat16 and w.dtype == torch.bfloat16
    M, K = a.shape
    N = w.shape[0]
    assert w.shape[1] == K
    if epi in (_lib.EPI_BF16, _lib.EPI_GELU_BF16, _lib.EPI_QKV) and out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
    if epi == _lib.EPI_F32 and out is None:
        out = torch.empty(M, N, dtype=torch.float32, device=a.device)
    e = Epi()
    e.bias = _c(bias)
    e.out = _c(out)
    e.ldo = out.stride(0) if out is not None else 0
    e.resid = _c(resid)
    e.ldr = resid.stride(0) if resid is not None else 0
    e.gate = _c(gate)
    e.gate_stride = gate.stride(0) if gate is not None else 0
    e.rows_per_b = rows_per_b
    e.out2 = _c(out2)
    e.ldo2 = out2.stride(0) if out2 is not None else 0
    e.qnorm_w = _c(qnorm_w)
    e.knorm_w = _c(knorm_w)
    e.hidden = hidden
    e.rope = 1 if rope_tab is not None else 0
    e.rope_T = rope_T
    e.rope_S = rope_S
    e.rope_tab = _c(rope_tab)
    e.eps = eps
    check(
        lib().ddit_gemm(
            ptr(a), a.stride(0), ptr(w), w.stride(0), M, N, K, epi, ctypes.byref(e), bn,
            stream_ptr(stream),
        )
    )
    return out if epi != _lib.EPI_RESID else resid


def attention(q, k, v, o, *, heads: int, num_seqs: int, Lq: int, Lk: int,
              q_map=(1, 0, 0, 1), kv_map=(1, 0, 0, 1), scale: float | None = None, stream=None,
              temporal: bool = False, tc: bool = True):
    """Attention over token-major bf16 matrices; maps = (inner, outer, inner_stride, tok): the
    tcgen05 FMHA (spatial / cross) or, with ``temporal``, the tcgen05 temporal kernel (q/k/v the
    three sections of one QKV matrix, T <= 64). ``tc`` is kept for callers; it must be True."""
    if not tc:
        raise ValueError("the mma.sync attention kernel was removed; only the tcgen05 kernels exist")
    a = Attn()
    a.q, a.ldq = ptr(q), q.stride(0)
    a.k, a.ldk = ptr(k), k.stride(0)
    a.v, a.ldv = ptr(v), v.stride(0)
    a.o, a.ldo = ptr(o), o.stride(0)
    a.heads, a.head_dim, a.num_seqs, a.Lq, a.Lk = heads, 72, num_seqs, Lq, Lk
    a.q_inner, a.q_outer, a.q_inner_stride, a.q_tok = q_map
    a.kv_inner, a.kv_outer, a.kv_inner_stride, a.kv_tok = kv_map
    a.scale = scale if scale is not None else 72 ** -0.5
    fn = lib().ddit_attention_temporal if temporal else lib().ddit_attention_tc
    check(fn(ctypes.byref(a), stream_ptr(stream)))
    return o


def conv(x: torch.Tensor, w: torch.Tensor, *, bias: torch.Tensor | None = None,
         residual: torch.Tensor | None = None, causal_time: bool = True, out=None, stream=None,
         gn_part: torch.Tensor | None = None, gn_groups: int = 0, gn_per_sample: bool = False):
    """Implicit-GEMM conv on tcgen05. x: [B,T,H,W,Cin] bf16 (channels-last);
    w: [Cout,kt,kh,kw,Cin] bf16; returns [B,T,H,W,Cout] bf16. ``gn_part`` (fp32, >= B*T*gn_groups*
    nblk*2 floats, nblk = ddit_conv_frame_tiles(H, W)): per-frame (``gn_per_sample``: per-sample,
    [B][G][T*nblk]) GroupNorm statistics partials of the output, written by the epilogue."""
    from ._lib import ConvArgs

    B, T, H, W, Cin = x.shape
    Cout, kt, kh, kw, Cin2 = w.shape
    assert Cin == Cin2 and x.is_contiguous() and w.is_contiguous()
    if out is None:
        out = torch.empty(B, T, H, W, Cout, dtype=torch.bfloat16, device=x.device)
    a = ConvArgs(ptr(x), ptr(out), ptr(w), _c(bias), _c(residual), B, T, H, W, Cin, Cout, kt, kh,
                 kw, 1 if causal_time else 0)
    if gn_part is not None:
        assert gn_part.dtype == torch.float32 and gn_part.is_contiguous()
        a.gn_part = ptr(gn_part)
        a.gn_groups = gn_groups
        a.gn_per_sample = 1 if gn_per_sample else 0
    check(lib().ddit_conv(ctypes.byref(a), stream_ptr(stream)))
    return out
