"""ctypes binding of ``libddit.so`` (the C ABI declared in ``include/ddit.h``).

There is no fallback: if the shared library is missing or fails to load, every
entry point raises.  ``torch`` is imported first so that its already-loaded CUDA
runtime (``libcudart.so.12``) is the one the library binds to.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch  # noqa: F401  (loads libcudart before libddit)

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("DDIT_LIB", _PKG / "libddit.so"))

DDIT_OK = 0
DDIT_E_INVALID = -2
DDIT_E_TMA = -3
DDIT_E_CUDA = -4
DDIT_E_LOOKUP = -5
DDIT_E_ALLOC = -6
DDIT_E_CONFIG = -7

EPI_BF16 = 0
EPI_GELU_BF16 = 1
EPI_RESID = 2
EPI_QKV = 3
EPI_F32 = 4


class DditError(RuntimeError):
    """A libddit entry point returned a non-zero code."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libddit error {code}: {message}")
        self.code = code


vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float


class Epi(ctypes.Structure):
    _fields_ = [
        ("bias", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("ldo", ctypes.c_int),
        ("resid", ctypes.c_void_p),
        ("ldr", ctypes.c_int),
        ("gate", ctypes.c_void_p),
        ("gate_stride", ctypes.c_int),
        ("rows_per_b", ctypes.c_int),
        ("out2", ctypes.c_void_p),
        ("ldo2", ctypes.c_int),
        ("qnorm_w", ctypes.c_void_p),
        ("knorm_w", ctypes.c_void_p),
        ("hidden", ctypes.c_int),
        ("rope", ctypes.c_int),
        ("rope_T", ctypes.c_int),
        ("rope_S", ctypes.c_int),
        ("rope_tab", ctypes.c_void_p),
        ("eps", ctypes.c_float),
    ]




class CConfig(ctypes.Structure):
    _fields_ = [
        ("depth", ci), ("hidden", ci), ("heads", ci), ("head_dim", ci), ("mlp_hidden", ci),
        ("in_channels", ci), ("out_channels", ci), ("caption_channels", ci),
        ("text_tokens", ci), ("freq_dim", ci), ("input_sq_size", ci), ("eps", cf),
    ]


class CBlock(ctypes.Structure):
    _fields_ = [
        ("scale_shift_table", vp), ("qkv_w", vp), ("qkv_b", vp), ("q_norm", vp), ("k_norm", vp),
        ("proj_w", vp), ("proj_b", vp), ("cq_w", vp), ("cq_b", vp), ("ckv_w", vp),
        ("ckv_b", vp), ("cproj_w", vp), ("cproj_b", vp), ("fc1_w", vp), ("fc1_b", vp),
        ("fc2_w", vp), ("fc2_b", vp),
    ]


class CWeights(ctypes.Structure):
    _fields_ = [
        ("x_emb_w", vp), ("x_emb_b", vp), ("t0_w", vp), ("t0_b", vp), ("t2_w", vp), ("t2_b", vp),
        ("f0_w", vp), ("f0_b", vp), ("f2_w", vp), ("f2_b", vp), ("tb_w", vp), ("tb_b", vp),
        ("y1_w", vp), ("y1_b", vp), ("y2_w", vp), ("y2_b", vp), ("y_null", vp),
        ("final_sst", vp), ("final_w", vp), ("final_b", vp), ("blocks", ctypes.POINTER(CBlock)),
    ]


class CReqDesc(ctypes.Structure):
    _fields_ = [
        ("latent_t", ci), ("latent_h", ci), ("latent_w", ci), ("height", ci), ("width", ci),
        ("dop", ci), ("rank", ci), ("num_steps", ci), ("guidance", cf), ("fps", cf),
    ]


class ConvArgs(ctypes.Structure):
    _fields_ = [
        ("x", vp), ("y", vp), ("w", vp), ("bias", vp), ("residual", vp),
        ("B", ci), ("T", ci), ("H", ci), ("W", ci), ("Cin", ci), ("Cout", ci),
        ("kt", ci), ("kh", ci), ("kw", ci), ("causal_time", ci),
        ("gn_part", vp), ("gn_groups", ci), ("gn_per_sample", ci),
    ]


class Attn(ctypes.Structure):
    _fields_ = [
        ("q", ctypes.c_void_p), ("ldq", ctypes.c_int),
        ("k", ctypes.c_void_p), ("ldk", ctypes.c_int),
        ("v", ctypes.c_void_p), ("ldv", ctypes.c_int),
        ("o", ctypes.c_void_p), ("ldo", ctypes.c_int),
        ("heads", ctypes.c_int), ("head_dim", ctypes.c_int), ("num_seqs", ctypes.c_int),
        ("Lq", ctypes.c_int), ("Lk", ctypes.c_int),
        ("q_inner", ctypes.c_int), ("q_outer", ctypes.c_int), ("q_inner_stride", ctypes.c_int),
        ("q_tok", ctypes.c_int),
        ("kv_inner", ctypes.c_int), ("kv_outer", ctypes.c_int), ("kv_inner_stride", ctypes.c_int),
        ("kv_tok", ctypes.c_int),
        ("scale", ctypes.c_float),
    ]


_SIGNATURES = {
    "ddit_set_gemm_2cta": [ci],
    "ddit_set_gemm_wide": [ci],
    "ddit_set_qkv_pad": [ci],
    "ddit_set_conv_2cta": [ci],
    "ddit_set_conv_tile_search": [ci],
    "ddit_set_pdl": [ci],
    "ddit_set_fused_exchange": [ci],
    "ddit_set_resid_reduce": [ci],
    "ddit_set_exchange_timeout_ms": [ci],
    "ddit_enable_peer_access": [ci, ci],
    "ddit_attention_temporal": [ctypes.POINTER(Attn), vp],
    "ddit_attention_tc": [ctypes.POINTER(Attn), vp],
    "ddit_ln_modulate": [vp, vp, ci, ci, vp, vp, ci, ci, ctypes.c_float, vp],
    "ddit_set_ln_variant": [ci],
    "ddit_model_create": [ctypes.POINTER(CConfig), ctypes.POINTER(CWeights), ctypes.POINTER(vp)],
    "ddit_request_workspace_bytes": [vp, ctypes.POINTER(CReqDesc), ctypes.POINTER(ctypes.c_uint64)],
    "ddit_request_shard": [vp, ctypes.POINTER(CReqDesc)] + [ctypes.POINTER(ci)] * 4,
    "ddit_request_open": [vp, ctypes.POINTER(CReqDesc), vp, ctypes.c_uint64, vp, vp,
                          ctypes.POINTER(vp)],
    "ddit_request_set_text": [vp, vp, vp],
    "ddit_request_copy_text": [vp, vp, vp],
    "ddit_request_share_text": [vp, vp, vp],
    "ddit_reshard": [ctypes.POINTER(vp), ctypes.POINTER(vp), ci, ctypes.POINTER(vp),
                     ctypes.POINTER(ci), ctypes.POINTER(ci), ci, vp, ctypes.POINTER(vp)],
    "ddit_request_reshard_ms": [vp, ctypes.POINTER(cf)],
    "ddit_request_exchange_buffers": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)],
    "ddit_request_set_peers": [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)],
    "ddit_dit_step": [vp, vp, ci, vp],
    "ddit_step_begin": [vp, vp, ci, vp],
    "ddit_step_phase": [vp, ci, vp],
    "ddit_step_end": [vp, vp, ci, vp],
    "ddit_step_barrier": [vp, vp],
    "ddit_request_status": [vp, vp, ctypes.POINTER(ctypes.c_uint32)],
    "ddit_request_timestep": [vp, ci, ctypes.POINTER(cf), ctypes.POINTER(cf)],
    "ddit_request_profile": [vp, ci],
    "ddit_request_xch_counts": [vp, ci, ctypes.POINTER(ci), ctypes.POINTER(ci)],
    "ddit_request_xch_pack": [vp, ci, vp, vp],
    "ddit_request_xch_unpack": [vp, ci, vp, vp],
    "ddit_request_set_option": [vp, ci, ci],
    "ddit_request_profile_read": [vp, ctypes.POINTER(cf), ctypes.POINTER(ci)],
    "ddit_conv": [ctypes.POINTER(ConvArgs), vp],
    "ddit_groupnorm": [vp, vp, vp, vp, vp, ci, ci, ci, ci, cf, ci, vp],
    "ddit_conv_frame_tiles": [ci, ci],
    "ddit_groupnorm_partials": [vp, vp, vp, ci, vp, vp, vp, ci, ci, ci, ci, cf, ci, vp],
    "ddit_upsample2x": [vp, vp, ci, ci, ci, ci, vp],
    "ddit_depth_to_time": [vp, vp, ci, ci, ci, ci, vp],
    "ddit_frames_out": [vp, vp, ci, ci, ci, ci, ci, ci, ci, vp],
    "ddit_conv_small": [vp, ci, vp, vp, vp, vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, vp],
    "ddit_softmax_rows": [vp, vp, ci, ci, ci, cf, vp],
    "ddit_transpose_bf16": [vp, vp, ci, ci, ci, ci, vp],
    "ddit_add_f32_bf16": [vp, vp, vp, ctypes.c_uint64, vp],
    "ddit_latent_gather": [vp, ci, ci, ctypes.POINTER(vp), ctypes.POINTER(ci), ctypes.POINTER(ci),
                           ci, ci, ci, vp],
    "ddit_ipc_export": [vp, vp, ctypes.POINTER(ctypes.c_uint64)],
    "ddit_ipc_import": [vp, ctypes.c_uint64, ctypes.POINTER(vp)],
    "ddit_ipc_close": [vp, ctypes.c_uint64],
}
_VOID_FUNCS = {"ddit_model_destroy": [vp], "ddit_request_close": [vp]}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libddit.so once; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the DDiT hot path)"
            )
        handle = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_GLOBAL)
        _declare(handle)
        _lib = handle
    return _lib


def _declare(h: ctypes.CDLL) -> None:
    vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    h.ddit_last_error.restype = ctypes.c_char_p
    h.ddit_last_error.argtypes = []
    h.ddit_version.restype = ci
    h.ddit_num_sms.restype = ci
    h.ddit_gemm.restype = ci
    h.ddit_gemm.argtypes = [vp, ci, vp, ci, ci, ci, ci, ci, ctypes.POINTER(Epi), ci, vp]
    h.ddit_launch_count.restype = ctypes.c_ulonglong
    h.ddit_launch_count.argtypes = []
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = ci
        fn.argtypes = argtypes
    for name, argtypes in _VOID_FUNCS.items():
        fn = getattr(h, name)
        fn.restype = None
        fn.argtypes = argtypes


def exported_entry_points() -> list[str]:
    """Every C-ABI function this binding declares (the symbol-export test checks them)."""
    return ["ddit_last_error", "ddit_version", "ddit_num_sms", "ddit_gemm", "ddit_launch_count",
            *_SIGNATURES, *_VOID_FUNCS]


def check(rc: int) -> None:
    if rc != DDIT_OK:
        msg = lib().ddit_last_error().decode(errors="replace")
        raise DditError(rc, msg)


def stream_ptr(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
