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
    for name, argtypes in _EXTRA_SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = ci
        fn.argtypes = argtypes


# Filled in by the modules that bind further entry points (kept in one table so the
# symbol-export test can check every declared function).
_EXTRA_SIGNATURES: dict[str, list] = {}


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
