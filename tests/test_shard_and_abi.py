"""CPU tests: shard / pad / exchange index math (product, C ABI and numpy oracle agree
bit-exactly), and the C-ABI library loads and exports every declared symbol."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import shard_ref
from paper_2506_13497_b200 import shapes

ROOT = Path(__file__).resolve().parents[1]

# label -> (T, S, N, T pads P=2/4/8, S pads P=2/4/8)
APPENDIX_B = {
    "144p-16f": (4, 144, 576, (4, 4, 8), (144, 144, 144)),
    "144p": (15, 144, 2160, (16, 16, 16), (144, 144, 144)),
    "240p": (15, 405, 6075, (16, 16, 16), (406, 408, 408)),
    "360p": (15, 920, 13800, (16, 16, 16), (920, 920, 920)),
    "480p-102f": (30, 1620, 48600, (30, 32, 32), (1620, 1620, 1624)),
    "720p-102f": (30, 3600, 108000, (30, 32, 32), (3600, 3600, 3600)),
}


@pytest.mark.parametrize("label", sorted(APPENDIX_B))
def test_registry_and_pads_match_appendix_b(label):
    T, S, N, tp, sp = APPENDIX_B[label]
    sh = shapes.shape_of(label)
    assert (sh.T, sh.S, sh.N) == (T, S, N)
    for P, a, b in zip((2, 4, 8), tp, sp):
        assert shard_ref.padded(T, P) == shapes.padded(T, P) == a
        assert shard_ref.padded(S, P) == shapes.padded(S, P) == b


@pytest.mark.parametrize("extent", [1, 4, 15, 30, 144, 405, 920, 1620, 3600])
@pytest.mark.parametrize("dop", [1, 2, 4, 8])
def test_shard_ranges_product_vs_oracle(extent, dop):
    ref = shard_ref.ranges(extent, dop)
    got = np.array([shapes.shard_range(extent, dop, r) for r in range(dop)])
    assert np.array_equal(ref, got)
    covered = np.concatenate([np.arange(lo, hi) for lo, hi in got])
    assert np.array_equal(covered, np.arange(extent))  # a partition, in order


@pytest.mark.parametrize("B,T,S,dop", [(2, 15, 405, 2), (2, 15, 405, 8), (2, 4, 144, 8), (1, 30, 17, 4), (2, 3, 5, 4)])
def test_exchange_is_a_bijection(B, T, S, dop):
    dst = shard_ref.exchange_sp_to_tp(B, T, S, dop)
    seen = set()
    for r in range(dop):
        for q, row in dst[r]:
            seen.add((int(q), int(row)))
    total = sum(len(shard_ref.temporal_tokens(B, T, S, dop, q)) for q in range(dop))
    assert len(seen) == total == B * T * S


def _lib():
    from paper_2506_13497_b200 import _lib

    return _lib


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib()
    h = L.lib()  # dlopen works without a GPU
    header = (ROOT / "include" / "ddit.h").read_text()
    declared = set(re.findall(r"DDIT_API\s+[\w\s\*]+?\b(ddit_\w+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(h, name), name
    assert set(L.exported_entry_points()) == declared
    assert h.ddit_version() >= 1


@pytest.mark.parametrize("label", ["240p", "144p-16f", "480p-102f"])
@pytest.mark.parametrize("dop", [1, 2, 4, 8])
def test_c_abi_shard_math_matches_oracle(label, dop):
    """The C++ geometry used by the step (pure host code) == the numpy oracle."""
    L = _lib()
    sh = shapes.shape_of(label)
    T, H, W = sh.latent
    for r in range(dop):
        d = L.CReqDesc(T, H, W, sh.height, sh.width, dop, r, 30, 7.0, 24.0)
        out = [ctypes.c_int() for _ in range(4)]
        L.check(L.lib().ddit_request_shard(None, ctypes.byref(d), *[ctypes.byref(o) for o in out]))
        got = [o.value for o in out]
        want = list(shard_ref.ranges(sh.T, dop)[r]) + list(shard_ref.ranges(sh.S, dop)[r])
        assert got == want


def test_c_abi_rejects_bad_dop():
    L = _lib()
    d = L.CReqDesc(15, 30, 54, 240, 426, 3, 0, 30, 7.0, 24.0)
    out = [ctypes.c_int() for _ in range(4)]
    rc = L.lib().ddit_request_shard(None, ctypes.byref(d), *[ctypes.byref(o) for o in out])
    assert rc == L.DDIT_E_LOOKUP


@pytest.mark.parametrize("T,frames", [(15, 51), (30, 102), (4, 16), (5, 17), (2, 5)])
@pytest.mark.parametrize("dop", [1, 2, 4])
def test_vae_shard_partitions_micro_batches(T, frames, dop):
    """VAE DoP split (vae.vae_shard): frame blocks tile [0, frames) in rank order; each rank's
    latent range is whole micro-batches covering exactly the micro-batches its frames fall in."""
    from paper_2506_13497_b200.vae import vae_shard
    from paper_2506_13497_b200.vae_weights import OPENSORA_VAE as cfg

    mz, mf = cfg.micro_z, cfg.micro_frame_size
    f_next = 0
    for r in range(dop):
        t_lo, t_hi, f_lo, f_hi = vae_shard(cfg, T, frames, dop, r)
        assert f_lo == f_next
        if f_hi > f_lo:
            assert t_lo == f_lo // mf * mz and t_hi == min(-(-f_hi // mf) * mz, T)
        f_next = f_hi
    assert f_next == frames
