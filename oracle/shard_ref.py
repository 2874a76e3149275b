"""ORACLE (test infrastructure only) -- numpy restatement of the sequence-parallel
shard / pad / exchange index math of the DoP-P step.

No reference code exists for it (the reference simulates SP only through the dit_step(res,
dop) curve, reference pkg/src/ditsim/profiles.py:69-76); the rules restated here are the
build's contract from SURVEY.md §8(e) and Appendix B: contiguous T-blocks of ceil(T/P) frames
for spatial blocks, contiguous S-blocks of ceil(S/P) tokens for temporal blocks, padding at
the end; a shard is laid out [B][t][s] row-major over its local extents. The pad columns of
SURVEY Appendix B are the golden vectors these functions are pinned to.
"""

from __future__ import annotations

import numpy as np


def chunk(extent: int, dop: int) -> int:
    return -(-extent // dop)


def ranges(extent: int, dop: int) -> np.ndarray:
    """[dop, 2] array of [lo, hi) per rank."""
    c = chunk(extent, dop)
    lo = np.minimum(np.arange(dop) * c, extent)
    hi = np.minimum((np.arange(dop) + 1) * c, extent)
    return np.stack([lo, hi], 1)


def spatial_tokens(B: int, T: int, S: int, dop: int, rank: int) -> np.ndarray:
    """Global token ids (b*T*S + t*S + s) of rank's spatial-phase rows, in row order."""
    lo, hi = ranges(T, dop)[rank]
    b, t, s = np.meshgrid(np.arange(B), np.arange(lo, hi), np.arange(S), indexing="ij")
    return (b * T * S + t * S + s).reshape(-1)


def temporal_tokens(B: int, T: int, S: int, dop: int, rank: int) -> np.ndarray:
    """Global token ids of rank's temporal-phase rows ([B][T][Sl] order)."""
    lo, hi = ranges(S, dop)[rank]
    b, t, s = np.meshgrid(np.arange(B), np.arange(T), np.arange(lo, hi), indexing="ij")
    return (b * T * S + t * S + s).reshape(-1)


def exchange_sp_to_tp(B: int, T: int, S: int, dop: int):
    """For every (src rank, src row) the (dst rank, dst row) of the spatial->temporal push."""
    where = {}
    for q in range(dop):
        for row, tok in enumerate(temporal_tokens(B, T, S, dop, q)):
            where[int(tok)] = (q, row)
    out = []
    for r in range(dop):
        out.append(np.array([where[int(tok)] for tok in spatial_tokens(B, T, S, dop, r)],
                            dtype=np.int64).reshape(-1, 2))
    return out


def padded(extent: int, dop: int) -> int:
    return chunk(extent, dop) * dop
