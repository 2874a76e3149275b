"""Resolution registry and the sequence-parallel shard/pad index math.

The reference carries only a resolution *label* per request (reference
pkg/src/ditsim/workload.py:69-74; frames are metadata), so the label ->
tensor-shape table is ours ([EXT] OpenSora-1.2 conventions):

* latent H, W = ceil(pixels / 8); latent T follows the 17-frame micro-batch rule of the
  OpenSora VAE (17 -> 5): 51 -> 15, 102 -> 30, 16 -> 4;
* tokens per frame S = ceil(Hl/2) * ceil(Wl/2) (patch 1x2x2), N = T * S.

Sharding (DSP-style dimension switching): spatial blocks run on a T-shard
(contiguous frame blocks of ceil(T/P) per rank, padded at the end), temporal blocks on an
S-shard (contiguous token blocks of ceil(S/P) per rank). Rank r owns
``[r*ceil(X/P), (r+1)*ceil(X/P)) ∩ [0, X)``. Layout of a shard in HBM is always
``[B][t][s][C]`` row-major over the local extents.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

MICRO_FRAMES = 17
TEMPORAL_DOWN = 4
SPATIAL_DOWN = 8
PATCH = (1, 2, 2)


def latent_frames(frames: int) -> int:
    """OpenSora VAE latent frame count ([EXT] VideoAutoencoderPipeline.get_latent_size)."""

    def tvae(t: int) -> int:
        pad = 0 if t % TEMPORAL_DOWN == 0 else TEMPORAL_DOWN - t % TEMPORAL_DOWN
        return (t + pad) // TEMPORAL_DOWN

    n = tvae(MICRO_FRAMES) * (frames // MICRO_FRAMES)
    rem = frames % MICRO_FRAMES
    if rem:
        n += tvae(rem)
    return n


@dataclass(frozen=True)
class VideoShape:
    label: str
    height: int  # pixels
    width: int
    frames: int

    @property
    def latent(self) -> tuple[int, int, int]:
        return (
            latent_frames(self.frames),
            math.ceil(self.height / SPATIAL_DOWN),
            math.ceil(self.width / SPATIAL_DOWN),
        )

    @property
    def T(self) -> int:
        return self.latent[0]

    @property
    def grid(self) -> tuple[int, int]:
        """Token grid (h, w) after the 1x2x2 patchify (pads odd latent sizes)."""
        _, hl, wl = self.latent
        return math.ceil(hl / PATCH[1]), math.ceil(wl / PATCH[2])

    @property
    def S(self) -> int:
        h, w = self.grid
        return h * w

    @property
    def N(self) -> int:
        return self.T * self.S


# label -> shape. Plain labels mean 51 frames (workload.py:23 DEFAULT_FRAMES).
REGISTRY: dict[str, VideoShape] = {
    "144p": VideoShape("144p", 144, 256, 51),
    "240p": VideoShape("240p", 240, 426, 51),
    "360p": VideoShape("360p", 360, 640, 51),
    "480p": VideoShape("480p", 480, 854, 51),
    "720p": VideoShape("720p", 720, 1280, 51),
    "144p-16f": VideoShape("144p-16f", 144, 256, 16),
    "480p-102f": VideoShape("480p-102f", 480, 854, 102),
    "720p-102f": VideoShape("720p-102f", 720, 1280, 102),
}


def shape_of(label: str) -> VideoShape:
    try:
        return REGISTRY[label]
    except KeyError:
        raise LookupError(f"resolution {label!r} has no shape in the registry") from None


# ---------------------------------------------------------------- shard / pad math
def shard_size(extent: int, dop: int) -> int:
    return -(-extent // dop)


def padded(extent: int, dop: int) -> int:
    return shard_size(extent, dop) * dop


def shard_range(extent: int, dop: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of ``extent`` owned by ``rank`` of ``dop``; empty ranges have lo == hi."""
    if not 0 <= rank < dop:
        raise ValueError(f"rank {rank} outside dop {dop}")
    c = shard_size(extent, dop)
    lo = min(rank * c, extent)
    hi = min((rank + 1) * c, extent)
    return lo, hi


def t_shard(shape: VideoShape, dop: int, rank: int) -> tuple[int, int]:
    return shard_range(shape.T, dop, rank)


def s_shard(shape: VideoShape, dop: int, rank: int) -> tuple[int, int]:
    return shard_range(shape.S, dop, rank)
