"""On-disk format for the DiT group's output: the denoised latent of a request,
and optionally its decoded frames, as written when the DiT->VAE hand-off leaves the DiT group
through storage instead of NVLink (the paper hands the latent to the VAE workers, PAPER.md:476;
the reference persists only workloads, reference workload.py:129-176).

Layout (little endian), one file per request::

    offset  size  field
    0       8     magic b"DDITLAT1"
    8       4     header length H (bytes of the JSON header that follows)
    12      H     JSON header: {"request_id", "resolution", "steps", "dtype", "shape",
                  "frames_dtype", "frames_shape", "payload_bytes", "crc32", ...user meta}
    12+H    pad   zero bytes up to a 256-byte boundary (so the payload can be mmapped / DMA'd)
    P       N     latent payload: C-contiguous array of `shape` in `dtype` ("f32" | "bf16")
    P+N     M     optional frames payload ("u8" [F][H][W][3] or "bf16" [3][F][H][W])

``crc32`` covers both payloads. ``load_latent`` verifies magic, lengths and checksum and raises
``LatentFormatError`` on any mismatch.
"""

from __future__ import annotations

import json
import zlib
from pathlib import Path

import numpy as np
import torch

MAGIC = b"DDITLAT1"
ALIGN = 256
_DT = {"f32": (torch.float32, 4), "bf16": (torch.bfloat16, 2), "u8": (torch.uint8, 1)}


class LatentFormatError(ValueError):
    """The file is not a valid DDiT latent file (bad magic, truncated, checksum mismatch)."""


def _name(t: torch.Tensor) -> str:
    for k, (dt, _) in _DT.items():
        if t.dtype == dt:
            return k
    raise LatentFormatError(f"unsupported dtype {t.dtype}")


def _bytes(t: torch.Tensor) -> bytes:
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        t = t.view(torch.int16)
    return t.numpy().tobytes()


def save_latent(path: str | Path, latent: torch.Tensor, *, request_id: int, resolution: str,
                steps: int, frames: torch.Tensor | None = None, **meta) -> int:
    """Write one request's latent (and frames); returns the file size in bytes."""
    lat = _bytes(latent)
    frm = _bytes(frames) if frames is not None else b""
    hdr = {"request_id": int(request_id), "resolution": resolution, "steps": int(steps),
           "dtype": _name(latent), "shape": list(latent.shape),
           "frames_dtype": _name(frames) if frames is not None else None,
           "frames_shape": list(frames.shape) if frames is not None else None,
           "payload_bytes": len(lat), "frames_bytes": len(frm),
           "crc32": zlib.crc32(frm, zlib.crc32(lat)) & 0xFFFFFFFF, **meta}
    h = json.dumps(hdr, sort_keys=True).encode()
    head = MAGIC + len(h).to_bytes(4, "little") + h
    pad = (-len(head)) % ALIGN
    path = Path(path)
    tmp = path.with_suffix(path.suffix + ".tmp")
    with open(tmp, "wb") as f:
        f.write(head + b"\0" * pad)
        f.write(lat)
        f.write(frm)
    tmp.replace(path)  # atomic publish: readers never see a partial file
    return len(head) + pad + len(lat) + len(frm)


def _tensor(buf: bytes, dtype: str, shape) -> torch.Tensor:
    tdt, size = _DT[dtype]
    n = int(np.prod(shape)) if shape else 1
    if len(buf) != n * size:
        raise LatentFormatError("payload length does not match shape")
    if dtype == "bf16":
        return torch.from_numpy(np.frombuffer(buf, dtype=np.int16).copy()).view(torch.bfloat16).reshape(shape)
    npdt = {"f32": np.float32, "u8": np.uint8}[dtype]
    return torch.from_numpy(np.frombuffer(buf, dtype=npdt).copy()).reshape(shape)


def load_latent(path: str | Path) -> tuple[torch.Tensor, torch.Tensor | None, dict]:
    """Read a latent file: (latent, frames or None, header)."""
    data = Path(path).read_bytes()
    if len(data) < 12 or data[:8] != MAGIC:
        raise LatentFormatError("bad magic")
    hl = int.from_bytes(data[8:12], "little")
    if 12 + hl > len(data):
        raise LatentFormatError("truncated header")
    try:
        hdr = json.loads(data[12:12 + hl])
    except ValueError as e:
        raise LatentFormatError(f"bad header: {e}") from None
    p = 12 + hl
    p += (-p) % ALIGN
    n, m = hdr["payload_bytes"], hdr.get("frames_bytes", 0)
    if p + n + m != len(data):
        raise LatentFormatError("truncated payload")
    lat, frm = data[p:p + n], data[p + n:p + n + m]
    if zlib.crc32(frm, zlib.crc32(lat)) & 0xFFFFFFFF != hdr["crc32"]:
        raise LatentFormatError("checksum mismatch")
    z = _tensor(lat, hdr["dtype"], hdr["shape"])
    f = _tensor(frm, hdr["frames_dtype"], hdr["frames_shape"]) if hdr.get("frames_dtype") else None
    return z, f, hdr
