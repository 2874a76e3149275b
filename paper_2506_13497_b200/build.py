"""In-tree build of the sm_100a C-ABI library ``libddit.so``.

Every ``csrc/*.cu`` is compiled with nvcc for ``sm_100a`` (``-gencode
arch=compute_100a,code=sm_100a -lineinfo``) and linked into one shared object that
lives next to this file, so it travels to the GPU box with the repo snapshot.
The library links the CUDA runtime by soname (``libcudart.so.12``); when torch is
imported first, its already-loaded runtime is reused.
"""

from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG.parent / "build" / "obj"
LIB = PKG / "libddit.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    f"-I{CSRC}",
    f"-I{INCLUDE}",
]


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _digest(paths: list[Path]) -> str:
    h = hashlib.sha256()
    for p in sorted(CSRC.glob("*")) + sorted(INCLUDE.glob("*.h")):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    # flags without the absolute include paths, so the stamp survives the move to the GPU box
    h.update(" ".join(ARCH + [f for f in FLAGS if not f.startswith("-I")]).encode())
    return h.hexdigest()[:16]


def _compile(src: Path) -> Path:
    obj = BUILD / (src.stem + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True) -> Path:
    """Compile csrc/*.cu for sm_100a and link ``libddit.so`` (skipped if up to date)."""
    srcs = _sources()
    stamp = PKG / ".libddit.stamp"
    digest = _digest(srcs)
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == digest:
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    cmd = [
        NVCC,
        *ARCH,
        "-shared",
        "-o",
        str(LIB),
        *map(str, objs),
        "-cudart",
        "shared",
        "-Xlinker",
        "-rpath,/usr/local/cuda/lib64",
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    stamp.write_text(digest)
    if verbose:
        print(f"[ddit] built {LIB} from {len(srcs)} sources", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
