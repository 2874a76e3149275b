"""Link an experimental variant of libddit.so: one source recompiled with extra nvcc flags, the
other objects reused from the regular build (run build() first).
Usage: python scripts/build_variant.py NAME SOURCE.cu|/abs/path/SOURCE.cu -DFOO=1 ...  ->  paper_2506_13497_b200/libddit_NAME.so
(load it with DDIT_LIB=paper_2506_13497_b200/libddit_NAME.so)."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_13497_b200 import build as b

name, src, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build(verbose=False)
out_dir = b.BUILD.parent / f"var_{name}"
out_dir.mkdir(parents=True, exist_ok=True)
obj = out_dir / (Path(src).stem + ".o")
src_path = Path(src) if Path(src).is_absolute() else b.CSRC / src  # absolute: e.g. an older revision
subprocess.run([b.NVCC, *b.ARCH, *b.FLAGS, *extra, "-c", str(src_path), "-o", str(obj)], check=True)
if obj.stem not in {s.stem for s in b._sources()}:
    sys.exit(f"{src}: the variant source must keep the name of the csrc file it replaces")
objs = [obj if o.stem == obj.stem else o for o in (b.BUILD / (s.stem + ".o") for s in b._sources())]
lib = b.PKG / f"libddit_{name}.so"
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-cudart", "shared",
                "-Xlinker", "-rpath,/usr/local/cuda/lib64"], check=True)
print(lib)
