"""bench.py as the driver launches it, on the one-GPU box: `--gpus 2` without torchrun spawns its
own two ranks (sharing the device, gloo plumbing) and prints one JSON line with the exchange
object; the line must parse and carry the contract keys."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_self_spawns_two_ranks(cuda):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline", "--label", "144p"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["exchange"]["mode"] == "fused" and d["exchange"]["exchanges_per_step"] == 56
    assert "not a scaling number" in d["config"]["parallelism"]
