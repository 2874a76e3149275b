"""DoP-2/4 across processes (CUDA IPC peer stores + flag barrier) == single-process DoP 1."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("fused", ["1", "0"], ids=["fused-xch", "xch-kernel"])
@pytest.mark.parametrize("dop", [2, 4])
def test_multiprocess_group_matches_dop1(cuda, dop, fused):
    """Real processes with CUDA-IPC peer buffers and the flag barrier; the exchange fused into
    the fc2 GEMM (DDIT_FUSED_XCH=1) or as the separate kernel."""
    port = 29600 + 2 * dop + int(fused)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={dop}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "scripts" / "group_check.py"), "144p"]
    env = dict(os.environ, OMP_NUM_THREADS="1", DDIT_FUSED_XCH=fused)
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    print(res.stdout[-3000:], res.stderr[-3000:])
    assert res.returncode == 0
    assert "PASS" in res.stdout


def test_multiprocess_group_ranks_without_frames(cuda):
    """DoP 8 over T = 4 latent frames (144p-16f): ranks 4..7 own no frames in the spatial phase,
    run no fc2 GEMM there and must still publish their exchange flags (stand-alone kernel) while
    the other ranks' fused GEMM epilogues signal -- real processes, flag barrier, CUDA graphs."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29650", str(ROOT / "scripts" / "group_check.py"),
           "144p-16f"]
    env = dict(os.environ, OMP_NUM_THREADS="1", DDIT_FUSED_XCH="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    print(res.stdout[-3000:], res.stderr[-3000:])
    assert res.returncode == 0
    assert "PASS" in res.stdout
