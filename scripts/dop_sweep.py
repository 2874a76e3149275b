"""Per-(resolution, DoP) STDiT3-XL/2 step latency on ONE B200 -> profiles/ + a dit-profile/1 document.

DoP 1 is measured directly (CUDA-graph replay of the real step, CUDA events, best of --reps).
DoP P > 1 runs the real P-rank DSP step as virtual ranks on the one GPU (every rank's kernels and
its exchange pushes, in lockstep on one stream; bit-exact with DoP 1) and reports
  * group_serial_ms  -- the whole group on one GPU (all P ranks' work, serialised);
  * rank_ms          -- per rank, device time of its own kernels by class (per-launch CUDA events);
  * rank_step_ms     -- per rank, device time of its share of every phase (CUDA events around each
                        rank's begin / phase / end calls: its kernels + its exchange pushes);
  * projected_ms     -- max over ranks of rank_step_ms + the rank's exchange bytes over NVLink at
                        the measured 770 GB/s peer-copy rate (B200_PROFILING.md), i.e. the DoP-P
                        step latency on P GPUs with no compute/transfer overlap (the local pushes
                        are counted as well: conservative). Flagged "virtual": true.
Usage: python scripts/dop_sweep.py [labels...] [--dops 1,2,4,8] [--reps 3] [--out file]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import shapes, weights
from paper_2506_13497_b200.executor import exchange_bytes
from paper_2506_13497_b200.stdit import STDiTModel, StepRequest, VirtualGroup

NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
_peaks = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK_TFLOPS = (json.loads(_peaks.read_text())["bf16_tflops_sustained"] if _peaks.exists() else 1400.0)


def step_flops(cfg, shape):
    """Algorithmic FLOPs of one CFG step (the bench.py formula)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_bench", Path(__file__).resolve().parents[1] / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.step_flops(cfg, shape)


def ev_time(fn, reps: int) -> float:
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("labels", nargs="*", default=["144p", "240p", "360p"])
    ap.add_argument("--dops", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/dop_sweep.json")
    a = ap.parse_args()
    dops = [int(x) for x in a.dops.split(",")]
    dev = torch.device("cuda:0")
    cfg = weights.XL2
    W = weights.init_weights(cfg, seed=3, device=dev)
    model = STDiTModel(cfg, W, dev)
    del W
    rows = []
    for label in a.labels:
        sh = shapes.shape_of(label)
        z0, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
        for P in dops:
            t0 = time.time()
            row = {"resolution": label, "dop": P, "latent": list(sh.latent), "T": sh.T, "S": sh.S}
            if P == 1:
                req = StepRequest(model, sh, y)
                z = z0.clone().contiguous()
                req.graph_step(z, 1)
                torch.cuda.synchronize()
                row["step_ms"] = ev_time(lambda: req.graph_step(z, 1), a.reps)
                req.profile(True)
                req.step(z, 1)
                prof = req.profile_read()
                req.profile(False)
                row["rank_ms"] = [{k: round(v[0], 4) for k, v in prof.items()}]
                row["projected_ms"] = row["step_ms"]
                req.close()
                del req
            else:
                grp = VirtualGroup(model, sh, y, P)
                parts = grp.split(z0)
                grp.step(parts, 1)
                torch.cuda.synchronize()
                row["group_serial_ms"] = ev_time(lambda: grp.step(parts, 1), a.reps)
                timed = [grp.step_timed(parts, 1) for _ in range(a.reps)]
                row["rank_step_ms"] = [round(min(t[r] for t in timed), 4) for r in range(P)]
                for r in grp.ranks:
                    r.profile(True)
                grp.step(parts, 1)
                torch.cuda.synchronize()
                per = []
                for r in grp.ranks:
                    prof = r.profile_read()
                    r.profile(False)
                    per.append({k: round(v[0], 4) for k, v in prof.items()})
                row["rank_ms"] = per
                xb = [exchange_bytes(sh, P, r, cfg.hidden) for r in range(P)]
                row["exchange_bytes_per_rank"] = xb
                row["nvlink_ms_model"] = round(max(xb) / (NVLINK_GBS * 1e9) * 1e3, 4)
                # rank time from per-phase events (its kernels + its local exchange pushes, no
                # per-launch event gaps); the pushes then cross NVLink instead of local HBM
                comp = max(row["rank_step_ms"])
                row["projected_ms"] = round(comp + row["nvlink_ms_model"], 4)
                row["virtual"] = True
                for r in grp.ranks:
                    r.close()
                del grp, parts
            # roofline: algorithmic FLOPs of the step (bench.step_flops) per GPU over the
            # (projected) latency, against the measured sustained bf16 peak
            fl = step_flops(cfg, sh)["total"]
            row["step_tflop"] = round(fl / 1e12, 3)
            row["tflops_per_gpu"] = round(fl / P / (row["projected_ms"] * 1e-3) / 1e12, 1)
            row["frac_of_sustained_bf16"] = round(row["tflops_per_gpu"] / PEAK_TFLOPS, 3)
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            row["wall_s"] = round(time.time() - t0, 1)
            print(json.dumps(row), flush=True)
            rows.append(row)
    doc = {"gpu": torch.cuda.get_device_name(0), "model": "STDiT3-XL/2 (random init)", "cfg_batch": 2,
           "nvlink_gbs_model": NVLINK_GBS, "rows": rows}
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
