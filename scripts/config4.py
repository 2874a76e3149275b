"""BASELINE config 4: one request on a DiT group of DoP 4 decoupled from a VAE group of DoP 1 / 2
(StaticDopPolicy(4, decouple_vae=True, vae_dop=q), the reference policies.py:151-190 semantics),
every step, the latent hand-off and the VAE decode executed on this B200 (DoP-4 group as virtual
ranks reported at its emulated 4-GPU latency; VAE ranks one after another, the slowest counted).
Usage: python scripts/config4.py [240p 360p ...] [--steps 30] [--out gpurun_out/config4.json]"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import sched, weights
from paper_2506_13497_b200.executor import B200Executor
from paper_2506_13497_b200.vae_weights import OPENSORA_VAE, init_vae_weights


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("labels", nargs="*", default=["240p", "360p"])
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default="gpurun_out/config4.json")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = weights.XL2
    W = weights.init_weights(cfg, seed=3, device=dev)
    vW = init_vae_weights(OPENSORA_VAE, seed=7, device=dev)
    # the profile only has to make DoP 4 a candidate; the executor measures everything
    doc = json.loads((Path(__file__).resolve().parents[1] / "profiles" / "r01_trace_replay_c5.json").read_text())
    table = sched.load_profiles(doc["profile"])
    rows = []
    for label in a.labels:
        for q in (1, 2):
            dt = sched.derive_dop_table(table, vae_dop=q)
            ex = B200Executor(cfg, W, num_steps=a.steps, emulate_group=True, vae_cfg=OPENSORA_VAE,
                              vae_weights=vW)
            wl = [sched.ArrivalRecord(0, 0.0, label, a.steps)]
            # warm-up request (opens the group, captures nothing the timed one reuses unfairly:
            # the pooled rank state is re-bound to the new caption as in serving)
            sched.Simulation(sched.ClusterTopology(1, 4), table, dt, wl,
                             sched.StaticDopPolicy(4, decouple_vae=True, vae_dop=q), executor=ex).run()
            ex.step_seconds.clear()
            ex.vae_seconds.clear()
            res = sched.Simulation(sched.ClusterTopology(1, 4), table, dt,
                                   [sched.ArrivalRecord(1, 0.0, label, a.steps)],
                                   sched.StaticDopPolicy(4, decouple_vae=True, vae_dop=q), executor=ex).run()
            m = sched.compute_metrics(res)
            steps = [s for _, _, s in ex.step_seconds]
            _, handoff, decode = ex.vae_seconds[-1]
            row = {"resolution": label, "dit_dop": 4, "vae_dop": q, "steps": len(steps),
                   "dit_seconds": round(sum(steps), 4), "step_ms_mean": round(1e3 * sum(steps) / len(steps), 3),
                   "handoff_ms": round(1e3 * handoff, 3), "vae_decode_ms": round(1e3 * decode, 2),
                   "request_latency_s": round(m.avg_latency, 4), "gpu_seconds": round(m.cumulative_occupancy, 3)}
            print(json.dumps(row), flush=True)
            rows.append(row)
            ex.close()
            for mdl in ex.models.values():
                mdl.close()
            del ex
            torch.cuda.empty_cache()
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"gpu": torch.cuda.get_device_name(0), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
