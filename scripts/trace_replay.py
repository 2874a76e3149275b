"""BASELINE config 5: a mixed-resolution Poisson trace through the greedy step-granularity
allocator on 8 GPUs, driven by B200-measured step times.

1. Profile (on this B200): STDiT3-XL/2 step latency per resolution at DoP 1 (measured) and DoP
   2/4/8 (every rank's kernels measured as virtual ranks on this GPU, max over ranks + its exchange
   bytes over NVLink at the measured 770 GB/s), VAE decode per resolution (measured). Emitted as the
   reference's dit-profile/1 document; B values derived with derive_dop_table
   (reference profiles.py:276-288).
2. Predicted: the reference semantics in virtual time (sched.Simulation, executor=None) over the
   workload `generate(WorkloadSpec(1/3 144p / 240p / 360p, 48 requests, rate, seed 0))`
   (reference workload.py:97-126, configs/experiment.json mix) -> avg / p99 latency and
   GPU-seconds (reference metrics.py:40-54).
3. Replayed: the same engine with B200Executor -- every denoise step and every VAE decode of every
   request actually runs on the GPU (DoP-P groups as virtual ranks, reported at their emulated
   P-GPU latency), the clock advanced by the measured durations -> the same metrics.
Usage: python scripts/trace_replay.py [--rates 0.25,0.5,0.75,1.0] [--real-rates 0.5,1.0]
                                      [--requests 48] [--steps 30] [--out gpurun_out/trace_replay.json]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2506_13497_b200 import sched, shapes, weights
from paper_2506_13497_b200.executor import B200Executor
from paper_2506_13497_b200.sched.engine import RequestState
from paper_2506_13497_b200.vae import VAEDecoder
from paper_2506_13497_b200.vae_weights import OPENSORA_VAE, init_vae_weights

LABELS = ("144p", "240p", "360p")


def metrics_of(res) -> dict:
    m = sched.compute_metrics(res)
    kinds = [r.kind for r in res.trace]
    return {"avg_latency_s": round(m.avg_latency, 4), "p99_latency_s": round(m.p99_latency, 4),
            "gpu_seconds": round(m.cumulative_occupancy, 3), "promotions": kinds.count("promotion")}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rates", default="0.25,0.5,0.75,1.0")
    ap.add_argument("--real-rates", default="0.5,1.0")
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default="gpurun_out/trace_replay.json")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = weights.XL2
    W = weights.init_weights(cfg, seed=3, device=dev)
    vW = init_vae_weights(OPENSORA_VAE, seed=7, device=dev)
    t0 = time.time()

    # ---- 1. profile
    ex = B200Executor(cfg, W, num_steps=a.steps, emulate_group=True)
    entries = []
    for res in LABELS:
        sh = shapes.shape_of(res)
        for d in (1, 2, 4, 8):
            req = RequestState(90_000 + len(entries), res, 0.0, a.steps)
            ex.dit_step(req, tuple(range(d)), 0, None)  # open + warm-up
            times = [ex._run_step(ex.live[req.request_id], 1 + i) for i in range(5)]
            ex._close(ex.live.pop(req.request_id))
            e = {"resolution": res, "dop": d, "dit_step_seconds": round(min(times), 6)}
            if d == 1:
                dec = VAEDecoder(OPENSORA_VAE, vW, dev)
                z = torch.randn((1, cfg.in_channels, *sh.latent), device=dev)
                dec.decode(z, sh.frames, sh.height, sh.width)
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                dec.decode(z, sh.frames, sh.height, sh.width)
                s1.record()
                s1.synchronize()
                e["vae_seconds"] = round(s0.elapsed_time(s1) / 1e3, 6)
                del dec
            else:
                e["emulated"] = True
            entries.append(e)
            print(json.dumps(e), flush=True)
    ex.step_seconds.clear()
    doc = {"schema": "dit-profile/1", "dop_candidates": [1, 2, 4, 8], "entries": entries}
    table = sched.load_profiles(doc)
    dt = sched.derive_dop_table(table)
    print("B values:", dt.by_resolution, flush=True)
    out = {"gpu": torch.cuda.get_device_name(0), "profile": doc, "b_values": dt.by_resolution,
           "topology": "1 node x 8 GPUs", "requests": a.requests, "denoise_steps": a.steps,
           "mix": {k: "1/3" for k in LABELS}, "predicted": {}, "replayed": {}}
    topo = sched.ClusterTopology(1, 8)
    mix = {k: 1 / 3 for k in LABELS}

    def workload(rate):
        spec = sched.WorkloadSpec(proportions=mix, total_requests=a.requests, arrival_rate=rate,
                                  seed=0, denoise_steps=a.steps)
        return sched.generate(spec)

    # ---- 2. predicted (virtual time, reference semantics)
    for r in [float(x) for x in a.rates.split(",") if x]:
        t1 = time.perf_counter()
        res = sched.Simulation(topo, table, dt, workload(r), sched.GreedyPolicy(dt)).run()
        out["predicted"][f"{r:g}"] = {**metrics_of(res),
                                      "sim_seconds": round(time.perf_counter() - t1, 4)}
        print("predicted", r, out["predicted"][f"{r:g}"], flush=True)

    # ---- 3. replayed (every step and decode executed on the B200)
    for r in [float(x) for x in a.real_rates.split(",") if x]:
        t1 = time.time()
        rex = B200Executor(cfg, W, num_steps=a.steps, emulate_group=True, vae_cfg=OPENSORA_VAE,
                           vae_weights=vW)
        tp = time.time()
        ngroups = rex.preopen(LABELS, 8)  # the 15 buddy groups per resolution, opened up front
        t_pre = time.time() - tp
        res = sched.Simulation(topo, table, dt, workload(r), sched.GreedyPolicy(dt), executor=rex).run()
        steps = len(rex.step_seconds)
        out["replayed"][f"{r:g}"] = {
            **metrics_of(res), "steps_executed": steps, "vae_decodes": len(rex.vae_seconds),
            "reshards": len(rex.reshard_seconds),
            "reshard_ms_max": round(1e3 * max(rex.reshard_seconds), 3) if rex.reshard_seconds else None,
            # promotion cost on a real P'-GPU group: host work (re-bind + enqueue) + the slowest
            # new rank's device time (ranks re-shard concurrently on their own GPUs)
            "reshard_host_ms_max": (round(1e3 * max(rex.reshard_host_seconds), 3)
                                    if rex.reshard_host_seconds else None),
            "reshard_host_ms_mean": (round(1e3 * sum(rex.reshard_host_seconds)
                                           / len(rex.reshard_host_seconds), 3)
                                     if rex.reshard_host_seconds else None),
            "promotion_ms_max": (round(1e3 * max(h + d for h, d in zip(rex.reshard_host_seconds,
                                                                        rex.reshard_seconds)), 3)
                                 if rex.reshard_seconds else None),
            # wall time until done on THIS box: the emulated group's virtual ranks re-shard one
            # after another on one GPU, so it is ~P' x the device time (not a multi-GPU number)
            "reshard_wall_ms_max_emulated": (round(1e3 * max(rex.reshard_wall_seconds), 3)
                                             if rex.reshard_wall_seconds else None),
            "reshard_ms_mean": (round(1e3 * sum(rex.reshard_seconds) / len(rex.reshard_seconds), 3)
                                if rex.reshard_seconds else None),
            "preopened_groups": ngroups, "preopen_seconds": round(t_pre, 2),
            "handoff_ms_max": round(1e3 * max(h for _, h, _ in rex.vae_seconds), 3),
            "wall_seconds": round(time.time() - t1, 1)}
        print("replayed", r, out["replayed"][f"{r:g}"], flush=True)
        rex.close()
        for m in rex.models.values():
            m.close()
        del rex
        torch.cuda.empty_cache()
    out["wall_seconds"] = round(time.time() - t0, 1)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
