#!/usr/bin/env python
"""bench.py -- the DDiT hot path on B200: one STDiT3-XL/2 denoise step (RFLOW, CFG batch 2)
at 240p x 51 frames (latent 15x30x54, N = 6075 tokens per sample), BASELINE.json configs[1],
at DoP = --gpus (one process per GPU, DSP sequence parallelism inside the step).

Metric (BASELINE.json): STDiT denoise-step latency at DoP 1/2/4/8 -> "value" is the latency
of one step in ms (lower is better), device-timed with CUDA events over exactly --steps steps
after --warmup untimed ones, max over ranks. "e2e" is the same step through the public API
with the latent in pinned host memory (H2D of z and D2H of z' inside the timed region).

Usage:  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
        N > 1 runs one process per GPU: under torchrun (the driver's launch), or, when started
        as a plain process, bench.py spawns the N ranks itself through torch.distributed.run.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

LABEL = "240p"
METRIC = "stdit_denoise_step_latency"


def parse() -> argparse.Namespace:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--label", default=LABEL)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly, no CUDA graph")
    ap.add_argument("--xch", default="fused", choices=["fused", "kernel", "nccl"],
                    help="DoP > 1 all-to-all: fused into the fc2 GEMM epilogue (peer stores, "
                         "default), the stand-alone peer-store kernel, or packed rows through "
                         "ncclAllToAll (the baseline arm)")
    return ap.parse_args()


# ------------------------------------------------------------------ algorithmic work
def step_flops(cfg, shape, include_text_kv: bool = True) -> dict:
    """FLOPs of one CFG step: per block pair 2*28*N*C^2 linear +
    4*T*S^2*C spatial + 4*S*T^2*C temporal attention + 2*4*N*Ly*C cross attention, plus the
    (cacheable, computed once per request here) 2*4*Ly*C^2 text K/V projection; + 64*N*C exit."""
    B, C, Ly, L = 2, cfg.hidden, cfg.text_tokens, cfg.depth
    T, S = shape.T, shape.S
    N = T * S
    lin = 2 * 28 * N * C * C
    sp = 4 * T * S * S * C
    tp = 4 * S * T * T * C
    cr = 2 * 4 * N * Ly * C
    kv = 2 * 4 * Ly * C * C
    total = B * (L * (lin + sp + tp + cr + (kv if include_text_kv else 0)) + 64 * N * C)
    return {"total": total, "gemm": B * L * lin, "attention": B * L * (sp + tp + cr)}


def load_peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU baseline (oracle)
_ORACLE = {}


def _oracle_state(label: str):
    """Weights / inputs of the CPU oracle for the full 28-layer XL/2 step (built once)."""
    if label not in _ORACLE:
        from oracle import stdit3  # the checker / CPU baseline only
        from paper_2506_13497_b200 import shapes, weights

        torch.set_num_threads(os.cpu_count() or 1)
        cfg = weights.XL2
        sh = shapes.shape_of(label)
        W = weights.init_weights(cfg, seed=3)
        z, y = weights.synthetic_inputs(cfg, sh.latent)
        with torch.inference_mode():
            text = stdit3.prepare_text(W, y)
        _ORACLE[label] = (cfg, sh, W, z, text)
    return _ORACLE[label]


def cpu_reference_step_ms(label: str, step: int = 3) -> tuple[float, dict]:
    """ONE real step of the fp32 torch-CPU restatement (oracle/stdit3.py) on the host cores:
    STDiT3-XL/2, all 28 block pairs, the bench's shape, CFG batch 2 -- the same workload as the
    GPU arm, timed (no extrapolation)."""
    from oracle import stdit3

    cfg, sh, W, z, text = _oracle_state(label)
    with torch.inference_mode():
        t0 = time.perf_counter()
        stdit3.denoise_step(W, cfg, z, text, step, sh.height, sh.width)
        ms = (time.perf_counter() - t0) * 1e3
    info = {
        "cores": torch.get_num_threads(),
        "cpu": _cpu_model(),
        "sample": (f"one full STDiT3-XL/2 denoise step (28 block pairs, {label} x 51, CFG batch 2) "
                   "of the fp32 torch-CPU oracle port, timed end to end"),
    }
    return ms, info


def _cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sched_cpu_baseline() -> dict:
    """SURVEY.md §8(d) CPU path (1): the scheduling loop itself -- the greedy step-granularity
    allocator + serving engine (sched.Simulation + GreedyPolicy, the reference semantics
    bit for bit) on BASELINE config 5's trace (48 requests, 1/3 each 144p/240p/360p, Poisson
    rate 1.0, seed 0, 8 GPUs) in virtual time, fed the B200-measured profile. Host cost per
    step event, single-threaded Python."""
    from paper_2506_13497_b200 import sched

    doc = None
    f = ROOT / "profiles" / "r01_trace_replay_c5.json"
    if f.exists():
        try:
            doc = json.loads(f.read_text())["profile"]
        except Exception:
            doc = None
    table = sched.load_profiles(doc) if doc else sched.default_profile()
    dt = sched.derive_dop_table(table)
    spec = sched.WorkloadSpec(proportions={"144p": 1 / 3, "240p": 1 / 3, "360p": 1 / 3},
                              total_requests=48, arrival_rate=1.0, seed=0)
    best = None
    for _ in range(5):
        wl = sched.generate(spec)
        t0 = time.perf_counter()
        res = sched.Simulation(sched.ClusterTopology(1, 8), table, dt, wl, sched.GreedyPolicy(dt)).run()
        el = time.perf_counter() - t0
        best = el if best is None else min(best, el)
    nstep = sum(1 for r in res.trace if r.kind == sched.EventKind.STEP_COMPLETE)
    m = sched.compute_metrics(res)
    return {"value": round(best / max(nstep, 1) * 1e6, 2), "unit": "us/step_event", "cores": 1,
            "kind": "port", "step_events": nstep, "sim_seconds": round(best, 4),
            "avg_latency_s": round(m.avg_latency, 4), "p99_latency_s": round(m.p99_latency, 4),
            "profile": "B200-measured (profiles/r01_trace_replay_c5.json)" if doc else "default",
            "sample": "config-5 trace, 48 requests, rate 1.0, seed 0, 1 node x 8 GPUs, best of 5"}


# ------------------------------------------------------------------ our arm
def run_ours(args) -> dict | None:
    import torch.distributed as dist

    from paper_2506_13497_b200 import shapes, weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest, launch_count

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one GPU per rank; on a box with fewer GPUs than ranks (a 1-GPU test box) the ranks share
    # devices round-robin and the plumbing falls back to gloo (NCCL needs a GPU per rank)
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    shared_gpus = world > ndev
    if args.xch == "kernel":
        os.environ["DDIT_FUSED_XCH"] = "0"
    if world > 1:
        if shared_gpus:
            if args.xch == "nccl":
                raise SystemExit("--xch nccl needs one GPU per rank (NCCL rejects shared devices)")
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = weights.XL2
    sh = shapes.shape_of(args.label)
    # random-init XL/2 weights on the device (same seed on every rank)
    W = weights.init_weights(cfg, seed=3, device=dev)
    model = STDiTModel(cfg, W, dev)
    del W
    torch.cuda.empty_cache()
    z_full, y = weights.synthetic_inputs(cfg, sh.latent, device=dev)
    grp = None
    if world > 1 and args.xch == "nccl":
        from paper_2506_13497_b200.dist import NcclGroupStep

        grp = NcclGroupStep(model, sh, y)
        req = grp.req
    elif world > 1:
        from paper_2506_13497_b200.dist import GroupStep

        grp = GroupStep(model, sh, y)
        req = grp.req
    else:
        req = StepRequest(model, sh, y)
    sd = req.shard
    z = z_full[:, :, sd.t_lo:sd.t_hi].contiguous()
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    nccl = world > 1 and args.xch == "nccl"
    use_graph = not args.no_graph and not nccl  # the NCCL arm launches eagerly
    run_step = grp.step if nccl else (req.graph_step if use_graph else req.step)
    for i in range(args.warmup):
        run_step(z, i % 30) if nccl else req.step(z, i % 30)
    if use_graph:  # capture every step index the timed loops use (outside the timed region)
        for i in range(args.steps):
            run_step(z, (args.warmup + i) % 30)
    barrier()

    # ---- device-timed region: K steps, inputs resident in HBM
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = launch_count()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        run_step(z, (args.warmup + i) % 30)
    e1.record(stream)
    barrier()
    launches = launch_count() - launches0
    if world > 1:
        req.status()  # raises if a peer never signalled (bounded barrier spin)
    if use_graph:  # graph replays do not pass through the launch counter: count one step
        l0 = launch_count()
        req.step(z, 0)
        launches = (launch_count() - l0) * args.steps
        barrier()
    ms_step = e0.elapsed_time(e1) / args.steps

    # ---- the same K steps again with an event pair around every launch (roofline evidence:
    # per-kernel-class device time on the launching stream)
    req.profile(True)
    if nccl:
        grp.timing = True
        grp.read_timing()
    barrier()
    e0.record(stream)
    for i in range(args.steps):
        (grp.step if nccl else req.step)(z, (args.warmup + i) % 30)
    e1.record(stream)
    barrier()
    ms_total = e0.elapsed_time(e1)
    prof = req.profile_read()
    req.profile(False)
    a2a_ms = grp.read_timing() / args.steps if nccl else None
    if nccl:
        grp.timing = False
    clk = clocks.stop()

    # ---- e2e: through the public step API with the latent in pinned host memory
    z_host = z.cpu().pin_memory()
    barrier()
    e0.record(stream)
    for i in range(args.steps):
        z.copy_(z_host, non_blocking=True)
        run_step(z, (args.warmup + i) % 30)
        z_host.copy_(z, non_blocking=True)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    zbytes = z.numel() * 4

    if world > 1:
        from paper_2506_13497_b200.executor import exchange_bytes

        xb = exchange_bytes(sh, world, rank, cfg.hidden)
        xfer_ms = a2a_ms if nccl else prof["exchange"][0] / args.steps
    cdev = torch.device("cpu") if shared_gpus else dev
    t_step = torch.tensor([ms_step, e2e_ms], device=cdev)
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
        zb = torch.tensor([zbytes], device=cdev, dtype=torch.float64)
        dist.all_reduce(zb)
        zbytes = int(zb.item())
    ms_step, e2e_ms = t_step.tolist()
    if rank != 0:
        dist.destroy_process_group()
        return None

    fl = step_flops(cfg, sh, include_text_kv=False)
    peaks, peak_src = load_peaks()
    gemm_ms, gemm_n = prof["gemm"]
    # GEMM FLOPs this rank executed per step (its M rows), over the timed steps
    M_sp = 2 * (sd.t_hi - sd.t_lo) * sh.S
    M_tp = 2 * sh.T * (sd.s_hi - sd.s_lo)
    gemm_flops_step = cfg.depth * (M_sp + M_tp) * 14 * cfg.hidden * cfg.hidden * 2
    achieved = gemm_flops_step * args.steps / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    traffic = None
    tfile = ROOT / "profiles" / "gemm_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    out = {
        "metric": METRIC,
        "value": round(ms_step, 4),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) latent and caption embedding; random-init XL/2 weights)",
        "config": {
            "workload": f"STDiT3-XL/2 denoise step, {args.label} x 51 frames "
                        f"(latent {sh.T}x{sh.latent[1]}x{sh.latent[2]}, {sh.N} tokens/sample), "
                        "CFG batch 2, RFLOW Euler update",
            "dop": world,
            "parallelism": (f"sp{world} (DSP T-shard/S-shard all-to-all: "
                            + {"fused": "fused into the fc2 GEMM epilogue as peer stores",
                               "kernel": "stand-alone peer-store exchange kernel",
                               "nccl": "packed rows through ncclAllToAll"}[args.xch] + ")"
                            + (f"; {world} ranks sharing {ndev} GPU(s): not a scaling number"
                               if shared_gpus else "")) if world > 1 else "none",
            "step_tflop": round(fl["total"] / 1e12, 3),
            "l2": "inputs larger than L2 (2.2 GB of bf16 weights + >1 GB activations per step)",
            "launch": "CUDA graph per step index (captured before the timed region)" if use_graph
                      else "eager launches",
        },
        "e2e": {
            "value": round(e2e_ms, 4),
            "unit": "ms",
            "h2d_bytes_per_step": zbytes,
            "d2h_bytes_per_step": zbytes,
        },
        "gpu_launches": int(launches),
        "achieved_step_tflops": round(fl["total"] / (ms_step * 1e-3) / 1e12, 1),
        "roofline": {
            "bound": "tensor",
            "kernel": "tcgen05 GEMM (gemm_bf16_tn_kernel)",
            "achieved": round(achieved, 1) if achieved else None,
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4) if achieved else None,
            "traffic": traffic,
            "peak_source": peak_src + " bf16 sustained",
            "gemm_launches": gemm_n,
            "share_of_step": round(gemm_ms / ms_total, 4) if ms_total > 0 else None,
            "how": "second timed pass of the same K steps with a CUDA-event pair around every "
                   "launch on the launching stream; achieved = executed GEMM FLOPs / GEMM time",
        },
        "breakdown_ms_per_step": {k: round(v[0] / args.steps, 3) for k, v in prof.items()},
        "clocks": clk,
    }
    if world > 1:
        xi = {"mode": args.xch, "bytes_per_rank_per_step": xb,
              "exchanges_per_step": 2 * cfg.depth, "row_dtype": "f32"}
        if nccl:
            xi.update({"a2a_ms_per_step_rank0": round(xfer_ms, 3),
                       "nvlink_gbs_rank0": round(xb / (xfer_ms * 1e-3) / 1e9, 1) if xfer_ms else None,
                       "how": "CUDA events around every all_to_all_single on rank 0"})
        else:
            xi.update({"barrier_wait_ms_per_step_rank0": round(xfer_ms, 3),
                       "how": "rows stored into peer memory by the fc2 epilogue (fused) or the "
                              "exchange kernel; the listed time is the flag-barrier wait"})
        if shared_gpus:
            xi["note"] = "ranks share one GPU: peer stores are local, no NVLink figure"
        out["exchange"] = xi
    if world == 1 and not args.no_cpu_baseline:
        cms, info = cpu_reference_step_ms(args.label)
        out["cpu_baseline"] = {"value": round(cms, 1), "unit": "ms", "kind": "port", **info}
        out["cpu_baseline_sched"] = sched_cpu_baseline()
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(args) -> dict | None:
    """The reference has no STDiT implementation (it looks the step time up,
    reference pkg/src/ditsim/profiles.py:69-76); its CPU implementation of the path is therefore
    the oracle port (fp32 torch, every host core), run on the SAME workload as our arm: each of
    the W + K steps is one full 28-layer XL/2 step at the bench shape (no extrapolation)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    vals = []
    info = {}
    t_start = time.perf_counter()
    for i in range(args.warmup + args.steps):
        ms, info = cpu_reference_step_ms(args.label, step=(i % 30))
        if i >= args.warmup:
            vals.append(ms)
    v = sum(vals) / len(vals)
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 1),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(v, 1),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded N(0,1) latent and caption embedding; random-init XL/2 weights)",
        "config": {"workload": f"STDiT3-XL/2 denoise step, {args.label} x 51 frames (28 block pairs), "
                               "CFG batch 2 (fp32 CPU oracle port; the reference ships no model code)",
                   "dop": 1},
        "cpu_baseline": {"value": round(v, 1), "unit": "ms", "kind": "port", **info,
                         "min_ms": round(min(vals), 1), "max_ms": round(max(vals), 1)},
        "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_seconds": round(time.perf_counter() - t_start, 1),
    }


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: launch the N ranks ourselves (one process per GPU, the same
    command the driver uses) and pass rank 0's JSON line through."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
