"""Cross-check the B200-measured profile in the UNMODIFIED reference simulator.

Run in the build container (where /root/reference exists; CPU only):
    python scripts/reference_crosscheck.py [profiles/r01_trace_replay_c5.json]
Loads the dit-profile/1 document that scripts/trace_replay.py measured on a B200, feeds it to the
reference ``ditsim`` (read-only import from /root/reference/pkg/src) -- load_profiles,
derive_dop_table, generate, Simulation + GreedyPolicy, compute_metrics -- for the same config-5
workload, and records the reference's predicted avg / p99 latency and GPU-seconds next to this
repo's own prediction (sched, bit-exact re-implementation) and the replay that executed every
step on the GPU, plus the reference's occupancy lower bound (optimal.solve_optimal) for the
cost-over-optimum. Output: profiles/r01_reference_crosscheck.json (read by
tests/test_sched_golden.py::test_reference_crosscheck_of_b200_profile).
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")


def main() -> None:
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r01_trace_replay_c5.json"
    run = json.loads(src.read_text())
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    import ditsim as ds  # the unmodified reference

    table = ds.load_profiles(run["profile"])
    dt = ds.derive_dop_table(table)
    mix = {k: 1 / 3 for k in ("144p", "240p", "360p")}
    out = {"source": str(src.relative_to(ROOT)), "b_values": dict(dt.by_resolution), "rates": {}}
    for rate in sorted(set(run["predicted"]) | set(run["replayed"]), key=float):
        spec = ds.WorkloadSpec(proportions=mix, total_requests=run["requests"], arrival_rate=float(rate),
                               seed=0, denoise_steps=run["denoise_steps"])
        res = ds.Simulation(ds.ClusterTopology(1, 8), table, dt, ds.generate(spec), ds.GreedyPolicy(dt)).run()
        m = ds.compute_metrics(res)
        out["rates"][rate] = {
            "reference": {"avg_latency_s": round(m.avg_latency, 4), "p99_latency_s": round(m.p99_latency, 4),
                          "gpu_seconds": round(m.cumulative_occupancy, 3)},
            "ours_predicted": run["predicted"].get(rate),
            "b200_replayed": run["replayed"].get(rate),
        }
        print(rate, out["rates"][rate], flush=True)
    # the reference's occupancy lower bound for the same mix (optimal.solve_optimal with the batch
    # model, as its experiment harness computes it, experiment.py:289-308) -> cost over optimum of
    # the greedy trace on the B200-measured profile
    from ditsim.optimal import BatchModel, InfeasibleError, solve_optimal

    try:
        opt = solve_optimal(ds.ClusterTopology(1, 8), table, mix, BatchModel(run["requests"]),
                            steps=run["denoise_steps"], include_vae=True)
        out["optimal_gpu_seconds"] = round(opt.total_gpu_seconds, 3)
        for rec in out["rates"].values():
            rec["reference"]["cost_over_optimum"] = round(rec["reference"]["gpu_seconds"] / opt.total_gpu_seconds, 4)
            if rec.get("b200_replayed"):
                rec["b200_replayed_cost_over_optimum"] = round(
                    rec["b200_replayed"]["gpu_seconds"] / opt.total_gpu_seconds, 4)
    except InfeasibleError as e:  # pragma: no cover
        out["optimal_gpu_seconds"] = None
        out["optimal_error"] = str(e)
    print("optimal GPU-seconds:", out.get("optimal_gpu_seconds"), flush=True)
    (ROOT / "profiles" / "r01_reference_crosscheck.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
