"""Scheduling parity: paper_2506_13497_b200.sched replays the reference's own recorded
outputs (tests/golden/sched_golden.json.gz, generated from /root/reference by
tests/golden/make_sched_golden.py) and must match bit for bit."""
import gzip
import hashlib
import json
from pathlib import Path

import pytest

from paper_2506_13497_b200 import sched

G = json.loads(gzip.decompress((Path(__file__).parent / "golden" / "sched_golden.json.gz").read_bytes()))


def h(x):
    return float(x).hex()


def test_profiles_b_values_and_change_rates():
    for case in G["profiles"]:
        t = sched.load_profiles(case["doc"])
        for thr, want in case["optimal"].items():
            got = {r.name: sched.optimal_dop(t, r.name, float(thr)) for r in t.resolutions}
            assert got == want
        for name, rates in case["change"].items():
            assert [h(sched.change_rate(t, name, d)) for d in (2, 4, 8)] == rates


def test_default_profile_b_values():
    t = sched.load_profiles(G["default_profile"])
    assert sched.derive_dop_table(t).by_resolution == {"144p": 1, "240p": 2, "360p": 4}


def test_default_profile_matches_reference_bundle():
    """sched.default_profile() == the reference's bundled document (ditsim.default_profile(),
    reference profiles.py:291-300), recorded in the golden file."""
    a = sched.default_profile()
    b = sched.load_profiles(G["default_profile"])
    assert a == b
    assert sched.derive_dop_table(a).by_resolution == {"144p": 1, "240p": 2, "360p": 4}
    # the 360p VAE share at DoP 4 is exactly 1/7 (reference test_profiles.py:170-173)
    total = sched.estimate_execution_time(a, "360p", 4, 30)
    assert abs(a.vae("360p") / total - 1 / 7) <= 1e-12


def _handle(spec):
    return sched.AllocationHandle(tuple(sched.Block(s, o) for s, o in spec))


def _hid(hd):
    return [[b.start, b.order] for b in hd.blocks]


@pytest.mark.parametrize("idx", range(12))
def test_allocator_replay(idx):
    case = G["alloc"][idx]
    pool = sched.GpuPool(sched.ClusterTopology(case["nodes"], case["gpn"]))
    for step, op in enumerate(case["log"]):
        kind = op["op"]
        if kind == "allocate":
            r = pool.allocate(op["size"])
            got = None if r is None else _hid(r)
        elif kind == "allocate_group":
            r = pool.allocate_group(op["size"])
            got = None if r is None else _hid(r)
        elif kind == "release":
            pool.release(_handle(op["handle"]))
            got = None
        elif kind == "keep_lowest":
            kept, freed = pool.release_keep_lowest(_handle(op["handle"]), op["keep"])
            got = [_hid(kept), list(freed)]
        elif kind == "try_best":
            r = pool.try_best_alloc(op["target"], None, (1, 2, 4, 8))
            got = None if r is None else _hid(r)
        elif kind == "try_best_grow":
            held = _handle(op["handle"])
            r = pool.try_best_alloc(op["target"], held, (1, 2, 4, 8))
            got = {"same": r is held, "handle": _hid(r)}
        elif kind == "retract":
            got = list(pool.retract_to(_handle(op["handle"]), _handle(op["sub"])))
        else:  # pragma: no cover
            raise AssertionError(kind)
        assert got == op["result"], (step, op)
        assert pool.snapshot() == op["snapshot"], (step, kind)


def test_workload_streams():
    for case in G["workloads"]:
        recs = sched.generate(sched.WorkloadSpec(**case["spec"]))
        assert [[r.request_id, h(r.arrival_time), r.resolution, r.denoise_steps] for r in recs] == case["records"]


def _policy(key, dt):
    if key == "greedy":
        return sched.GreedyPolicy(dt)
    if key == "greedy-nopromo":
        return sched.GreedyPolicy(dt, promotion=False)
    if key == "sdop4-dec":
        return sched.StaticDopPolicy(4, decouple_vae=True)
    return sched.StaticDopPolicy(int(key[4:]))


PROFILES = {}


@pytest.mark.parametrize("idx", range(len(G["sims"])))
def test_simulation_replay(idx):
    case = G["sims"][idx]
    prof_docs = {"default": G["default_profile"]}
    if case["profile"] not in prof_docs:
        from golden.make_sched_golden import random_profile_doc

        prof_docs[case["profile"]] = random_profile_doc(int(case["profile"][4:]))
    t = sched.load_profiles(prof_docs[case["profile"]])
    dt = sched.derive_dop_table(t, vae_dop=case["vae_dop"])
    recs = sched.generate(sched.WorkloadSpec(proportions=case["mix"], **case["workload"]))
    res = sched.Simulation(sched.ClusterTopology(*case["topology"]), t, dt, recs,
                           _policy(case["policy_key"], dt)).run()
    m = sched.compute_metrics(res)
    trace = "".join(r.to_json_line() + "\n" for r in res.trace)
    if "trace" in case:
        assert trace == case["trace"]
    assert hashlib.sha256(trace.encode()).hexdigest() == case["trace_sha256"]
    assert res.policy_name == case["policy"]
    assert h(res.cumulative_occupancy) == case["occupancy"]
    assert h(m.avg_latency) == case["avg"] and h(m.p99_latency) == case["p99"]
    got = [[r.request_id, r.resolution, h(r.arrival), h(r.start), h(r.finish), h(r.gpu_seconds),
            [[h(a), w] for a, w in r.dop_history]] for r in res.requests]
    assert got == case["requests"]


def test_reference_crosscheck_of_b200_profile():
    """The dit-profile/1 document measured on a B200 (profiles/r01_trace_replay_c5.json), fed to
    the unmodified reference simulator (scripts/reference_crosscheck.py, run where
    /root/reference exists), and to this repo's scheduler give the same config-5 predictions."""
    import json
    from pathlib import Path

    from paper_2506_13497_b200 import sched

    root = Path(__file__).resolve().parents[1]
    run = json.loads((root / "profiles" / "r01_trace_replay_c5.json").read_text())
    ref = json.loads((root / "profiles" / "r01_reference_crosscheck.json").read_text())
    table = sched.load_profiles(run["profile"])
    dt = sched.derive_dop_table(table)
    assert dict(dt.by_resolution) == ref["b_values"]
    mix = {k: 1 / 3 for k in ("144p", "240p", "360p")}
    for rate, rec in ref["rates"].items():
        spec = sched.WorkloadSpec(proportions=mix, total_requests=run["requests"],
                                  arrival_rate=float(rate), seed=0, denoise_steps=run["denoise_steps"])
        res = sched.Simulation(sched.ClusterTopology(1, 8), table, dt, sched.generate(spec),
                               sched.GreedyPolicy(dt)).run()
        m = sched.compute_metrics(res)
        assert round(m.avg_latency, 4) == rec["reference"]["avg_latency_s"]
        assert round(m.p99_latency, 4) == rec["reference"]["p99_latency_s"]
        assert round(m.cumulative_occupancy, 3) == rec["reference"]["gpu_seconds"]
