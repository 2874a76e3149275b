"""Generate the scheduling golden fixtures FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):
    python tests/golden/make_sched_golden.py
It imports the unmodified reference ``ditsim`` (read-only, /root/reference/pkg/src), drives it
through allocator op sequences, greedy / static-DoP simulations and workload generation, and
writes the outcomes as JSON next to this script. tests/test_sched_golden.py replays the same
inputs through paper_2506_13497_b200.sched and requires identical outputs (bit-exact floats
via repr / hex).
"""

from __future__ import annotations

import copy
import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")


def load_ref():
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    import ditsim  # noqa: E402

    return ditsim


# ------------------------------------------------------------------ allocator fuzz
def alloc_ops(ds, nodes, gpn, seed, n_ops):
    """Random op sequence driven through the reference pool; records ops, results, snapshots."""
    rng = random.Random(seed)
    pool = ds.GpuPool(ds.ClusterTopology(nodes, gpn))
    handles: list = []  # live handles (reference objects)
    log = []

    def hid(h):
        return [[b.start, b.order] for b in h.blocks]

    for _ in range(n_ops):
        kind = rng.choice(["allocate", "allocate", "allocate_group", "release", "keep_lowest",
                           "try_best", "try_best_grow", "retract"])
        op = {"op": kind}
        res = None
        if kind == "allocate":
            size = rng.choice([1, 1, 2, 4, 8, 16][: 3 + (gpn >= 8) + (gpn >= 16)])
            size = min(size, gpn)
            op["size"] = size
            h = pool.allocate(size)
            res = None if h is None else hid(h)
            if h is not None:
                handles.append(h)
        elif kind == "allocate_group":
            size = rng.randint(1, gpn)
            op["size"] = size
            h = pool.allocate_group(size)
            res = None if h is None else hid(h)
            if h is not None:
                handles.append(h)
        elif kind == "release" and handles:
            i = rng.randrange(len(handles))
            op["handle"] = hid(handles[i])
            pool.release(handles.pop(i))
        elif kind == "keep_lowest" and handles:
            i = rng.randrange(len(handles))
            h = handles[i]
            keep = rng.choice([k for k in (1, 2, 4, 8) if k <= h.count] or [1])
            try:  # skip calls the reference rejects (it mutates before raising)
                copy.deepcopy(pool).release_keep_lowest(h, keep)
            except ds.AllocationError:
                continue
            op["handle"], op["keep"] = hid(h), keep
            kept, freed = pool.release_keep_lowest(h, keep)
            handles[i] = kept
            res = [hid(kept), list(freed)]
        elif kind == "try_best":
            target = rng.choice([1, 2, 4, 8])
            op["target"] = target
            h = pool.try_best_alloc(target, None, (1, 2, 4, 8))
            res = None if h is None else hid(h)
            if h is not None:
                handles.append(h)
        elif kind == "try_best_grow" and handles:
            singles = [i for i, h in enumerate(handles) if len(h.blocks) == 1]
            if not singles:
                continue
            i = rng.choice(singles)
            h = handles[i]
            target = rng.choice([1, 2, 4, 8])
            op["handle"], op["target"] = hid(h), target
            g = pool.try_best_alloc(target, h, (1, 2, 4, 8))
            res = {"same": g is h, "handle": hid(g)}
            handles[i] = g
        elif kind == "retract" and handles:
            cands = [i for i, h in enumerate(handles) if len(h.blocks) == 1 and h.count > 1]
            if not cands:
                continue
            i = rng.choice(cands)
            h = handles[i]
            b = h.blocks[0]
            sub_order = rng.randrange(b.order)
            sub_start = b.start + rng.randrange(1 << (b.order - sub_order)) * (1 << sub_order)
            sub = ds.AllocationHandle((ds.Block(sub_start, sub_order),))
            op["handle"], op["sub"] = hid(h), hid(sub)
            res = list(pool.retract_to(h, sub))
            handles[i] = sub
        else:
            continue
        op["result"] = res
        op["snapshot"] = pool.snapshot()
        log.append(op)
    return log


# ------------------------------------------------------------------ simulations
def f2s(x):
    return float(x).hex()


def sim_record(ds, topo, profile, dop_table, workload, policy, overheads=None):
    kw = {} if overheads is None else {"overheads": overheads}
    res = ds.Simulation(topo, profile, dop_table, workload, policy, **kw).run()
    m = ds.compute_metrics(res)
    trace = "".join(r.to_json_line() + "\n" for r in res.trace)
    out = {
        "policy": res.policy_name,
        "occupancy": f2s(res.cumulative_occupancy),
        "avg": f2s(m.avg_latency),
        "p99": f2s(m.p99_latency),
        "trace_sha256": hashlib.sha256(trace.encode()).hexdigest(),
        "trace_len": len(res.trace),
        "requests": [[r.request_id, r.resolution, f2s(r.arrival), f2s(r.start), f2s(r.finish),
                      f2s(r.gpu_seconds), [[f2s(t), w] for t, w in r.dop_history]]
                     for r in res.requests],
    }
    if len(res.trace) <= 400:
        out["trace"] = trace
    return out


def random_profile_doc(seed, res_names=("144p", "240p", "360p", "480p")):
    rng = random.Random(seed)
    entries = []
    for name in res_names:
        base = rng.uniform(0.1, 2.0)
        t = base
        for i, d in enumerate((1, 2, 4, 8)):
            if i:
                t = t * rng.uniform(0.45, 1.05)
            e = {"resolution": name, "dop": d, "dit_step_seconds": t}
            if d == 1:
                e["vae_seconds"] = rng.uniform(0.1, 3.0)
            entries.append(e)
    return {"schema": "dit-profile/1", "dop_candidates": [1, 2, 4, 8], "entries": entries}


def main():
    ds = load_ref()
    out: dict = {"reference": str(REF), "generator": "tests/golden/make_sched_golden.py"}
    prof = ds.default_profile()
    default_doc = {"schema": "dit-profile/1", "dop_candidates": list(prof.dop_candidates),
                   "entries": []}
    for r in prof.resolutions:
        for d in prof.profiled_dops(r.name):
            e = {"resolution": r.name, "dop": d, "dit_step_seconds": prof.dit_step(r.name, d)}
            if d == 1:
                e["vae_seconds"] = prof.vae(r.name, 1)
            default_doc["entries"].append(e)
    out["default_profile"] = default_doc
    # profiles: B values and change rates
    pcases = []
    for doc_seed, doc in [("default", default_doc)] + [(s, random_profile_doc(s)) for s in range(6)]:
        t = ds.load_profiles(doc)
        case = {"seed": doc_seed, "doc": doc, "optimal": {}, "change": {}}
        for thr in (0.0, 0.05, 0.2):
            case["optimal"][str(thr)] = {r.name: ds.optimal_dop(t, r.name, thr) for r in t.resolutions}
        for r in t.resolutions:
            case["change"][r.name] = [f2s(ds.change_rate(t, r.name, d)) for d in (2, 4, 8)]
        pcases.append(case)
    out["profiles"] = pcases
    # allocator fuzz
    out["alloc"] = [{"nodes": n, "gpn": g, "seed": s, "log": alloc_ops(ds, n, g, s, 300)}
                    for (n, g) in ((1, 8), (2, 4), (2, 8), (1, 16)) for s in range(3)]
    # workloads
    wl = []
    for spec in [dict(proportions={"144p": 1 / 3, "240p": 1 / 3, "360p": 1 / 3}, total_requests=48,
                      arrival_rate=0.5, seed=0),
                 dict(proportions={"144p": 0.5, "360p": 0.25, "240p": 0.25}, total_requests=37,
                      arrival_rate=1.7, seed=11),
                 dict(proportions={"240p": 0.2, "144p": 0.8}, total_requests=10, burst=True, seed=3)]:
        recs = ds.generate(ds.WorkloadSpec(**spec))
        wl.append({"spec": spec, "records": [[r.request_id, f2s(r.arrival_time), r.resolution,
                                              r.denoise_steps] for r in recs]})
    out["workloads"] = wl
    # simulations
    sims = []
    mix = {"144p": 1 / 3, "240p": 1 / 3, "360p": 1 / 3}
    for doc_name, doc in [("default", default_doc), ("rand1", random_profile_doc(1)),
                          ("rand4", random_profile_doc(4))]:
        t = ds.load_profiles(doc)
        names = [r.name for r in t.resolutions][:3]
        mixd = {n: 1 / len(names) for n in names}
        for topo in ((1, 8), (2, 8)):
            for wspec in [dict(total_requests=48, arrival_rate=0.5, seed=0),
                          dict(total_requests=48, burst=True, seed=0),
                          dict(total_requests=60, arrival_rate=2.0, seed=5)]:
                recs = ds.generate(ds.WorkloadSpec(proportions=mixd, **wspec))
                for vae_dop in (1, 2):
                    dt = ds.derive_dop_table(t, vae_dop=vae_dop)
                    pols = [("greedy", lambda: ds.GreedyPolicy(dt)),
                            ("greedy-nopromo", lambda: ds.GreedyPolicy(dt, promotion=False))]
                    if vae_dop == 1:
                        pols += [(f"sdop{d}", (lambda d=d: ds.StaticDopPolicy(d))) for d in (1, 2, 4)]
                        pols += [("sdop4-dec", lambda: ds.StaticDopPolicy(4, decouple_vae=True))]
                    for pname, mk in pols:
                        rec = sim_record(ds, ds.ClusterTopology(*topo), t, dt, recs, mk())
                        rec.update({"profile": doc_name, "topology": list(topo), "workload": wspec,
                                    "mix": mixd, "vae_dop": vae_dop, "policy_key": pname})
                        sims.append(rec)
    out["sims"] = sims
    data = json.dumps(out, separators=(",", ":")).encode()
    (HERE / "sched_golden.json.gz").write_bytes(gzip.compress(data, mtime=0))
    print(f"wrote {HERE / 'sched_golden.json.gz'}: {len(out['alloc'])} alloc logs, {len(sims)} sims")


if __name__ == "__main__":
    main()
