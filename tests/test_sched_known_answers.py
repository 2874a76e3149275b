"""Known-answer vectors the reference's own tests pin, restated against the
B200 framework's scheduler, plus a live differential fuzz vs the reference when it is
importable (build container only)."""
import random
import sys
from pathlib import Path

import pytest

from paper_2506_13497_b200 import sched
from paper_2506_13497_b200.sched import AllocationHandle, Block, ClusterTopology, GpuPool


def pool8():
    return GpuPool(ClusterTopology(1, 8))


def test_empty_pool_allocate_pair():  # reference tests/test_allocator.py:19-22
    assert pool8().allocate(2).gpu_ids == (0, 1)


def test_split_and_alignment():  # :24-40
    p = pool8()
    assert p.allocate(4).gpu_ids == (0, 1, 2, 3)
    assert p.allocate(4).gpu_ids == (4, 5, 6, 7)
    assert p.allocate(1) is None


def test_failure_leaves_pool_unchanged():  # :42-47
    p = pool8()
    p.allocate(8)
    before = p.snapshot()
    assert p.allocate(2) is None
    assert p.snapshot() == before


def test_coalesce_to_one_block():  # :69-76
    p = GpuPool(ClusterTopology(1, 4))
    hs = [p.allocate(1) for _ in range(4)]
    for hd in hs:
        p.release(hd)
    assert p.snapshot()["free_blocks"] == [{"node": 0, "start": 0, "order": 2}]


def test_lowest_start_not_best_fit():  # SURVEY Appendix A.1 golden vector
    p = pool8()
    a = p.allocate(2)
    p.allocate(1)
    p.release(a)
    assert p.allocate(1).gpu_ids == (0,)


def test_keep_lowest():  # :108-113
    p = pool8()
    hd = p.allocate(4)
    kept, freed = p.release_keep_lowest(hd, 1)
    assert kept.gpu_ids == (0,) and freed == (1, 2, 3)


def test_bandwidth_aware_partition():  # :131-141
    assert sched.bandwidth_aware_partition(ClusterTopology(1, 8), 0, 7, 1) == 7
    assert sched.bandwidth_aware_partition(ClusterTopology(2, 4), 2, 4, 2) == 2


def test_try_best_grow_returns_held_when_blocked():  # :162-181
    p = pool8()
    a = p.allocate(2)
    p.allocate(2)
    assert p.try_best_alloc(4, a) is a


def test_try_best_grow_one_to_four():  # :188-192
    p = pool8()
    a = p.allocate(1)
    g = p.try_best_alloc(4, a)
    assert g.gpu_ids == (0, 1, 2, 3)


def test_retract_frees_the_rest():  # :221-230
    p = pool8()
    big = p.allocate(8)
    freed = p.retract_to(big, AllocationHandle((Block(0, 1),)))
    assert sorted(freed) == [2, 3, 4, 5, 6, 7]


def _default_table():
    import gzip, json
    g = json.loads(gzip.decompress((Path(__file__).parent / "golden" / "sched_golden.json.gz").read_bytes()))
    return sched.load_profiles(g["default_profile"])


def test_demo03_greedy_lifecycle_numbers():
    """Reference demos/03_greedy_lifecycle.py:22-29: hungry 360p request 2 starts on (6,7),
    promoted at 3.28125 to (4,5,6,7), dit_complete at 8.673874999999999 on (4,),
    vae_complete at 9.845749999999999; occupancy 64.22675."""
    t = _default_table()
    dt = sched.derive_dop_table(t)
    wl = [sched.ArrivalRecord(0, 0.0, "360p", 30), sched.ArrivalRecord(1, 0.0, "240p", 10),
          sched.ArrivalRecord(2, 0.0, "360p", 30)]
    res = sched.Simulation(ClusterTopology(1, 8), t, dt, wl, sched.GreedyPolicy(dt)).run()
    ev = [(r.time, r.kind, r.gpu_ids) for r in res.trace if r.request_id == 2]
    assert (0.0, "start", (6, 7)) in ev
    assert (3.28125, "promotion", (4, 5, 6, 7)) in ev
    assert (8.673874999999999, "dit_complete", (4,)) in ev
    assert (9.845749999999999, "vae_complete", (4,)) in ev
    assert res.cumulative_occupancy == 64.22675


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not present (GPU box)")
@pytest.mark.parametrize("seed", range(25))
def test_live_differential_greedy(seed):
    """Random profiles / mixes / loads through both schedulers: identical traces."""
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    import ditsim as ref

    rng = random.Random(1000 + seed)
    names = ["144p", "240p", "360p"]
    entries = []
    for n in names:
        t = rng.uniform(0.1, 1.5)
        for i, d in enumerate((1, 2, 4, 8)):
            t = t * (rng.uniform(0.45, 1.05) if i else 1.0)
            e = {"resolution": n, "dop": d, "dit_step_seconds": t}
            if d == 1:
                e["vae_seconds"] = rng.uniform(0.05, 2.0)
            entries.append(e)
    doc = {"schema": "dit-profile/1", "dop_candidates": [1, 2, 4, 8], "entries": entries}
    w = [rng.random() + 0.05 for _ in names]
    mix = {n: x / sum(w) for n, x in zip(names, w)}
    mix[names[-1]] = 1.0 - sum(mix[n] for n in names[:-1])
    spec = dict(proportions=mix, total_requests=rng.randint(5, 80),
                arrival_rate=rng.uniform(0.2, 4.0), seed=seed, denoise_steps=rng.randint(1, 30))
    topo = rng.choice([(1, 8), (2, 8), (1, 4), (2, 4)])
    vae_dop = rng.choice([1, 2])
    out = []
    for lib in (ref, sched):
        t = lib.load_profiles(doc)
        dt = lib.derive_dop_table(t, vae_dop=vae_dop)
        recs = lib.generate(lib.WorkloadSpec(**spec))
        res = lib.Simulation(lib.ClusterTopology(*topo), t, dt, recs, lib.GreedyPolicy(dt)).run()
        out.append(([r.to_json_line() for r in res.trace], res.cumulative_occupancy))
    assert out[0] == out[1]
