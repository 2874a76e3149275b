"""B200ProfileTable (paper_2506_13497_b200.boundary) inside the UNMODIFIED reference engine:
the duck type must (1) leave every scheduling decision exactly as the virtual-time run on the
same table, (2) call the executor once per denoise step with the right step index, GPU group
and re-shard source, and once per VAE with the DiT and retained groups. CPU: a recording fake
executor stands in for the B200 (tests/test_boundary_gpu.py runs the real one)."""
import pytest

from paper_2506_13497_b200.boundary import B200ProfileTable
from refsim import ditsim


class FakeExecutor:
    def __init__(self):
        self.steps = []
        self.vaes = []

    def dit_step(self, request, gpu_ids, step, resharded_from):
        self.steps.append((request.request_id, tuple(gpu_ids), step, resharded_from))
        return 1e-3

    def vae(self, request, dit_gpu_ids, vae_gpu_ids):
        self.vaes.append((request.request_id, tuple(dit_gpu_ids), tuple(vae_gpu_ids)))
        return 2e-3


def _trace(res):
    return [(r.time, r.kind, r.request_id, r.gpu_ids) for r in res.trace]


@pytest.mark.parametrize("rate", [0.5, 1.0, None])
def test_profiled_mode_keeps_reference_decisions(rate):
    ds = ditsim()
    table = ds.default_profile()
    dt = ds.derive_dop_table(table)
    spec = ds.WorkloadSpec(proportions={"144p": 1 / 3, "240p": 1 / 3, "360p": 1 / 3},
                           total_requests=24, arrival_rate=rate, burst=rate is None, seed=3)
    topo = ds.ClusterTopology(1, 8)
    virt = ds.Simulation(topo, table, dt, ds.generate(spec), ds.GreedyPolicy(dt)).run()
    ex = FakeExecutor()
    bt = B200ProfileTable(table, ex)
    real = ds.Simulation(topo, bt, dt, ds.generate(spec), ds.GreedyPolicy(dt)).run()
    assert _trace(real) == _trace(virt)
    assert ds.compute_metrics(real) == ds.compute_metrics(virt)
    # one executed step per denoise step, indices 0..n-1 in order, on the group the trace shows
    per_req = {}
    for rid, ids, step, src in ex.steps:
        per_req.setdefault(rid, []).append((ids, step, src))
    promos = {(r.request_id, r.gpu_ids) for r in virt.trace if r.kind == "promotion"}
    for rid, calls in per_req.items():
        assert [s for _, s, _ in calls] == list(range(30))
        for (ids, _, src), prev in zip(calls[1:], calls[:-1]):
            if ids != prev[0]:
                assert src == prev[0] and (rid, ids) in promos
            else:
                assert src is None
    assert len(per_req) == 24 and len(ex.vaes) == 24
    for rid, dit_ids, vae_ids in ex.vaes:
        assert dit_ids == per_req[rid][-1][0]
        assert set(vae_ids) <= set(dit_ids) and vae_ids == tuple(sorted(dit_ids))[:len(vae_ids)]
    kinds = {e.kind for e in bt.executed}
    assert {"start", "step", "vae"} <= kinds


def test_measured_mode_charges_executor_seconds():
    ds = ditsim()
    table = ds.default_profile()
    dt = ds.derive_dop_table(table)
    wl = [ds.ArrivalRecord(0, 0.0, "240p", 4)]
    ex = FakeExecutor()
    res = ds.Simulation(ds.ClusterTopology(1, 8), B200ProfileTable(table, ex, mode="measured"), dt,
                        wl, ds.GreedyPolicy(dt)).run()
    done = [r.time for r in res.trace if r.kind == "vae_complete"]
    assert done == [pytest.approx(4 * 1e-3 + 2e-3)]


def test_lookup_errors_pass_through():
    ds = ditsim()
    bt = B200ProfileTable(ds.default_profile(), FakeExecutor())
    with pytest.raises(ds.ProfileLookupError):
        bt.dit_step("720p", 1)
    with pytest.raises(ds.ProfileLookupError):
        bt.vae("240p", 3)
    assert bt.dit_step("240p", 2) == 0.25  # a plain lookup runs nothing
    assert bt.profiled_dops("240p") == (1, 2, 4, 8) and bt.has_resolution("360p")
