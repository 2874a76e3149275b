"""The UNMODIFIED reference serving loop (ditsim.Simulation + GreedyPolicy, imported from the
baseline/_ref install) driving real B200 steps through B200ProfileTable, the reference's own
ProfileTable duck type (profiles.py:48-90): allocator decisions equal the virtual-time run,
every step / re-shard / VAE decode actually runs on the GPU, and each request's final latent
equals the same steps at DoP 1."""
import dataclasses

import pytest
import torch

from refsim import ditsim

pytestmark = pytest.mark.gpu


def _doc():
    return {"schema": "dit-profile/1", "dop_candidates": [1, 2, 4], "entries": [
        {"resolution": "144p-16f", "dop": 1, "dit_step_seconds": 0.5, "vae_seconds": 0.2},
        {"resolution": "144p-16f", "dop": 2, "dit_step_seconds": 0.25},
        {"resolution": "144p-16f", "dop": 4, "dit_step_seconds": 0.24},
        {"resolution": "144p", "dop": 1, "dit_step_seconds": 0.8, "vae_seconds": 0.3},
        {"resolution": "144p", "dop": 2, "dit_step_seconds": 0.4},
        {"resolution": "144p", "dop": 4, "dit_step_seconds": 0.15},
    ]}


def test_reference_engine_runs_real_steps(cuda):
    ds = ditsim()
    from paper_2506_13497_b200 import shapes, weights
    from paper_2506_13497_b200.boundary import B200ProfileTable
    from paper_2506_13497_b200.executor import B200Executor
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    steps = 8
    table = ds.load_profiles(_doc())
    dt = ds.derive_dop_table(table)
    wl = [ds.ArrivalRecord(0, 0.0, "144p-16f", 2), ds.ArrivalRecord(1, 0.0, "144p", steps),
          ds.ArrivalRecord(2, 0.0, "144p-16f", 3), ds.ArrivalRecord(3, 0.0, "144p", 5)]
    topo = ds.ClusterTopology(1, 4)
    virt = ds.Simulation(topo, table, dt, wl, ds.GreedyPolicy(dt)).run()
    ex = B200Executor(cfg, W, num_steps=steps)
    bt = B200ProfileTable(table, ex)
    res = ds.Simulation(topo, bt, dt, wl, ds.GreedyPolicy(dt)).run()
    assert [(r.time, r.kind, r.request_id, r.gpu_ids) for r in res.trace] == \
        [(r.time, r.kind, r.request_id, r.gpu_ids) for r in virt.trace]
    kinds = [e.kind for e in bt.executed]
    assert kinds.count("vae") == 4 and "promotion" in kinds
    assert sum(1 for k in kinds if k != "vae") == sum(r.denoise_steps for r in wl)
    meas = bt.measured_seconds()
    print("measured device seconds behind the reference engine:",
          {k: round(v, 5) for k, v in meas.items()})
    assert all(e.measured_seconds > 0 for e in bt.executed)
    model = STDiTModel(cfg, W, cuda)
    for rec in wl:
        sh = shapes.shape_of(rec.resolution)
        z, y = weights.synthetic_inputs(cfg, sh.latent, seed_z=2 * rec.request_id,
                                        seed_y=2 * rec.request_id + 1)
        req = StepRequest(model, sh, y.to(cuda), num_steps=steps)
        zd = z.to(cuda).contiguous()
        for i in range(rec.denoise_steps):
            req.step(zd, i)
        torch.cuda.synchronize()
        assert torch.equal(ex.final_latents[rec.request_id], zd), rec.request_id
    ex.close()
