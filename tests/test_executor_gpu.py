"""The reference serving loop semantics driving real B200 steps: greedy allocator decisions with
promotions (re-shard P -> P' at step boundaries) and the DiT -> VAE latent hand-off. The final
latent of every request must equal running the same steps at DoP 1 (sharding, exchange and
re-shards are numerically invisible)."""
import dataclasses

import pytest
import torch

pytestmark = pytest.mark.gpu


def _profile_doc():
    # synthetic times shaped so 144p-16f wants DoP 2 and 240p-like wants 4 (promotions happen)
    return {"schema": "dit-profile/1", "dop_candidates": [1, 2, 4], "entries": [
        {"resolution": "144p-16f", "dop": 1, "dit_step_seconds": 0.5, "vae_seconds": 0.2},
        {"resolution": "144p-16f", "dop": 2, "dit_step_seconds": 0.25},
        {"resolution": "144p-16f", "dop": 4, "dit_step_seconds": 0.24},
        {"resolution": "144p", "dop": 1, "dit_step_seconds": 0.8, "vae_seconds": 0.3},
        {"resolution": "144p", "dop": 2, "dit_step_seconds": 0.4},
        {"resolution": "144p", "dop": 4, "dit_step_seconds": 0.15},
    ]}


def test_engine_drives_real_steps_with_promotions(cuda):
    from paper_2506_13497_b200 import sched, shapes, weights
    from paper_2506_13497_b200.executor import B200Executor
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    steps = 8
    ex = B200Executor(cfg, W, num_steps=steps)
    t = sched.load_profiles(_profile_doc())
    dt = sched.derive_dop_table(t)
    assert dt.by_resolution == {"144p-16f": 2, "144p": 4}
    # request 0 takes GPUs (0,1); request 1 starts hungry on (2,3) and is promoted to 4 GPUs
    # once request 0's short DiT and VAE release (0,1)
    wl = [sched.ArrivalRecord(0, 0.0, "144p-16f", 2), sched.ArrivalRecord(1, 0.0, "144p", steps),
          sched.ArrivalRecord(2, 0.0, "144p-16f", 3), sched.ArrivalRecord(3, 0.0, "144p", 5)]
    sim = sched.Simulation(sched.ClusterTopology(1, 4), t, dt, wl, sched.GreedyPolicy(dt), executor=ex)
    res = sim.run()
    kinds = [r.kind for r in res.trace]
    assert kinds.count("vae_complete") == 4
    assert "promotion" in kinds, "scenario must exercise a promotion"
    assert len(ex.final_latents) == 4
    # every request's final latent == the same steps at DoP 1
    model = STDiTModel(cfg, W, cuda)
    for rec in wl:
        sh = shapes.shape_of(rec.resolution)
        z, y = weights.synthetic_inputs(cfg, sh.latent, seed_z=2 * rec.request_id, seed_y=2 * rec.request_id + 1)
        req = StepRequest(model, sh, y.to(cuda), num_steps=steps)
        zd = z.to(cuda).contiguous()
        for i in range(rec.denoise_steps):
            req.step(zd, i)
        torch.cuda.synchronize()
        assert torch.equal(ex.final_latents[rec.request_id], zd), rec.request_id


def test_latent_gather_regroups_shards(cuda):
    from paper_2506_13497_b200.executor import latent_gather
    from paper_2506_13497_b200 import shapes

    T = 15
    z = torch.randn(1, 4, T, 18, 32, device=cuda)
    for P, Q in [(1, 2), (2, 4), (4, 8), (2, 1), (8, 1), (1, 8)]:
        src = []
        for r in range(P):
            lo, hi = shapes.shard_range(T, P, r)
            src.append((z[:, :, lo:hi].contiguous(), lo, hi))
        for q in range(Q):
            lo, hi = shapes.shard_range(T, Q, q)
            d = torch.empty(1, 4, hi - lo, 18, 32, device=cuda)
            latent_gather(d, lo, hi, src)
            torch.cuda.synchronize()
            assert torch.equal(d, z[:, :, lo:hi])


def test_profile_b200_emits_loadable_document(cuda):
    from paper_2506_13497_b200 import sched, weights
    from paper_2506_13497_b200.executor import profile_b200

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    doc = profile_b200(cfg, W, ["144p-16f"], dops=(1, 2), repeats=2, vae_seconds={"144p-16f": 0.1})
    t = sched.load_profiles(doc)
    assert t.dit_step("144p-16f", 1) > 0 and t.dit_step("144p-16f", 2) > 0


def test_engine_with_vae_decode(cuda):
    """Decoupled DiT -> VAE through the engine: the retained master GPU decodes the gathered
    latent; the video equals decoding the DoP-1 latent."""
    from paper_2506_13497_b200 import sched, shapes, weights, vae_weights as vw
    from paper_2506_13497_b200.executor import B200Executor
    from paper_2506_13497_b200.vae import VAEDecoder

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    VW = vw.init_vae_weights(vw.TINY_VAE)
    ex = B200Executor(cfg, W, num_steps=3, vae_cfg=vw.TINY_VAE, vae_weights=VW, keep_videos=True)
    t = sched.load_profiles(_profile_doc())
    dt = sched.derive_dop_table(t)
    wl = [sched.ArrivalRecord(0, 0.0, "144p-16f", 3)]
    res = sched.Simulation(sched.ClusterTopology(1, 4), t, dt, wl, sched.GreedyPolicy(dt), executor=ex).run()
    assert [r.kind for r in res.trace][-1] == "vae_complete"
    sh = shapes.shape_of("144p-16f")
    video = ex.videos[0]
    assert video.shape == (1, 3, sh.frames, sh.height, sh.width)
    ref = VAEDecoder(vw.TINY_VAE, VW, cuda).decode(ex.final_latents[0], sh.frames, sh.height, sh.width)
    torch.cuda.synchronize()
    assert torch.equal(video, ref)
    assert ex.vae_seconds[0][2] > 0


@pytest.mark.parametrize("vae_dop", [2, 4])
def test_vae_dop_splits_micro_batches(cuda, vae_dop):
    """VAE DoP q: each rank's frame block (temporal micro-batches it overlaps, spatial decode of
    its own frames) concatenates to the DoP-1 video exactly."""
    from paper_2506_13497_b200 import vae_weights as vw
    from paper_2506_13497_b200.vae import VAEDecoder, vae_shard

    cfg = vw.TINY_VAE
    W = vw.init_vae_weights(cfg)
    T, frames, h, w = 15, 51, 4, 6
    z = torch.randn(1, 4, T, h, w, generator=torch.Generator().manual_seed(3)).to(cuda)
    dec = VAEDecoder(cfg, W, cuda)
    full = dec.decode(z, frames, 8 * h, 8 * w)
    parts = []
    for r in range(vae_dop):
        t_lo, t_hi, f_lo, f_hi = vae_shard(cfg, T, frames, vae_dop, r)
        if f_hi > f_lo:
            f0 = t_lo // cfg.micro_z * cfg.micro_frame_size
            nf = min(-(-(t_hi - t_lo) // cfg.micro_z) * cfg.micro_frame_size, frames - f0)
            parts.append(dec.decode(z[:, :, t_lo:t_hi].contiguous(), nf, 8 * h, 8 * w,
                                    frames=(f_lo - f0, f_hi - f0)))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, dim=2), full)


def test_engine_with_vae_dop2(cuda, tmp_path):
    """Decoupled DiT(DoP 4) -> VAE(DoP 2) (BASELINE config 4): the policy keeps the two lowest
    GPUs, each decodes its micro-batches; the video equals decoding the DoP-1 latent. The hand-off
    is also spilled in the on-disk latent format and reads back exactly."""
    from paper_2506_13497_b200 import sched, shapes, weights, vae_weights as vw
    from paper_2506_13497_b200.executor import B200Executor
    from paper_2506_13497_b200.vae import VAEDecoder

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    VW = vw.init_vae_weights(vw.TINY_VAE)
    ex = B200Executor(cfg, W, num_steps=2, vae_cfg=vw.TINY_VAE, vae_weights=VW, keep_videos=True,
                      latent_dir=str(tmp_path))
    t = sched.load_profiles(_profile_doc())
    dt = sched.derive_dop_table(t, vae_dop=2)
    wl = [sched.ArrivalRecord(0, 0.0, "144p", 2)]  # 144p x 51 frames: 3 micro-batches
    res = sched.Simulation(sched.ClusterTopology(1, 4), t, dt, wl, sched.GreedyPolicy(dt), executor=ex).run()
    dc = [r for r in res.trace if r.kind == "dit_complete"][0]
    assert dc.gpu_ids == (0, 1)  # retained: the two lowest of the DiT group (0..3)
    sh = shapes.shape_of("144p")
    ref = VAEDecoder(vw.TINY_VAE, VW, cuda).decode(ex.final_latents[0], sh.frames, sh.height, sh.width)
    torch.cuda.synchronize()
    assert torch.equal(ex.videos[0], ref)
    from paper_2506_13497_b200.latent_io import load_latent

    z, frames, hdr = load_latent(tmp_path / "req0.ddlat")
    assert torch.equal(z, ex.final_latents[0].cpu()) and torch.equal(frames, ex.videos[0].cpu())
    assert hdr["dit_gpu_ids"] == [0, 1, 2, 3] and hdr["vae_gpu_ids"] == [0, 1]


def test_wall_clock_engine_runs_groups_concurrently(cuda):
    """§8(f)1: the serving loop on wall-clock time -- steps, re-shards and the async DiT->VAE
    hand-off enqueued on per-group streams, STEP_COMPLETE / VAE_COMPLETE taken from CUDA events.
    Every request finishes, promotions happen, and each final latent equals the same steps at
    DoP 1 bit for bit (concurrency and async hand-off are numerically invisible)."""
    from paper_2506_13497_b200 import sched, shapes, weights
    from paper_2506_13497_b200.serving import AsyncB200Executor, WallClockSimulation
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W = weights.init_weights(cfg, seed=3)
    steps = 8
    ex = AsyncB200Executor(cfg, W, num_steps=steps)
    t = sched.load_profiles(_profile_doc())
    dt = sched.derive_dop_table(t)
    wl = [sched.ArrivalRecord(0, 0.0, "144p-16f", 2), sched.ArrivalRecord(1, 0.0, "144p", steps),
          sched.ArrivalRecord(2, 0.001, "144p-16f", 3), sched.ArrivalRecord(3, 0.002, "144p", 5),
          sched.ArrivalRecord(4, 0.05, "144p-16f", 4)]
    sim = WallClockSimulation(sched.ClusterTopology(1, 4), t, dt, wl, sched.GreedyPolicy(dt), ex)
    res = sim.run()
    kinds = [r.kind for r in res.trace]
    assert kinds.count("vae_complete") == len(wl)
    times = [r.time for r in res.trace]
    assert times == sorted(times)
    m = sched.compute_metrics(res)
    print(f"wall-clock engine: avg {m.avg_latency * 1e3:.2f} ms p99 {m.p99_latency * 1e3:.2f} ms, "
          f"{len(sim.device_seconds)} device completions, promotions {kinds.count('promotion')}")
    model = STDiTModel(cfg, W, cuda)
    torch.cuda.synchronize()
    for rec in wl:
        sh = shapes.shape_of(rec.resolution)
        z, y = weights.synthetic_inputs(cfg, sh.latent, seed_z=2 * rec.request_id, seed_y=2 * rec.request_id + 1)
        req = StepRequest(model, sh, y.to(cuda), num_steps=steps)
        zd = z.to(cuda).contiguous()
        for i in range(rec.denoise_steps):
            req.step(zd, i)
        torch.cuda.synchronize()
        assert torch.equal(ex.final_latents[rec.request_id], zd), rec.request_id
    ex.close()
