"""Parity at the configurations the bench and BASELINE.json quote:
the benchmarked step itself (STDiT3-XL/2, 28 block pairs, 240p x 51) against the fp32 CPU oracle,
the long-sequence regime (720p x 102: S = 3600 tokens per frame, T = 30) at XL/2 width, the
XL/2-width DoP 2/4/8 groups bit for bit against DoP 1, and a 10-step XL/2 trajectory.

Tolerance (north_star): bf16 compute vs the fp32 oracle, relative L2 <= 1e-2 on the denoised
latent z' of every step; the update v*dt itself <= 2e-2. DoP-P vs DoP 1: bit-exact.
"""
import dataclasses

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return (torch.linalg.vector_norm(a.float() - b.float()) / torch.linalg.vector_norm(b.float())).item()


def _setup(cfg, label, seed=3):
    from paper_2506_13497_b200 import shapes, weights

    W = weights.init_weights(cfg, seed=seed)
    sh = shapes.shape_of(label)
    z, y = weights.synthetic_inputs(cfg, sh.latent)
    return W, sh, z, y


def _oracle_step(cfg, W, sh, z, text, step):
    import os

    from oracle import stdit3  # the checker

    torch.set_num_threads(os.cpu_count() or 1)
    with torch.inference_mode():
        return stdit3.denoise_step(W, cfg, z, text, step, sh.height, sh.width)


def _text(W, y):
    from oracle import stdit3

    with torch.inference_mode():
        return stdit3.prepare_text(W, y)


@pytest.fixture(scope="module")
def xl2_240p(cuda):
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel

    cfg = weights.XL2
    W, sh, z, y = _setup(cfg, "240p")
    model = STDiTModel(cfg, W, cuda)
    return cfg, W, sh, z, y, model


def test_bench_config_step_matches_oracle(xl2_240p, cuda):
    """bench.py's workload exactly: XL/2 (28 block pairs, C = 1152), 240p x 51 (latent
    15 x 30 x 54, 6075 tokens per sample), CFG batch 2, one RFLOW step, DoP 1."""
    from paper_2506_13497_b200.stdit import StepRequest

    cfg, W, sh, z, y, model = xl2_240p
    step = 3
    req = StepRequest(model, sh, y.to(cuda))
    zd = z.to(cuda).contiguous()
    req.graph_step(zd, step)  # the bench replays the step from a CUDA graph
    torch.cuda.synchronize()
    out = zd.cpu()
    req.close()
    ref = _oracle_step(cfg, W, sh, z, _text(W, y), step)
    e_z, e_v = rel_l2(out, ref), rel_l2(out - z, ref - z)
    print(f"XL/2 28L 240p x51 step {step}: relL2 z'={e_z:.2e} update={e_v:.2e}")
    assert e_z <= 1e-2 and e_v <= 2e-2


@pytest.mark.parametrize("fused", [1, 0], ids=["fused-xch", "xch-kernel"])
@pytest.mark.parametrize("dop", [2, 4, 8])
def test_bench_config_dop_matches_dop1_bitexact(xl2_240p, cuda, dop, fused):
    """The same 28-layer XL/2 240p step split over a DoP 2/4/8 group (virtual ranks on one
    device: T-shards 8/7, 4/4/4/3, 2x7+1; S-shards of 405 tokens ragged at every P) gives
    DoP 1's latent bit for bit, with the exchange fused into fc2 or as the separate kernel."""
    from paper_2506_13497_b200 import _lib
    from paper_2506_13497_b200.stdit import StepRequest, VirtualGroup

    cfg, W, sh, z, y, model = xl2_240p
    yd = y.to(cuda)
    z1 = z.to(cuda).contiguous()
    r1 = StepRequest(model, sh, yd)
    r1.step(z1, 7)
    _lib.lib().ddit_set_fused_exchange(fused)
    try:
        grp = VirtualGroup(model, sh, yd, dop)
    finally:
        _lib.lib().ddit_set_fused_exchange(1)
    parts = grp.split(z.to(cuda))
    grp.step(parts, 7)
    zp = torch.cat(parts, dim=2)
    torch.cuda.synchronize()
    diff = (zp - z1).abs().max().item()
    print(f"XL/2 28L 240p DoP {dop} ({'fused' if fused else 'kernel'} exchange): max |diff| {diff}")
    assert torch.equal(zp, z1)
    for r in grp.ranks:
        r.close()
    r1.close()


def test_long_sequence_720p_step_matches_oracle(cuda):
    """BASELINE config 3's regime at XL/2 width: 720p x 102 (latent 30 x 90 x 160, S = 3600
    tokens per frame, T = 30 frames, 108 000 tokens per sample), one block pair."""
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.XL2, depth=1)
    W, sh, z, y = _setup(cfg, "720p-102f")
    assert (sh.S, sh.T) == (3600, 30)
    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    zd = z.to(cuda).contiguous()
    req.step(zd, 5)
    torch.cuda.synchronize()
    out = zd.cpu()
    req.close()
    model.close()
    ref = _oracle_step(cfg, W, sh, z, _text(W, y), 5)
    e_z, e_v = rel_l2(out, ref), rel_l2(out - z, ref - z)
    print(f"XL/2-width 720p x102 (S=3600, T=30) depth 1: relL2 z'={e_z:.2e} update={e_v:.2e}")
    assert e_z <= 1e-2 and e_v <= 2e-2


def test_xl2_ten_step_trajectory_matches_oracle(cuda):
    """Ten consecutive RFLOW steps of the real model (XL/2, 28 block pairs) at 144p x 51 on the
    GPU against the oracle chained on its own output: the error stays per-step sized."""
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = weights.XL2
    W, sh, z, y = _setup(cfg, "144p")
    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    text = _text(W, y)
    zd = z.to(cuda).contiguous()
    zr = z.clone()
    errs = []
    for step in range(10):
        req.step(zd, step)
        zr = _oracle_step(cfg, W, sh, zr, text, step)
        torch.cuda.synchronize()
        errs.append(rel_l2(zd.cpu(), zr))
    req.close()
    model.close()
    print("XL/2 28L 144p x51 trajectory relL2 per step:", " ".join(f"{e:.2e}" for e in errs))
    assert max(errs) <= 1e-2
