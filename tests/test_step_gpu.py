"""The full STDiT3 denoise step on the B200 (libddit) vs the fp32 CPU oracle.

Tolerance (north_star): bf16 compute vs the fp32 reference, relative L2 <= 1e-2 per step on
the denoised latent z'; the update v*dt itself (the part the step computes) is held to
<= 2e-2 relative L2.
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


def _oracle(cfg, W, sh, z, y, step):
    from oracle import stdit3

    return stdit3.denoise_step(W, cfg, z, stdit3.prepare_text(W, y), step, sh.height, sh.width)


def _gpu(cfg, W, sh, z, y, step, cuda):
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    zd = z.to(cuda).contiguous()
    req.step(zd, step)
    torch.cuda.synchronize()
    return zd.cpu()


@pytest.mark.parametrize("step", [0, 17, 29])
def test_tiny_step_matches_oracle(cuda, step):
    from paper_2506_13497_b200 import weights

    cfg = weights.TINY
    W, sh, z, y = _setup(cfg, "144p-16f")
    ref = _oracle(cfg, W, sh, z, y, step)
    out = _gpu(cfg, W, sh, z, y, step, cuda)
    e_z, e_v = rel_l2(out, ref), rel_l2(out - z, ref - z)
    print(f"tiny step {step}: relL2 z'={e_z:.2e} update={e_v:.2e}")
    assert e_z <= 1e-2 and e_v <= 2e-2


@pytest.mark.parametrize("label", ["240p", "144p"])
def test_xl2_width_step_matches_oracle(cuda, label):
    """Full XL/2 width (C=1152, 16 heads) at the real token counts, depth reduced to 1 block
    pair so the CPU oracle stays within seconds."""
    from paper_2506_13497_b200 import weights

    cfg = dataclasses.replace(weights.XL2, depth=1)
    W, sh, z, y = _setup(cfg, label)
    ref = _oracle(cfg, W, sh, z, y, 3)
    out = _gpu(cfg, W, sh, z, y, 3, cuda)
    e_z, e_v = rel_l2(out, ref), rel_l2(out - z, ref - z)
    print(f"xl2-depth1 {label}: relL2 z'={e_z:.2e} update={e_v:.2e}")
    assert e_z <= 1e-2 and e_v <= 2e-2


@pytest.mark.parametrize("fused", [1, 0], ids=["fused-xch", "xch-kernel"])
@pytest.mark.parametrize("label", ["144p", "240p", "144p-16f"])
@pytest.mark.parametrize("dop", [2, 4, 8])
def test_virtual_dop_matches_dop1(cuda, dop, label, fused):
    """DoP-P shards + exchange (virtual ranks on one device) reproduce the DoP-1 step, with the
    exchange fused into the fc2 GEMM epilogue (peer stores) or as the separate kernel.
    144p: T=15 (ragged T shards), S=144; 240p: S=405 (ragged S shards at every P);
    144p-16f: T=4, so at P=8 ranks 4..7 own no frames (no spatial-phase GEMM: they signal through
    the stand-alone exchange kernel)."""
    from paper_2506_13497_b200 import _lib, weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest, VirtualGroup

    cfg = dataclasses.replace(weights.TINY, depth=2)
    W, sh, z, y = _setup(cfg, label)
    model = STDiTModel(cfg, W, cuda)
    yd = y.to(cuda)
    z1 = z.to(cuda).contiguous()
    StepRequest(model, sh, yd).step(z1, 5)
    _lib.lib().ddit_set_fused_exchange(fused)
    try:
        grp = VirtualGroup(model, sh, yd, dop)
    finally:
        _lib.lib().ddit_set_fused_exchange(1)
    parts = grp.split(z.to(cuda))
    grp.step(parts, 5)
    zp = torch.cat(parts, dim=2)
    torch.cuda.synchronize()
    assert torch.equal(zp, z1), f"max diff {(zp - z1).abs().max().item()}"


@pytest.mark.parametrize("step", [0, 17, 29])
def test_tiny_step_matches_golden_fixture(cuda, step):
    """Against the committed oracle vectors (tests/golden/stdit_tiny_golden.pt) -- no oracle
    run needed on the GPU box."""
    from pathlib import Path

    from paper_2506_13497_b200 import shapes, weights

    g = torch.load(Path(__file__).parent / "golden" / "stdit_tiny_golden.pt")
    cfg = weights.TINY
    W = weights.init_weights(cfg, seed=3)
    sh = shapes.shape_of("144p-16f")
    z, y = weights.synthetic_inputs(cfg, sh.latent)
    assert torch.equal(z, g["z"])
    out = _gpu(cfg, W, sh, z, y, step, cuda)
    ref = g[f"z_{step}"]
    assert rel_l2(out, ref) <= 1e-2 and rel_l2(out - z, ref - z) <= 2e-2


def test_step_has_one_attention_path(cuda):
    """Spatial / cross attention always run the tcgen05 FMHA: the retired option that selected
    the mma.sync flash kernel is refused (no silent second backend on the step path)."""
    from paper_2506_13497_b200._lib import DditError
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.XL2, depth=1)
    W, sh, z, y = _setup(cfg, "240p")
    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    with pytest.raises(DditError):
        req.set_option(1, 0)
    req.set_option(1, 1)  # accepted (the only path)
    zd = z.to(cuda).contiguous()
    req.step(zd, 3)
    torch.cuda.synchronize()
    assert torch.isfinite(zd).all()
    req.close()
    model.close()


def test_graph_replay_matches_eager(cuda):
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = weights.TINY
    W, sh, z, y = _setup(cfg, "144p-16f")
    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    z1 = z.to(cuda).contiguous()
    z2 = z.to(cuda).contiguous()
    for step in (0, 1, 2):
        req.step(z1, step)
        req.graph_step(z2, step)
    torch.cuda.synchronize()
    assert torch.equal(z1, z2)


def test_tiny_full_trajectory_matches_oracle(cuda):
    """All 30 RFLOW steps (the whole denoising trajectory) of the tiny config on the GPU vs the
    fp32 CPU oracle from the same z0: bf16 errors must not compound over the trajectory."""
    from oracle import stdit3
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W, sh, z, y = _setup(cfg, "144p-16f")
    text = stdit3.prepare_text(W, y)
    model = STDiTModel(cfg, W, cuda)
    req = StepRequest(model, sh, y.to(cuda))
    zd = z.to(cuda).contiguous()
    zr = z.clone()
    errs = []
    for step in range(30):
        req.step(zd, step)
        zr = stdit3.denoise_step(W, cfg, zr, text, step, sh.height, sh.width)
        torch.cuda.synchronize()
        errs.append(rel_l2(zd.cpu(), zr))
    print("trajectory relL2 every 5 steps:", [f"{e:.1e}" for e in errs[::5]], f"final {errs[-1]:.2e}")
    assert max(errs) <= 2e-2


def test_xl2_full_depth_step_matches_oracle(cuda):
    """The real model (STDiT3-XL/2, all 28 block pairs, C = 1152) at a real shape (144p x 51:
    latent 15x18x32, 2160 tokens per sample) against the fp32 oracle, one step."""
    from paper_2506_13497_b200 import weights

    cfg = weights.XL2
    W, sh, z, y = _setup(cfg, "144p")
    ref = _oracle(cfg, W, sh, z, y, 11)
    out = _gpu(cfg, W, sh, z, y, 11, cuda)
    e_z, e_v = rel_l2(out, ref), rel_l2(out - z, ref - z)
    print(f"xl2 full depth 144p: relL2 z'={e_z:.2e} update={e_v:.2e}")
    assert e_z <= 1e-2 and e_v <= 2e-2


def test_rebound_and_broadcast_text_state_match_fresh_requests(cuda):
    """ddit_request_set_text (re-binding a pooled rank state to a new caption) and
    ddit_request_copy_text (the promotion broadcast) give exactly the step of a freshly opened
    request with that caption."""
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=2)
    W, sh, z, y = _setup(cfg, "144p-16f")
    _, y2 = weights.synthetic_inputs(cfg, sh.latent, seed_z=7, seed_y=8)
    model = STDiTModel(cfg, W, cuda)
    fresh = StepRequest(model, sh, y2.to(cuda))
    z_ref = z.to(cuda).contiguous()
    fresh.step(z_ref, 4)
    pooled = StepRequest(model, sh, y.to(cuda))  # opened for another caption
    pooled.set_text(y2.to(cuda))
    z_a = z.to(cuda).contiguous()
    pooled.step(z_a, 4)
    other = StepRequest(model, sh, y.to(cuda))
    other.copy_text_from(fresh)
    z_b = z.to(cuda).contiguous()
    other.step(z_b, 4)
    torch.cuda.synchronize()
    assert torch.equal(z_a, z_ref) and torch.equal(z_b, z_ref)
    fourth = StepRequest(model, sh, y.to(cuda))
    fourth.share_text_from(fresh)  # y-embedding copied, cross K/V recomputed on this rank
    z_c = z.to(cuda).contiguous()
    fourth.step(z_c, 4)
    torch.cuda.synchronize()
    assert torch.equal(z_c, z_ref)


@pytest.mark.parametrize("dop", [4, 8])
def test_virtual_dop_long_clip_matches_dop1(cuda, dop):
    """BASELINE config 3's long-clip shape (720p x 102: T = 30, S = 3600 tokens per frame) at
    DoP 4 / 8 (virtual ranks, fused exchange) reproduces DoP 1 bit for bit (reduced width)."""
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest, VirtualGroup

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W, sh, z, y = _setup(cfg, "720p-102f")
    model = STDiTModel(cfg, W, cuda)
    yd = y.to(cuda)
    z1 = z.to(cuda).contiguous()
    StepRequest(model, sh, yd).step(z1, 9)
    grp = VirtualGroup(model, sh, yd, dop)
    parts = grp.split(z.to(cuda))
    grp.step(parts, 9)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, dim=2), z1)


@pytest.mark.parametrize("label", ["144p", "240p", "144p-16f"])
@pytest.mark.parametrize("dop", [2, 4, 8])
def test_staged_exchange_matches_dop1(cuda, dop, label):
    """The NCCL arm's staged exchange (pack per destination -> all-to-all -> unpack per source;
    the collective emulated on one device) reproduces the DoP-1 step bit for bit: checks the
    pack / unpack layouts for ragged T and S shards and for ranks that own no frames."""
    from paper_2506_13497_b200 import weights
    from paper_2506_13497_b200.stdit import STDiTModel, StagedVirtualGroup, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=2)
    W, sh, z, y = _setup(cfg, label)
    model = STDiTModel(cfg, W, cuda)
    yd = y.to(cuda)
    z1 = z.to(cuda).contiguous()
    StepRequest(model, sh, yd).step(z1, 5)
    grp = StagedVirtualGroup(model, sh, yd, dop)
    parts = grp.split(z.to(cuda))
    grp.step(parts, 5)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, dim=2), z1)


def test_exchange_barrier_times_out_instead_of_hanging(cuda):
    """A DoP-2 rank whose peer never signals: the flag-barrier spin gives up after the bound,
    records the silent rank in the request status and the stream drains (no GPU hang)."""
    import time

    from paper_2506_13497_b200 import _lib, weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = dataclasses.replace(weights.TINY, depth=1)
    W, sh, z, y = _setup(cfg, "144p-16f")
    model = STDiTModel(cfg, W, cuda)
    r0 = StepRequest(model, sh, y.to(cuda), dop=2, rank=0)
    xs, xt, fl = r0.exchange_buffers()
    r0.set_peers([xs, xs], [xt, xt], [fl, fl + 64])  # rank 1's flag slot: never written
    lib = _lib.lib()
    lib.ddit_set_exchange_timeout_ms(200)
    try:
        zl = z[:, :, r0.shard.t_lo:r0.shard.t_hi].to(cuda).contiguous()
        r0.begin(zl, 0)
        r0.phase(0)  # spatial block: rows pushed + this rank's epoch published; rank 1 is silent
        t0 = time.time()
        _lib.check(lib.ddit_step_barrier(r0.handle, _lib.stream_ptr()))
        torch.cuda.synchronize()
        assert time.time() - t0 < 10
        with pytest.raises(_lib.DditError, match="rank"):
            r0.status()
    finally:
        lib.ddit_set_exchange_timeout_ms(0)


@pytest.mark.parametrize("cfg_name,label", [("TINY", "144p-16f"), ("XL2", "240p")])
def test_padded_qkv_tiles_bit_identical(cuda, cfg_name, label):
    """The QKV GEMM on per-head padded weights (256 x 240 tiles, 80-column head slots) gives the
    same step bit for bit as the unpadded 256 x 144 tiles (XL/2 width at depth 1; tiny: 4 heads)."""
    from paper_2506_13497_b200 import _lib, weights
    from paper_2506_13497_b200.stdit import STDiTModel, StepRequest

    cfg = getattr(weights, cfg_name)
    if cfg_name == "XL2":
        cfg = dataclasses.replace(cfg, depth=1)
    W, sh, z, y = _setup(cfg, label)
    model = STDiTModel(cfg, W, cuda)
    outs = []
    for pad in (1, 0):
        _lib.lib().ddit_set_qkv_pad(pad)
        try:
            req = StepRequest(model, sh, y.to(cuda))
        finally:
            _lib.lib().ddit_set_qkv_pad(1)
        zd = z.to(cuda).contiguous()
        req.step(zd, 4)
        torch.cuda.synchronize()
        outs.append(zd.cpu())
        req.close()
    assert torch.equal(outs[0], outs[1])
