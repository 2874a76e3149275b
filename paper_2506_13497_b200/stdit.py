"""Host side of the B200 STDiT3 step: device weights, requests, the step call.

PyTorch only provides device memory and streams here; every FLOP of the step runs in
libddit.so (include/ddit.h). This is the callee that replaces the reference's timing
lookup ``ProfileTable.dit_step(resolution, dop)`` (reference pkg/src/ditsim/profiles.py:69-76)
at the engine's step sites (engine.py:245, :289, :292).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, lib, stream_ptr
from .shapes import VideoShape
from .weights import STDiTConfig

from ._lib import CBlock, CConfig, CReqDesc, CWeights

vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float


# ------------------------------------------------------------------ weights on the device
_BLOCK_MAP = [
    ("scale_shift_table", "scale_shift_table", "f32"),
    ("qkv_w", "attn.qkv.weight", "bf16"), ("qkv_b", "attn.qkv.bias", "f32"),
    ("q_norm", "attn.q_norm.weight", "f32"), ("k_norm", "attn.k_norm.weight", "f32"),
    ("proj_w", "attn.proj.weight", "bf16"), ("proj_b", "attn.proj.bias", "f32"),
    ("cq_w", "cross_attn.q_linear.weight", "bf16"), ("cq_b", "cross_attn.q_linear.bias", "f32"),
    ("ckv_w", "cross_attn.kv_linear.weight", "bf16"), ("ckv_b", "cross_attn.kv_linear.bias", "f32"),
    ("cproj_w", "cross_attn.proj.weight", "bf16"), ("cproj_b", "cross_attn.proj.bias", "f32"),
    ("fc1_w", "mlp.fc1.weight", "bf16"), ("fc1_b", "mlp.fc1.bias", "f32"),
    ("fc2_w", "mlp.fc2.weight", "bf16"), ("fc2_b", "mlp.fc2.bias", "f32"),
]
_TOP_MAP = [
    ("t0_w", "t_embedder.mlp.0.weight", "bf16"), ("t0_b", "t_embedder.mlp.0.bias", "f32"),
    ("t2_w", "t_embedder.mlp.2.weight", "bf16"), ("t2_b", "t_embedder.mlp.2.bias", "f32"),
    ("f0_w", "fps_embedder.mlp.0.weight", "bf16"), ("f0_b", "fps_embedder.mlp.0.bias", "f32"),
    ("f2_w", "fps_embedder.mlp.2.weight", "bf16"), ("f2_b", "fps_embedder.mlp.2.bias", "f32"),
    ("tb_w", "t_block.1.weight", "bf16"), ("tb_b", "t_block.1.bias", "f32"),
    ("y1_w", "y_embedder.y_proj.fc1.weight", "bf16"), ("y1_b", "y_embedder.y_proj.fc1.bias", "f32"),
    ("y2_w", "y_embedder.y_proj.fc2.weight", "bf16"), ("y2_b", "y_embedder.y_proj.fc2.bias", "f32"),
    ("y_null", "y_embedder.y_embedding", "f32"),
    ("final_sst", "final_layer.scale_shift_table", "f32"),
    ("final_w", "final_layer.linear.weight", "f32"), ("final_b", "final_layer.linear.bias", "f32"),
]


class STDiTModel:
    """STDiT3 weights resident on one device + the libddit model handle."""

    def __init__(self, cfg: STDiTConfig, weights: dict[str, torch.Tensor], device="cuda:0"):
        if cfg.head_dim != 72:
            raise ValueError("libddit supports head_dim 72 (STDiT3-XL/2 family)")
        self.cfg = cfg
        self.device = torch.device(device)
        self._keep: list[torch.Tensor] = []

        def put(name: str, kind: str) -> int:
            t = weights[name]
            t = t.to(self.device, torch.bfloat16 if kind == "bf16" else torch.float32).contiguous()
            self._keep.append(t)
            return t.data_ptr()

        w = CWeights()
        xw = weights["x_embedder.proj.weight"].reshape(cfg.hidden, -1)
        xw = xw.to(self.device, torch.float32).contiguous()
        self._keep.append(xw)
        w.x_emb_w = xw.data_ptr()
        w.x_emb_b = put("x_embedder.proj.bias", "f32")
        for field, name, kind in _TOP_MAP:
            setattr(w, field, put(name, kind))
        nblk = 2 * cfg.depth
        blocks = (CBlock * nblk)()
        for i in range(cfg.depth):
            for j, kind_name in enumerate(("spatial", "temporal")):
                b = blocks[2 * i + j]
                for field, name, kind in _BLOCK_MAP:
                    setattr(b, field, put(f"{kind_name}_blocks.{i}.{name}", kind))
        w.blocks = blocks
        self._blocks = blocks
        c = CConfig(cfg.depth, cfg.hidden, cfg.heads, cfg.head_dim, cfg.mlp_hidden,
                    cfg.in_channels, cfg.out_channels, cfg.caption_channels, cfg.text_tokens,
                    cfg.freq_dim, cfg.input_sq_size, cfg.eps)
        handle = vp()
        with torch.cuda.device(self.device):
            check(lib().ddit_model_create(ctypes.byref(c), ctypes.byref(w), ctypes.byref(handle)))
        self.handle = handle

    def close(self) -> None:
        if self.handle:
            lib().ddit_model_destroy(self.handle)
            self.handle = vp()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


@dataclass(frozen=True)
class Shard:
    t_lo: int
    t_hi: int
    s_lo: int
    s_hi: int


class StepRequest:
    """One video on one rank of a DoP-``dop`` group: workspace + cached text K/V."""

    def __init__(self, model: STDiTModel, shape: VideoShape, y_cond: torch.Tensor, *, dop: int = 1,
                 rank: int = 0, num_steps: int = 30, guidance: float = 7.0, fps: float = 24.0,
                 stream=None):
        self.model = model
        self.shape = shape
        T, H, W = shape.latent
        self.desc = CReqDesc(T, H, W, shape.height, shape.width, dop, rank, num_steps, guidance, fps)
        h = lib()
        nbytes = ctypes.c_uint64()
        check(h.ddit_request_workspace_bytes(model.handle, ctypes.byref(self.desc), ctypes.byref(nbytes)))
        sh = [ci() for _ in range(4)]
        check(h.ddit_request_shard(model.handle, ctypes.byref(self.desc), *[ctypes.byref(x) for x in sh]))
        self.shard = Shard(*(x.value for x in sh))
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=model.device)
        base = self.workspace.data_ptr()
        self._ws_ptr = (base + 255) & ~255
        y = y_cond.to(model.device, torch.float32).reshape(model.cfg.text_tokens, -1).contiguous()
        self._y = y
        handle = vp()
        check(h.ddit_request_open(model.handle, ctypes.byref(self.desc), self._ws_ptr, nbytes.value,
                                  y.data_ptr(), stream_ptr(stream), ctypes.byref(handle)))
        self.handle = handle

    @property
    def local_frames(self) -> int:
        return self.shard.t_hi - self.shard.t_lo

    def timestep(self, step: int) -> tuple[float, float]:
        t, dt = cf(), cf()
        check(lib().ddit_request_timestep(self.handle, step, ctypes.byref(t), ctypes.byref(dt)))
        return t.value, dt.value

    def step(self, z_local: torch.Tensor, step: int, stream=None) -> torch.Tensor:
        """z_local (device fp32 [1|., 4, Tl, Hl, Wl], contiguous) is updated in place."""
        assert z_local.is_cuda and z_local.dtype == torch.float32 and z_local.is_contiguous()
        check(lib().ddit_dit_step(self.handle, z_local.data_ptr(), step, stream_ptr(stream)))
        return z_local

    def graph_step(self, z_local: torch.Tensor, step: int) -> torch.Tensor:
        """The same step replayed from a CUDA graph (captured on first use per step index and
        latent buffer): the ~570 kernel launches of a step become one graph launch."""
        key = (step, z_local.data_ptr())
        graphs = self.__dict__.setdefault("_graphs", {})
        g = graphs.get(key)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            scratch = torch.empty_like(z_local)
            scratch.copy_(z_local)
            with torch.cuda.graph(g):
                self.step(z_local, step)
            z_local.copy_(scratch)  # capture does not execute; keep the caller's latent intact
            graphs[key] = g
        g.replay()
        return z_local

    # phase API (virtual ranks in lockstep on one device)
    def begin(self, z_local, step, stream=None):
        check(lib().ddit_step_begin(self.handle, z_local.data_ptr(), step, stream_ptr(stream)))

    def phase(self, k, stream=None):
        check(lib().ddit_step_phase(self.handle, k, stream_ptr(stream)))

    def end(self, z_local, step, stream=None):
        check(lib().ddit_step_end(self.handle, z_local.data_ptr(), step, stream_ptr(stream)))

    def set_text(self, y_cond: torch.Tensor, stream=None) -> None:
        """Re-bind this (pooled) rank state to a new caption [1|., 300, 4096]."""
        y = y_cond.to(self.model.device, torch.float32).reshape(self.model.cfg.text_tokens, -1).contiguous()
        self._y = y
        check(lib().ddit_request_set_text(self.handle, y.data_ptr(), stream_ptr(stream)))

    def copy_text_from(self, src: "StepRequest", stream=None) -> None:
        """Broadcast src's text embedding + cross-attention K/V cache into this rank (a peer copy
        when src lives on another GPU) -- the promotion-time state transfer."""
        check(lib().ddit_request_copy_text(self.handle, src.handle, stream_ptr(stream)))

    def share_text_from(self, src: "StepRequest", stream=None) -> None:
        """Promotion-time text state: copy src's 1.4 MB y-embedding (peer copy across GPUs) and
        recompute the cross-attention K/V cache on this rank's GPU (bit-identical to copying it)."""
        check(lib().ddit_request_share_text(self.handle, src.handle, stream_ptr(stream)))

    def exchange_buffers(self) -> tuple[int, int, int]:
        a, b, c = vp(), vp(), vp()
        check(lib().ddit_request_exchange_buffers(self.handle, ctypes.byref(a), ctypes.byref(b),
                                                  ctypes.byref(c)))
        return a.value, b.value, c.value

    def status(self, stream=None) -> int:
        """Synchronise ``stream`` and raise if the group's exchange barrier timed out (a peer
        never signalled); 0 when healthy."""
        v = ctypes.c_uint32()
        check(lib().ddit_request_status(self.handle, stream_ptr(stream), ctypes.byref(v)))
        return v.value

    def set_option(self, option: int, value: int) -> None:
        check(lib().ddit_request_set_option(self.handle, option, value))

    def profile(self, enable: bool) -> None:
        check(lib().ddit_request_profile(self.handle, 1 if enable else 0))

    def profile_read(self) -> dict[str, tuple[float, int]]:
        """Per-class (ms, launches) since profiling was enabled: gemm, attention, elementwise,
        exchange."""
        ms = (cf * 4)()
        n = (ci * 4)()
        check(lib().ddit_request_profile_read(self.handle, ms, n))
        names = ("gemm", "attention", "elementwise", "exchange")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def step_host(self, z_host: torch.Tensor, step: int, z_dev: torch.Tensor, stream=None) -> torch.Tensor:
        """End-to-end step through host memory: H2D of z, the step, D2H of z' (in place)."""
        z_dev.copy_(z_host, non_blocking=True)
        self.step(z_dev, step, stream)
        z_host.copy_(z_dev, non_blocking=True)
        return z_host

    # staged all-to-all (DDIT_OPT_EXTERNAL_XCH): the caller moves the rows between phases
    def xch_counts(self, phase: int) -> tuple[list[int], list[int]]:
        """Rows (of C fp32) this rank sends to / receives from every rank after ``phase``."""
        P = self.desc.dop
        snd, rcv = (ci * P)(), (ci * P)()
        check(lib().ddit_request_xch_counts(self.handle, phase, snd, rcv))
        return list(snd), list(rcv)

    def xch_pack(self, phase: int, send: torch.Tensor, stream=None) -> None:
        check(lib().ddit_request_xch_pack(self.handle, phase, send.data_ptr(), stream_ptr(stream)))

    def xch_unpack(self, phase: int, recv: torch.Tensor, stream=None) -> None:
        check(lib().ddit_request_xch_unpack(self.handle, phase, recv.data_ptr(), stream_ptr(stream)))

    def set_peers(self, x_sp: list[int], x_tp: list[int], flags: list[int] | None) -> None:
        n = len(x_sp)
        A = (vp * n)(*x_sp)
        Bv = (vp * n)(*x_tp)
        F = (vp * n)(*flags) if flags is not None else None
        check(lib().ddit_request_set_peers(self.handle, A, Bv, F))

    def close(self) -> None:
        if self.handle:
            lib().ddit_request_close(self.handle)
            self.handle = vp()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class VirtualGroup:
    """DoP-P sequence parallelism simulated on ONE device: P rank requests whose exchange
    pushes target each other's buffers, driven phase-by-phase in lockstep on one stream
    (stream order replaces the cross-rank barrier). Used to check that the DoP-P shard /
    exchange path reproduces DoP 1 on a single GPU."""

    def __init__(self, model: STDiTModel, shape: VideoShape, y_cond, dop: int, **kw):
        self.ranks = [StepRequest(model, shape, y_cond, dop=dop, rank=r, **kw) for r in range(dop)]
        bufs = [r.exchange_buffers() for r in self.ranks]
        for r in self.ranks:
            r.set_peers([b[0] for b in bufs], [b[1] for b in bufs], None)
        self.depth = model.cfg.depth

    def split(self, z: torch.Tensor) -> list[torch.Tensor]:
        return [z[:, :, r.shard.t_lo:r.shard.t_hi].contiguous() for r in self.ranks]

    def step(self, z_parts: list[torch.Tensor], step: int, stream=None) -> list[torch.Tensor]:
        for r, z in zip(self.ranks, z_parts):
            r.begin(z, step, stream)
        for k in range(2 * self.depth):
            for r in self.ranks:
                r.phase(k, stream)
        for r, z in zip(self.ranks, z_parts):
            r.end(z, step, stream)
        return z_parts


    def step_timed(self, z_parts: list[torch.Tensor], step: int) -> list[float]:
        """The same lockstep step with a CUDA-event pair around every rank's share of each phase
        (its kernels and its exchange pushes). Returns per-rank device ms: what each rank's GPU
        spends on the step when the ranks run on P GPUs (cross-rank waiting excluded)."""
        s = torch.cuda.current_stream()

        def ev():
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            return e

        spans: list[list[tuple]] = [[] for _ in self.ranks]
        for i, (r, z) in enumerate(zip(self.ranks, z_parts)):
            a = ev()
            r.begin(z, step)
            spans[i].append((a, ev()))
        for k in range(2 * self.depth):
            for i, r in enumerate(self.ranks):
                a = ev()
                r.phase(k)
                spans[i].append((a, ev()))
        for i, (r, z) in enumerate(zip(self.ranks, z_parts)):
            a = ev()
            r.end(z, step)
            spans[i].append((a, ev()))
        s.synchronize()
        return [sum(a.elapsed_time(b) for a, b in sp) for sp in spans]


DDIT_OPT_TC_ATTENTION = 1
DDIT_OPT_EXTERNAL_XCH = 2


class StagedVirtualGroup(VirtualGroup):
    """DoP-P on one device with the staged exchange the NCCL arm uses: after every phase each
    rank packs its outgoing rows per destination (``xch_pack``), the all-to-all is done by
    concatenating send blocks into every rank's receive buffer on the device (what ncclAllToAllv
    does between GPUs), and each rank unpacks (``xch_unpack``). Checks the pack/unpack layout
    against DoP 1 without a second GPU."""

    def __init__(self, model: STDiTModel, shape: VideoShape, y_cond, dop: int, **kw):
        self.ranks = [StepRequest(model, shape, y_cond, dop=dop, rank=r, **kw) for r in range(dop)]
        for r in self.ranks:
            r.set_option(DDIT_OPT_EXTERNAL_XCH, 1)
        self.depth = model.cfg.depth
        self.C = model.cfg.hidden
        self.counts = [[r.xch_counts(d) for d in (0, 1)] for r in self.ranks]
        rows = max(max(sum(c[0]), sum(c[1])) for rc in self.counts for c in rc)
        dev = model.device
        self.send = [torch.empty((max(rows, 1), self.C), device=dev) for _ in self.ranks]
        self.recv = [torch.empty((max(rows, 1), self.C), device=dev) for _ in self.ranks]

    def all_to_all(self, phase: int, stream=None) -> None:
        d = phase & 1
        P = len(self.ranks)
        for q in range(P):
            off = 0
            for r in range(P):
                snd = self.counts[r][d][0]
                lo = sum(snd[:q])
                n = snd[q]
                self.recv[q][off:off + n].copy_(self.send[r][lo:lo + n])
                off += n

    def step(self, z_parts: list[torch.Tensor], step: int, stream=None) -> list[torch.Tensor]:
        for r, z in zip(self.ranks, z_parts):
            r.begin(z, step, stream)
        for k in range(2 * self.depth):
            for r in self.ranks:
                r.phase(k, stream)
            for r, sb in zip(self.ranks, self.send):
                r.xch_pack(k, sb, stream)
            self.all_to_all(k, stream)
            for r, rb in zip(self.ranks, self.recv):
                r.xch_unpack(k, rb, stream)
        for r, z in zip(self.ranks, z_parts):
            r.end(z, step, stream)
        return z_parts


def launch_count() -> int:
    """Kernel launches issued by libddit in this process (bench evidence)."""
    return int(lib().ddit_launch_count())
