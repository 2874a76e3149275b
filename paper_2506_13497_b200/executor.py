"""Real B200 work behind the serving loop's step sites, and the measured profile.

``B200Executor`` implements ``sched.StepExecutor``: plugged into ``sched.Simulation(...,
executor=...)`` it runs the actual STDiT3 step wherever the reference only looks a time up --
DiT step at start (reference pkg/src/ditsim/engine.py:245), after a promotion (:289), steady
state (:292) -- and the DiT->VAE hand-off before the VAE (:305). The engine's clock advances by
the measured (CUDA-event) durations, so traces are driven by real step times while every
allocator / policy decision stays the reference's.

* A request's latent lives as per-rank T-shards on the GPUs of its group. On a promotion
  P -> P' (the engine jumps from the applied set to the final pending set, SURVEY Appendix
  A.6) the new group's ranks gather their new frame ranges from the old shards with
  ``ddit_latent_gather`` (peer loads) before the step -- the reference's 1 ms + 1 ms constants
  (engine.py:52-61) become a measured re-shard.
* Engine GPU ids map onto physical devices ``gpu_id % device_count``. A group whose ids land
  on distinct devices runs one rank per device concurrently with the peer-store exchange; any
  other group (all on one device, or more ranks than devices, e.g. DoP 4 on a 2-GPU box) runs
  as virtual ranks in lockstep on the device of its first id (``VirtualGroup``).
* Rank states (workspace, tables, GEMM / attention plans) are pooled per (resolution, devices):
  a new request re-binds a pooled group to its caption (``ddit_request_set_text``); a promotion
  takes a pooled group for the new GPU set and broadcasts the text state from the old rank 0
  (``ddit_request_copy_text``) together with the latent re-shard, which is what the reference's
  broadcast + scale-up constants stand for. ``reshard_seconds`` is that device work (CUDA events,
  max over the new ranks when the group is emulated); ``reshard_host_seconds`` the host work of
  the promotion (re-bind + enqueue), ``reshard_wall_seconds`` the wall time including the device wait.
* ``profile_b200`` measures ``dit_step_seconds`` per (resolution, DoP) and emits the
  reference's ``dit-profile/1`` document (profiles.py:132-215).
"""

from __future__ import annotations

import ctypes
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import torch

from ._lib import check, lib
from .shapes import VideoShape, shape_of
from .sched.engine import RequestState
from .stdit import STDiTModel, StepRequest, VirtualGroup
from .weights import STDiTConfig, synthetic_inputs

vp, ci = ctypes.c_void_p, ctypes.c_int


def latent_gather(dst: torch.Tensor, t_lo: int, t_hi: int, sources: list[tuple[torch.Tensor, int, int]],
                  stream=None) -> None:
    """dst [1|., C, t_hi-t_lo, H, W] <- frames of the shards (tensor, t_lo, t_hi) that cover it."""
    from ._lib import stream_ptr

    n = len(sources)
    P = (vp * n)(*[s[0].data_ptr() for s in sources])
    lo = (ci * n)(*[s[1] for s in sources])
    hi = (ci * n)(*[s[2] for s in sources])
    C, HW = dst.shape[-4], dst.shape[-2] * dst.shape[-1]
    check(lib().ddit_latent_gather(dst.data_ptr(), t_lo, t_hi, P, lo, hi, n, C, HW, stream_ptr(stream)))


def reshard(new_ranks: list[StepRequest], new_shards: list[torch.Tensor], old_ranks: list[StepRequest],
            old_shards: list[torch.Tensor], streams=None) -> None:
    """Promotion P -> P' in one C call (``ddit_reshard``): every new rank, on its own device
    (and stream), gathers its frames from the old shards and takes the text state of old rank 0
    (1.4 MB y-embedding + local cross-K/V recompute)."""
    q, p = len(new_ranks), len(old_ranks)
    nr = (vp * q)(*[r.handle.value for r in new_ranks])
    nz = (vp * q)(*[z.data_ptr() for z in new_shards])
    oz = (vp * p)(*[z.data_ptr() for z in old_shards])
    lo = (ci * p)(*[r.shard.t_lo for r in old_ranks])
    hi = (ci * p)(*[r.shard.t_hi for r in old_ranks])
    st = (vp * q)(*[s.cuda_stream for s in streams]) if streams is not None else None
    check(lib().ddit_reshard(nr, nz, q, oz, lo, hi, p, old_ranks[0].handle, st))


def reshard_seconds(ranks: list[StepRequest]) -> list[float]:
    """Device seconds of the last ``reshard`` into each rank (synchronises on it)."""
    out = []
    for r in ranks:
        ms = ctypes.c_float()
        check(lib().ddit_request_reshard_ms(r.handle, ctypes.byref(ms)))
        out.append(ms.value / 1e3)
    return out


def exchange_bytes(sh: VideoShape, P: int, rank: int, C: int, B: int = 2) -> int:
    """Bytes rank ``rank`` of a DoP-P group pushes to its peers in one step: 28 spatial->temporal
    exchanges (its T-shard rows outside its own S-shard) + 28 temporal->spatial ones (its S-shard
    rows outside its own T-shard), fp32 residual rows of C channels, CFG batch B."""
    if P == 1:
        return 0
    from .shapes import s_shard, t_shard

    t_lo, t_hi = t_shard(sh, P, rank)
    s_lo, s_hi = s_shard(sh, P, rank)
    Tl, Sl = t_hi - t_lo, s_hi - s_lo
    return 28 * (B * Tl * (sh.S - Sl) * C * 4 + B * (sh.T - Tl) * Sl * C * 4)


@dataclass
class _Live:
    """One request's device state on its current group."""

    gpu_ids: tuple[int, ...]
    ranks: list[StepRequest]
    shards: list[torch.Tensor]  # z T-shards, rank order
    group: VirtualGroup | None = None
    key: tuple = ()  # pool key: (resolution, devices)
    steps_done: int = 0
    history: list[tuple[int, ...]] = field(default_factory=list)


class B200Executor:
    """Executes real STDiT3 steps for ``sched.Simulation`` (see module docstring)."""

    def __init__(self, cfg: STDiTConfig, weights: dict[str, torch.Tensor], *,
                 shapes: dict[str, VideoShape] | None = None, num_steps: int = 30,
                 guidance: float = 7.0, seed_base: int = 0, vae_cfg=None, vae_weights=None,
                 keep_videos: bool = False, emulate_group: bool = False,
                 nvlink_gbs: float = 770.0, latent_dir: str | None = None):
        self.cfg = cfg
        self.ndev = max(torch.cuda.device_count(), 1)
        self.models: dict[int, STDiTModel] = {}
        self._weights = weights
        self.shapes = shapes or {}
        self.num_steps = num_steps
        self.guidance = guidance
        self.seed_base = seed_base
        self.live: dict[int, _Live] = {}
        self.final_latents: dict[int, torch.Tensor] = {}
        self.step_seconds: list[tuple[int, int, float]] = []  # (request, dop, seconds)
        self.reshard_seconds: list[float] = []
        self.vae_cfg = vae_cfg
        self._vae_weights = vae_weights
        self.vaes: dict[int, object] = {}
        self.keep_videos = keep_videos
        self.videos: dict[int, torch.Tensor] = {}
        self.vae_seconds: list[tuple[int, float, float]] = []  # (request, handoff s, decode s)
        # A group whose ranks share one device normally reports the whole group's time on that
        # device. With emulate_group it reports the DoP-P step latency the group would have on P
        # GPUs: max over ranks of each rank's own device time + its exchange bytes over NVLink
        # (measured 770 GB/s peer copy), so one B200 can replay an 8-GPU trace.
        self.emulate_group = emulate_group
        self.nvlink_gbs = nvlink_gbs
        self.pool: dict[tuple, list[_Live]] = {}  # (resolution, devices) -> idle groups
        self.pool_limit = 4
        self._enqueue_pool: ThreadPoolExecutor | None = None  # per-rank step enqueue threads
        # host work of a promotion: pool re-bind + enqueue of the one-call re-shard on every rank
        self.reshard_host_seconds: list[float] = []
        # wall time until the re-shard finished (host + device wait); with emulated groups the
        # virtual ranks' re-shards run one after another on one GPU, so this grows with P' there
        self.reshard_wall_seconds: list[float] = []
        # when set, every request's denoised latent (+ frames with keep_videos) is also written
        # in the latent_io on-disk format as the DiT group hands it off
        self.latent_dir = latent_dir

    # ---------------------------------------------------------------- helpers
    def device_of(self, gpu_id: int) -> int:
        return gpu_id % self.ndev

    def devices_of(self, gpu_ids: tuple[int, ...]) -> list[int]:
        """Device of every rank of a group: one per id when the ids land on distinct devices,
        else the whole group on the first id's device (virtual ranks)."""
        devs = [self.device_of(g) for g in gpu_ids]
        return devs if len(set(devs)) == len(devs) else [devs[0]] * len(devs)

    def _model(self, dev: int) -> STDiTModel:
        if dev not in self.models:
            self.models[dev] = STDiTModel(self.cfg, self._weights, torch.device("cuda", dev))
        return self.models[dev]

    def _shape(self, request: RequestState) -> VideoShape:
        return self.shapes.get(request.resolution) or shape_of(request.resolution)

    def _inputs(self, request: RequestState):
        sh = self._shape(request)
        return synthetic_inputs(self.cfg, sh.latent, seed_z=self.seed_base + 2 * request.request_id,
                                seed_y=self.seed_base + 2 * request.request_id + 1)

    def _open(self, request: RequestState, gpu_ids: tuple[int, ...],
              text_from: StepRequest | None = None) -> _Live:
        """A group for ``gpu_ids``: pooled if one is idle (re-bound to this request's caption, or
        given ``text_from``'s text state by a broadcast copy), else newly opened."""
        devs = self.devices_of(gpu_ids)
        key = (request.resolution, tuple(devs))
        idle = self.pool.get(key)
        if idle:
            live = idle.pop()
            live.gpu_ids = tuple(gpu_ids)
            live.steps_done, live.history = 0, []
            if text_from is None:
                _, y = self._inputs(request)
                for r, d in zip(live.ranks, devs):
                    with torch.cuda.device(d):
                        r.set_text(y)
            return live
        return self._open_new(request, gpu_ids)

    def _open_new(self, request: RequestState, gpu_ids: tuple[int, ...]) -> _Live:
        sh = self._shape(request)
        _, y = self._inputs(request)
        # more ranks than distinct devices (e.g. DoP 4 on a 2-GPU box): the whole group runs as
        # virtual ranks on the device of its first id (emulate_group reports its P-GPU time)
        devs = self.devices_of(gpu_ids)
        dop = len(gpu_ids)
        if len(set(devs)) == 1:
            model = self._model(devs[0])
            with torch.cuda.device(devs[0]):
                grp = VirtualGroup(model, sh, y.to(model.device), dop, num_steps=self.num_steps,
                                   guidance=self.guidance)
            ranks, group = grp.ranks, grp
        else:
            ranks = []
            for r, d in enumerate(devs):
                with torch.cuda.device(d):
                    ranks.append(StepRequest(self._model(d), sh, y.to(torch.device("cuda", d)), dop=dop,
                                             rank=r, num_steps=self.num_steps, guidance=self.guidance))
            bufs = [r.exchange_buffers() for r in ranks]
            for d in devs:
                for e in devs:
                    if d != e and torch.cuda.can_device_access_peer(d, e):
                        check(lib().ddit_enable_peer_access(d, e))
            for r in ranks:
                r.set_peers([b[0] for b in bufs], [b[1] for b in bufs], [b[2] for b in bufs])
            group = None
        shards = []
        for r, d in zip(ranks, devs):
            Tl = r.shard.t_hi - r.shard.t_lo
            shards.append(torch.empty((1, self.cfg.in_channels, Tl, *sh.latent[1:]),
                                      device=torch.device("cuda", d)))
        return _Live(tuple(gpu_ids), ranks, shards, group, key=(request.resolution, tuple(devs)))

    def preopen(self, resolutions, n_gpus: int) -> int:
        """Open one pooled group per (resolution, buddy block) before serving: the single
        GPUs, aligned pairs, quads and octet of an ``n_gpus`` node (15 groups for 8 GPUs) -- the
        only shapes the greedy allocator hands out (reference allocator.py:221-234, :356-408).
        A later start or promotion then re-binds an open group instead of allocating workspace,
        building tables and GEMM / attention plans. Returns the number of groups opened."""
        n = 0
        for res in resolutions:
            size = 1
            while size <= n_gpus:
                for start in range(0, n_gpus - size + 1, size):
                    ids = tuple(range(start, start + size))
                    probe = RequestState(1_000_000_000 + n, res, 0.0, self.num_steps)
                    live = self._open_new(probe, ids)
                    self.pool.setdefault(live.key, []).append(live)
                    n += 1
                size *= 2
        return n

    # ---------------------------------------------------------------- StepExecutor protocol
    def dit_step(self, request: RequestState, gpu_ids: tuple[int, ...], step: int,
                 resharded_from: tuple[int, ...] | None) -> float:
        t0 = time.perf_counter()
        live = self.live.get(request.request_id)
        if live is None:  # first step: latent z0 sharded over the group
            live = self._open(request, gpu_ids)
            z0, _ = self._inputs(request)
            for r, zs in zip(live.ranks, live.shards):
                zs.copy_(z0[:, :, r.shard.t_lo:r.shard.t_hi])
            self.live[request.request_id] = live
        elif tuple(gpu_ids) != live.gpu_ids:  # promotion P -> P': re-shard at the boundary
            new = self._open(request, gpu_ids, text_from=live.ranks[0])
            # one C call: every new rank gathers its z frames (peer loads) and takes the text
            # state (1.4 MB y-embedding + local cross-K/V recompute) on its own device
            reshard(new.ranks, new.shards, live.ranks, live.shards)
            t_enq = time.perf_counter()
            per = reshard_seconds(new.ranks)
            one_device = len({zs.device.index for zs in new.shards}) == 1
            # ranks on P GPUs re-shard concurrently; virtual ranks on one device ran one by one
            dev_s = max(per) if (self.emulate_group or not one_device) else sum(per)
            self.reshard_seconds.append(dev_s)
            self.reshard_wall_seconds.append(time.perf_counter() - t0)
            self.reshard_host_seconds.append(t_enq - t0)
            new.steps_done = live.steps_done
            new.history = live.history + [live.gpu_ids]
            self._close(live)
            self.live[request.request_id] = live = new
        secs = self._run_step(live, step)
        live.steps_done += 1
        self.step_seconds.append((request.request_id, len(gpu_ids), secs))
        if resharded_from is not None and self.reshard_seconds:
            secs += self.reshard_seconds[-1]
        return secs

    def _vae(self, dev: int):
        if dev not in self.vaes:
            from .vae import VAEDecoder

            self.vaes[dev] = VAEDecoder(self.vae_cfg, self._vae_weights, torch.device("cuda", dev))
        return self.vaes[dev]

    def vae(self, request: RequestState, dit_gpu_ids: tuple[int, ...],
            vae_gpu_ids: tuple[int, ...]) -> float:
        """DiT -> VAE hand-off and decode on the retained GPUs (K12 + K13). With ``q`` retained
        GPUs (the policy's vae_dop, reference policies.py:175-190) rank r owns an even block of
        video frames: it gathers the latent frames of the temporal micro-batches those frames
        fall in from the DiT T-shards (peer loads) and decodes only its frames
        (``vae.vae_shard``); the video is the ranks' frames in order. Seconds = max over ranks of
        gather + decode (device time; ranks of one device are emulated)."""
        live = self.live.pop(request.request_id)
        sh = self._shape(request)
        q = len(vae_gpu_ids)
        srcs = [(zs, r.shard.t_lo, r.shard.t_hi) for r, zs in zip(live.ranks, live.shards)]
        handoffs, decodes, parts, latents = [], [], [], []
        for rank, gid in enumerate(vae_gpu_ids):
            dev = self.device_of(gid)
            if self.vae_cfg is not None:
                from .vae import vae_shard

                t_lo, t_hi, f_lo, f_hi = vae_shard(self.vae_cfg, sh.T, sh.frames, q, rank)
                mf = self.vae_cfg.micro_frame_size
                f0 = t_lo // self.vae_cfg.micro_z * mf  # first frame of the rank's micro-batches
                part_frames = min(-(-(t_hi - t_lo) // self.vae_cfg.micro_z) * mf, sh.frames - f0)
            else:  # no decoder: the whole latent goes to the master
                t_lo, t_hi, f_lo, f_hi = (0, sh.T, 0, sh.frames) if rank == 0 else (0, 0, 0, 0)
            if t_hi <= t_lo:
                continue
            with torch.cuda.device(dev):
                z = torch.empty((1, self.cfg.in_channels, t_hi - t_lo, *sh.latent[1:]),
                                device=torch.device("cuda", dev))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                latent_gather(z, t_lo, t_hi, srcs)  # peer loads of the T-shards covering [t_lo, t_hi)
                b.record()
                b.synchronize()
                handoffs.append(a.elapsed_time(b) / 1e3)
                latents.append(z)
                if self.vae_cfg is not None:
                    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s0.record()
                    video = self._vae(dev).decode(z, part_frames, sh.height, sh.width,
                                                  frames=(f_lo - f0, f_hi - f0))
                    s1.record()
                    s1.synchronize()
                    decodes.append(s0.elapsed_time(s1) / 1e3)
                    parts.append(video)
        master = self.device_of(vae_gpu_ids[0])
        if q == 1 or self.vae_cfg is None:
            self.final_latents[request.request_id] = latents[0]
        else:  # the ranks' latent ranges overlap at micro-batch boundaries
            with torch.cuda.device(master):
                zf = torch.empty((1, self.cfg.in_channels, *sh.latent), device=torch.device("cuda", master))
                latent_gather(zf, 0, sh.T, srcs)
                # the source shards go back to the pool below: finish reading them first
                torch.cuda.current_stream().synchronize()
            self.final_latents[request.request_id] = zf
        self._close(live)
        if self.keep_videos and parts:
            self.videos[request.request_id] = (
                parts[0] if len(parts) == 1
                else torch.cat([v.to(torch.device("cuda", master)) for v in parts], dim=2))
        if self.latent_dir is not None:
            from pathlib import Path

            from .latent_io import save_latent

            Path(self.latent_dir).mkdir(parents=True, exist_ok=True)
            save_latent(Path(self.latent_dir) / f"req{request.request_id}.ddlat",
                        self.final_latents[request.request_id], request_id=request.request_id,
                        resolution=request.resolution, steps=live.steps_done,
                        frames=self.videos.get(request.request_id), dit_gpu_ids=list(dit_gpu_ids),
                        vae_gpu_ids=list(vae_gpu_ids))
        decodes += [0.0] * (len(handoffs) - len(decodes))
        slowest = max(range(len(handoffs)), key=lambda i: handoffs[i] + decodes[i])
        self.vae_seconds.append((request.request_id, handoffs[slowest], decodes[slowest]))
        return handoffs[slowest] + decodes[slowest]

    # ---------------------------------------------------------------- internals
    def _run_step(self, live: _Live, step: int) -> float:
        step = min(step, self.num_steps - 1)
        if live.group is not None and self.emulate_group and len(live.ranks) > 1:
            with torch.cuda.device(live.shards[0].device):
                per_rank = live.group.step_timed(live.shards, step)
            sh = live.ranks[0].shape
            P = len(live.ranks)
            xb = max(exchange_bytes(sh, P, r, self.cfg.hidden) for r in range(P))
            return max(per_rank) / 1e3 + xb / (self.nvlink_gbs * 1e9)
        if live.group is not None:
            dev = live.shards[0].device
            with torch.cuda.device(dev):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                live.group.step(live.shards, step)
                e.record()
                e.synchronize()
                return s.elapsed_time(e) / 1e3
        # one host thread per rank enqueues that rank's step on its own device (the C calls drop
        # the GIL): a rank whose kernels wait on peer flags never depends on the host having
        # already queued the peers' ~600 launches behind it
        def run(i: int):
            r, zs = live.ranks[i], live.shards[i]
            with torch.cuda.device(zs.device):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                r.step(zs, step)
                e.record()
                return s, e
        if len(live.ranks) == 1:
            evs = [run(0)]
        else:
            if self._enqueue_pool is None or self._enqueue_pool._max_workers < len(live.ranks):
                self._enqueue_pool = ThreadPoolExecutor(max_workers=max(8, len(live.ranks)))
            evs = list(self._enqueue_pool.map(run, range(len(live.ranks))))
        for _, e in evs:
            e.synchronize()
        return max(s.elapsed_time(e) for s, e in evs) / 1e3

    def _close(self, live: _Live) -> None:
        """Return the group's rank states to the pool (closed when the pool is full)."""
        idle = self.pool.setdefault(live.key, [])
        if len(idle) < self.pool_limit:
            idle.append(live)
            return
        for r in live.ranks:
            r.close()

    def close(self) -> None:
        if self._enqueue_pool is not None:
            self._enqueue_pool.shutdown()
            self._enqueue_pool = None
        for idle in self.pool.values():
            for live in idle:
                for r in live.ranks:
                    r.close()
        self.pool.clear()


def profile_b200(cfg: STDiTConfig, weights: dict[str, torch.Tensor], labels: list[str],
                 dops=(1, 2, 4, 8), repeats: int = 3, vae_seconds: dict[str, float] | None = None,
                 gpu_ids_of=None, vae_cfg=None, vae_weights=None) -> dict:
    """Measure dit_step_seconds per (resolution, DoP) on this machine's GPUs and return a
    ``dit-profile/1`` document (reference profiles.py:132-215). DoPs beyond the visible device
    count run as virtual ranks on one device (flagged ``"virtual": true`` in the entry)."""
    # groups wider than the visible devices run as virtual ranks; emulate_group makes their
    # entry the DoP-P latency (max over ranks + exchange bytes over NVLink), not the serialised
    # time of all ranks on one device
    ex = B200Executor(cfg, weights, emulate_group=True)
    entries = []
    for res in labels:
        for d in dops:
            req = RequestState(10_000 + len(entries), res, 0.0, 30)
            ids = tuple(range(d)) if gpu_ids_of is None else gpu_ids_of(d)
            ex.dit_step(req, ids, 0, None)  # warm-up + open
            times = [ex._run_step(ex.live[req.request_id], 1 + i) for i in range(repeats)]
            ex._close(ex.live.pop(req.request_id))
            e = {"resolution": res, "dop": d, "dit_step_seconds": min(times)}
            if len({ex.device_of(g) for g in ids}) < d:
                e["virtual"] = True
            if d == 1:
                if vae_cfg is not None:  # measured decode on one GPU (the VAE DoP DDiT uses)
                    from .vae import VAEDecoder

                    sh = shape_of(res)
                    dec = VAEDecoder(vae_cfg, vae_weights, torch.device("cuda", 0))
                    z = torch.randn((1, cfg.in_channels, *sh.latent), device="cuda:0")
                    dec.decode(z, sh.frames, sh.height, sh.width)
                    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s0.record()
                    dec.decode(z, sh.frames, sh.height, sh.width)
                    s1.record()
                    s1.synchronize()
                    e["vae_seconds"] = s0.elapsed_time(s1) / 1e3
                else:
                    e["vae_seconds"] = (vae_seconds or {}).get(res, 1e-6)
            entries.append(e)
    return {"schema": "dit-profile/1", "dop_candidates": list(dops), "entries": entries}
