"""Wall-clock serving: the reference serving loop with real time.

``sched.Simulation`` (the reference engine, reference pkg/src/ditsim/engine.py:179-364) advances a
virtual clock by the seconds each step site returns. ``WallClockSimulation`` keeps its handlers,
policy hooks and allocator unchanged but takes time from the machine:

* every DiT step, re-shard and DiT->VAE hand-off + decode is ENQUEUED on the request group's own
  CUDA streams (``AsyncB200Executor``) and the loop returns at once, so groups on disjoint GPUs
  (or, on a one-GPU box, concurrent streams of one GPU) run at the same time;
* a STEP_COMPLETE / VAE_COMPLETE event fires when the group's CUDA events complete, stamped with
  the device time elapsed since a clock-zero event recorded on every device at start;
* arrivals fire when the wall clock reaches ``arrival_time * time_scale``.

Decisions therefore follow measured times (they differ from the virtual-time run exactly where
real step times differ from the profile). Metrics come from ``sched.compute_metrics``
(reference metrics.py:40-54) over the wall-clock trace.

The DiT->VAE hand-off is asynchronous: the retained GPU's stream gathers the latent T-shards
(peer loads, ``ddit_latent_gather``) and decodes right behind them on the same stream; the DiT
group is returned to the pool only once that gather's event has completed, so released GPUs can
start other requests immediately (reference policies.py:175-190, engine.py:297-310) without
their buffers being reused under the reader.
"""

from __future__ import annotations

import heapq
import time
from dataclasses import dataclass, field

import torch

from .executor import B200Executor, _Live, latent_gather, reshard
from .sched.engine import EventKind, RequestStatus, SimResult, Simulation


@dataclass
class Pending:
    """Device work of one step / decode: done when every rank's end event has completed."""

    ends: list  # [(device, torch.cuda.Event)]
    starts: list = field(default_factory=list)
    on_done: object = None  # callable run once, when the engine observes completion

    def query(self) -> bool:
        return all(e.query() for _, e in self.ends)

    def device_seconds(self) -> float:
        if not self.starts:
            return 0.0
        return max(s.elapsed_time(e) for (_, s), (_, e) in zip(self.starts, self.ends)) / 1e3


class AsyncB200Executor(B200Executor):
    """``B200Executor`` whose step sites enqueue and return a ``Pending`` instead of waiting.

    Every pooled group owns one stream per rank device; a group taken from the pool first waits
    on the events recorded when it was released (its buffers may still be read by a hand-off).
    Multi-device groups launch each rank's step as one CUDA graph replay, so no rank's launch
    queue has to hold a whole eager step while it waits at the exchange barrier."""

    def __init__(self, *a, **kw):
        kw.setdefault("emulate_group", False)
        super().__init__(*a, **kw)
        self.clock_zero: dict[int, torch.cuda.Event] = {}
        self.step_log: list[tuple[int, int, int]] = []  # (request, step, dop)

    # ---- clock
    def mark_clock_zero(self, devices) -> None:
        for d in devices:
            with torch.cuda.device(d):
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                self.clock_zero[d] = e

    def device_time(self, p: Pending) -> float:
        """Seconds since clock zero at which the pending work finished (latest rank)."""
        return max(self.clock_zero[d].elapsed_time(e) for d, e in p.ends) / 1e3

    # ---- groups with streams
    def _streams(self, live: _Live) -> list:
        st = getattr(live, "streams", None)
        if st is None:
            st = []
            for zs in live.shards:
                st.append(torch.cuda.Stream(device=zs.device))
            live.streams = st
        return st

    def _take(self, live: _Live) -> list:
        """Streams of a group just taken (pooled or new), ordered after its last release."""
        st = self._streams(live)
        for s in st:
            # opening / re-binding the group (tables, caption embedding) ran on the device's
            # current stream
            s.wait_stream(torch.cuda.current_stream(s.device))
            for e in getattr(live, "release", ()):
                s.wait_event(e)
        live.release = []
        return st

    def _record_ends(self, live: _Live, starts=None) -> Pending:
        ends = []
        for s, zs in zip(live.streams, live.shards):
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ends.append((zs.device.index, e))
        return Pending(ends, starts or [])

    def _start_events(self, live: _Live) -> list:
        out = []
        for s, zs in zip(live.streams, live.shards):
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            out.append((zs.device.index, e))
        return out

    # ---- step sites
    def dit_step_async(self, request, gpu_ids, step: int, resharded_from) -> Pending:
        live = self.live.get(request.request_id)
        if live is None:
            live = self._open(request, gpu_ids)
            st = self._take(live)
            starts = self._start_events(live)
            z0, _ = self._inputs(request)
            for r, zs, s in zip(live.ranks, live.shards, st):
                with torch.cuda.stream(s):
                    zs.copy_(z0[:, :, r.shard.t_lo:r.shard.t_hi], non_blocking=True)
            self.live[request.request_id] = live
        elif tuple(gpu_ids) != live.gpu_ids:  # promotion: re-shard on the new group's streams
            new = self._open(request, gpu_ids, text_from=live.ranks[0])
            st = self._take(new)
            for s in st:
                for os_ in self._streams(live):
                    s.wait_stream(os_)
            starts = self._start_events(new)
            reshard(new.ranks, new.shards, live.ranks, live.shards, streams=st)
            new.steps_done = live.steps_done
            new.history = live.history + [live.gpu_ids]
            # the old group may be handed out again only after the gather has read it
            done = []
            for s, zs in zip(st, new.shards):
                e = torch.cuda.Event()
                e.record(s)
                done.append(e)
            live.release = done
            self._close(live)
            self.live[request.request_id] = live = new
        else:
            st = self._streams(live)
            starts = self._start_events(live)
        step = min(step, self.num_steps - 1)
        if live.group is not None:  # virtual ranks of one device: lockstep on the group stream
            for s in st[1:]:  # their z copies / re-shard gathers ran on the rank streams
                st[0].wait_stream(s)
            with torch.cuda.device(live.shards[0].device), torch.cuda.stream(st[0]):
                live.group.step(live.shards, step, stream=st[0])
        else:  # one rank per device: each rank's whole step is one graph replay on its stream
            for r, zs, s in zip(live.ranks, live.shards, st):
                with torch.cuda.device(zs.device), torch.cuda.stream(s):
                    r.graph_step(zs, step)
        live.steps_done += 1
        self.step_log.append((request.request_id, step, len(gpu_ids)))
        return self._record_ends(live, starts)

    def vae_async(self, request, dit_gpu_ids, vae_gpu_ids) -> Pending:
        live = self.live.pop(request.request_id)
        sh = self._shape(request)
        srcs = [(zs, r.shard.t_lo, r.shard.t_hi) for r, zs in zip(live.ranks, live.shards)]
        dit_streams = self._streams(live)
        ends, starts, gathers = [], [], []
        q = len(vae_gpu_ids)
        parts = []
        for rank, gid in enumerate(vae_gpu_ids):
            dev = self.device_of(gid)
            if self.vae_cfg is not None:
                from .vae import vae_shard

                t_lo, t_hi, f_lo, f_hi = vae_shard(self.vae_cfg, sh.T, sh.frames, q, rank)
                mf = self.vae_cfg.micro_frame_size
                f0 = t_lo // self.vae_cfg.micro_z * mf
                part_frames = min(-(-(t_hi - t_lo) // self.vae_cfg.micro_z) * mf, sh.frames - f0)
            else:
                t_lo, t_hi, f_lo, f_hi = (0, sh.T, 0, sh.frames) if rank == 0 else (0, 0, 0, 0)
            if t_hi <= t_lo:
                continue
            with torch.cuda.device(dev):
                s = self._vae_stream(dev)
                for ds in dit_streams:
                    s.wait_stream(ds)
                a = torch.cuda.Event(enable_timing=True)
                a.record(s)
                with torch.cuda.stream(s):
                    z = torch.empty((1, self.cfg.in_channels, t_hi - t_lo, *sh.latent[1:]),
                                    device=torch.device("cuda", dev))
                    latent_gather(z, t_lo, t_hi, srcs, stream=s)
                    g = torch.cuda.Event()
                    g.record(s)
                    gathers.append(g)
                    if self.vae_cfg is not None:
                        video = self._vae(dev).decode(z, part_frames, sh.height, sh.width,
                                                      frames=(f_lo - f0, f_hi - f0))
                        parts.append(video)
                    if rank == 0:
                        self.final_latents[request.request_id] = z
                b = torch.cuda.Event(enable_timing=True)
                b.record(s)
                starts.append((dev, a))
                ends.append((dev, b))
        live.release = gathers  # DiT buffers reusable once the hand-off has read them
        self._close(live)
        if self.keep_videos and parts:
            master = self.device_of(vae_gpu_ids[0])
            self.videos[request.request_id] = (
                parts[0] if len(parts) == 1
                else torch.cat([v.to(torch.device("cuda", master)) for v in parts], dim=2))
        return Pending(ends, starts)

    def _vae_stream(self, dev: int):
        vs = self.__dict__.setdefault("_vae_streams", {})
        if dev not in vs:
            vs[dev] = torch.cuda.Stream(device=dev)
        return vs[dev]


class _Adapter:
    """Executor protocol of ``Simulation`` on top of the async executor: each call enqueues the
    work, registers its ``Pending`` with the loop and returns 0 s (the completion time is taken
    from the device when the events complete)."""

    def __init__(self, sim: "WallClockSimulation", ex: AsyncB200Executor):
        self.sim, self.ex = sim, ex

    def dit_step(self, request, gpu_ids, step, resharded_from):
        self.sim._register(request.request_id, EventKind.STEP_COMPLETE,
                           self.ex.dit_step_async(request, gpu_ids, step, resharded_from))
        return 0.0

    def vae(self, request, dit_gpu_ids, vae_gpu_ids):
        self.sim._register(request.request_id, EventKind.VAE_COMPLETE,
                           self.ex.vae_async(request, dit_gpu_ids, vae_gpu_ids))
        return 0.0


class WallClockSimulation(Simulation):
    """The reference engine driven by real time (see module docstring).

    ``time_scale`` stretches (or compresses) the workload's arrival times; ``poll_s`` is the idle
    sleep of the host loop."""

    def __init__(self, topology, profile, dop_table, workload, policy, executor: AsyncB200Executor,
                 *, time_scale: float = 1.0, poll_s: float = 50e-6, **kw):
        super().__init__(topology, profile, dop_table, workload, policy, executor=None, **kw)
        self.async_executor = executor
        self.executor = _Adapter(self, executor)
        self.time_scale = time_scale
        self.poll_s = poll_s
        self._registered: dict[tuple[EventKind, int], Pending] = {}
        self._inflight: list[tuple[EventKind, int, Pending]] = []
        self.device_seconds: list[tuple[str, int, float]] = []  # (kind, request, device s)

    def _register(self, rid: int, kind: EventKind, p: Pending) -> None:
        self._registered[(kind, rid)] = p

    def schedule_event(self, time_s: float, kind: EventKind, request_id: int) -> None:
        p = self._registered.pop((kind, request_id), None)
        if p is not None:  # completion comes from the device, not from `time_s`
            self._inflight.append((kind, request_id, p))
            return
        super().schedule_event(time_s, kind, request_id)

    def run(self) -> SimResult:
        ex = self.async_executor
        devs = sorted({ex.device_of(g) for g in range(self.topology.total_gpus)})
        torch.cuda.synchronize()
        self.policy.attach(self)
        for rid in self._arrival_order:
            self.schedule_event(self.requests[rid].arrival_time * self.time_scale, EventKind.ARRIVAL, rid)
        dispatch = {
            EventKind.ARRIVAL: self._on_arrival,
            EventKind.STEP_COMPLETE: self._on_step,
            EventKind.DIT_COMPLETE: self._on_dit_complete,
            EventKind.VAE_COMPLETE: self._on_vae_complete,
        }
        t0 = time.perf_counter()
        ex.mark_clock_zero(devs)
        while self._heap or self._inflight:
            wall = time.perf_counter() - t0
            # completed device work, earliest device timestamp first
            done = []
            for item in self._inflight:
                if item[2].query():
                    done.append((ex.device_time(item[2]), item))
            cand = None
            if done:
                done.sort(key=lambda x: x[0])
                cand = ("dev", done[0][0], done[0][1])
            if self._heap and self._heap[0][0] <= wall and (cand is None or self._heap[0][0] <= cand[1]):
                t, _, kind, rid = heapq.heappop(self._heap)
                self.now = max(self.now, t)
                dispatch[kind](self.requests[rid])
                continue
            if cand is not None:
                _, t, item = cand
                self._inflight.remove(item)
                kind, rid, p = item
                self.device_seconds.append((kind.value, rid, p.device_seconds()))
                self.now = max(self.now, t)
                dispatch[kind](self.requests[rid])
                continue
            time.sleep(self.poll_s)
        undone = [r.request_id for r in self.requests.values() if r.status is not RequestStatus.DONE]
        if undone:
            raise RuntimeError(f"requests never finished: {undone}")
        from .sched.engine import RequestRecord

        recs = tuple(
            RequestRecord(s.request_id, s.resolution, s.arrival_time * self.time_scale, s.start_time,
                          s.finish_time, s.gpu_seconds, s.dop_history)
            for s in (self.requests[rid] for rid in self._arrival_order))
        return SimResult(recs, sum(r.gpu_seconds for r in recs), tuple(self._trace), self.policy.name)
