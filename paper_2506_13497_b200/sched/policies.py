"""Scheduling policies: the greedy step-granularity DoP allocator and the static-DoP baseline.

Same decision rules as the reference (reference pkg/src/ditsim/policies.py):

* ``GreedyPolicy`` (:96-197): FCFS best-effort starts via ``try_best_alloc``; hungry requests
  (started below their optimal DoP B) sit in a promote table; whenever GPUs free up every
  entry first accrues starvation ``(cur_step - last_step) * (t(dop_now) - t(B))`` (paper
  Eq. 5, :69-85), then entries are served by (-starvation, arrival, id) (:88-93), each growing
  its *granted* handle (pending promotions stack) toward B; an entry reaching B leaves the
  table at once. At DiT completion an unapplied promotion is retracted and the request
  scales down to the ``vae_dop`` lowest-id GPUs (decoupled DiT/VAE, :175-190).
* ``StaticDopPolicy`` (:204-268): fixed DoP, FCFS, optional decoupled VAE.

The paper's cluster-partition baselines (SPCI/DPCI, :275-496) are out of scope: they are
offline comparison points with no data-path work.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .allocator import AllocationHandle
from .engine import RequestState, RequestStatus, Simulation, SimulationError
from .profiles import DopTable


class SchedulingPolicy:
    """Engine-driven hooks; the engine owns timing, the policy owns resources."""

    name: str = "base"
    decouple_vae: bool = False

    def attach(self, sim: Simulation) -> None:
        pass

    def on_arrival(self, sim: Simulation, request: RequestState) -> None:
        raise NotImplementedError

    def on_resources_freed(self, sim: Simulation) -> None:
        raise NotImplementedError

    def on_dit_complete(self, sim: Simulation, request: RequestState
                        ) -> tuple[AllocationHandle, tuple[int, ...]]:
        raise NotImplementedError

    def on_request_done(self, sim: Simulation, request: RequestState) -> tuple[int, ...]:
        raise NotImplementedError


@dataclass
class PromoteEntry:
    request: RequestState
    starvation: float = 0.0
    last_step: int = 0


def update_starvation(entry: PromoteEntry, cur_step: int, cur_step_seconds: float,
                      opt_step_seconds: float) -> float:
    entry.starvation += (cur_step - entry.last_step) * (cur_step_seconds - opt_step_seconds)
    entry.last_step = cur_step
    return entry.starvation


def promotion_order(entries: Sequence[PromoteEntry]) -> list[PromoteEntry]:
    return sorted(entries, key=lambda e: (-e.starvation, e.request.arrival_time,
                                          e.request.request_id))


def _release_all(sim: Simulation, request: RequestState) -> tuple[int, ...]:
    ids = request.gpus.gpu_ids
    sim.pool.release(request.gpus)
    return ids


class GreedyPolicy(SchedulingPolicy):
    decouple_vae = True

    def __init__(self, dop_table: DopTable, promotion: bool = True, name: str = ""):
        self.dop_table = dop_table
        self.promotion = promotion
        self.name = name or ("greedy" if promotion else "greedy-nopromo")
        self._waiting: list[RequestState] = []
        self._table: dict[int, PromoteEntry] = {}

    def attach(self, sim: Simulation) -> None:
        self._waiting.clear()
        self._table.clear()

    def on_arrival(self, sim: Simulation, request: RequestState) -> None:
        self._waiting.append(request)
        self._admit(sim)

    def _assert_table(self, sim: Simulation) -> None:
        hungry = {r.request_id for r in sim.requests.values() if r.status is RequestStatus.HUNGRY}
        assert hungry == set(self._table), (hungry, set(self._table))

    def on_resources_freed(self, sim: Simulation) -> None:
        if self.promotion:
            self._assert_table(sim)
            if self._table:
                self._promote(sim)
        self._admit(sim)

    def _promote(self, sim: Simulation) -> None:
        for e in self._table.values():
            update_starvation(e, e.request.cur_step, sim.current_step_seconds(e.request),
                              sim.optimal_step_seconds(e.request))
        for e in promotion_order(list(self._table.values())):
            req = e.request
            target = self.dop_table.dit_dop(req.resolution)
            held = req.granted
            assert held is not None and held.count < target
            grown = sim.pool.try_best_alloc(target, held, sim.profile.dop_candidates)
            if grown is held or grown.count <= held.count:
                continue
            sim.set_pending_promotion(req, grown)
            if grown.count == target:
                del self._table[req.request_id]
                req.status = RequestStatus.RUNNING

    def _admit(self, sim: Simulation) -> None:
        for req in list(self._waiting):
            target = self.dop_table.dit_dop(req.resolution)
            handle = sim.pool.try_best_alloc(target, None, sim.profile.dop_candidates)
            if handle is None:
                continue
            assert handle.count <= target
            self._waiting.remove(req)
            hungry = handle.count < target
            sim.start_dit(req, handle, hungry)
            if hungry and self.promotion:
                self._table[req.request_id] = PromoteEntry(req)

    def on_dit_complete(self, sim: Simulation, request: RequestState
                        ) -> tuple[AllocationHandle, tuple[int, ...]]:
        freed: list[int] = []
        if request.pending_promotion is not None:  # never reached a step boundary
            freed.extend(sim.pool.retract_to(request.pending_promotion, request.gpus))
            request.pending_promotion = None
        self._table.pop(request.request_id, None)
        keep = min(self.dop_table.vae_dop, request.gpus.count)
        kept, rest = sim.pool.release_keep_lowest(request.gpus, keep)
        freed.extend(rest)
        return kept, tuple(freed)

    def on_request_done(self, sim: Simulation, request: RequestState) -> tuple[int, ...]:
        return _release_all(sim, request)


class StaticDopPolicy(SchedulingPolicy):
    def __init__(self, dop: int, decouple_vae: bool = False, vae_dop: int = 1, name: str = ""):
        if dop < 1 or dop & (dop - 1):
            raise SimulationError(f"static DoP must be a power of two, got {dop}")
        self.dop = dop
        self.decouple_vae = decouple_vae
        self.vae_dop = vae_dop
        self.name = name or f"sdop{dop}{'-decoupled' if decouple_vae else ''}"
        self._waiting: list[RequestState] = []

    def attach(self, sim: Simulation) -> None:
        if self.dop not in sim.profile.dop_candidates:
            raise SimulationError(f"static DoP {self.dop} is not a profiled candidate")
        if self.dop > sim.topology.gpus_per_node:
            raise SimulationError(
                f"static DoP {self.dop} exceeds the node size {sim.topology.gpus_per_node}")
        self._waiting.clear()

    def on_arrival(self, sim: Simulation, request: RequestState) -> None:
        self._waiting.append(request)
        self._admit(sim)

    def on_resources_freed(self, sim: Simulation) -> None:
        self._admit(sim)

    def _admit(self, sim: Simulation) -> None:
        while self._waiting:
            handle = sim.pool.allocate_group(self.dop)
            if handle is None:
                return
            sim.start_dit(self._waiting.pop(0), handle, hungry=False)

    def on_dit_complete(self, sim: Simulation, request: RequestState
                        ) -> tuple[AllocationHandle, tuple[int, ...]]:
        if not self.decouple_vae:
            return request.gpus, ()
        return sim.pool.release_keep_lowest(request.gpus, min(self.vae_dop, request.gpus.count))

    def on_request_done(self, sim: Simulation, request: RequestState) -> tuple[int, ...]:
        return _release_all(sim, request)
