"""``B200ProfileTable``: the reference's ``ProfileTable`` duck type with real B200 work behind it.

The unmodified reference serving loop (``ditsim.Simulation``) reaches GPU work only through two
lookups on the profile object it is given:

* ``profile.dit_step(resolution, dop)`` -- reference pkg/src/ditsim/profiles.py:69-76, called by
  the engine at ``start_dit`` (engine.py:245), after a promotion (:289), in steady state (:292),
  and, as pure lookups for the starvation order, by ``current_step_seconds`` /
  ``optimal_step_seconds`` (:228, :231);
* ``profile.vae(resolution, dop)`` -- profiles.py:78-85, called at ``_handle_dit_complete``
  (engine.py:305).

``B200ProfileTable`` answers both from a measured ``dit-profile/1`` table and, at the three
execution sites and the VAE site, additionally executes the request's real step (or hand-off +
VAE decode) on the B200 through ``executor.B200Executor`` -- the same calls our own engine makes
with ``Simulation(..., executor=...)``. The execution site and its request are identified from
the caller's frame (the engine passes only ``(resolution, dop)``), so ``ditsim`` needs no change.

Clock modes:

* ``"profiled"`` (default): the engine is charged the table's seconds, so every allocator /
  policy decision is exactly the virtual-time run's on that table, while the B200 really runs
  each step in that order; ``measured`` records what each call took on the device.
* ``"measured"``: the engine is charged the measured device seconds (a real-time replay driven by
  the unmodified reference loop).

Lookups that are not execution sites (starvation, ``estimate_execution_time``, ``optimal_dop``)
always return the table value, as in the reference.
"""

from __future__ import annotations

import sys
from dataclasses import dataclass
from typing import Any

_STEP_SITES = {"start_dit": "start", "_handle_step_complete": "step"}
_VAE_SITES = {"_handle_dit_complete"}


@dataclass(frozen=True)
class Executed:
    """One real call made behind the duck type."""

    kind: str  # "start" | "step" | "promotion" | "vae"
    request_id: int
    resolution: str
    gpu_ids: tuple[int, ...]
    step: int
    table_seconds: float
    measured_seconds: float


class B200ProfileTable:
    """Duck-typed ``ProfileTable`` (reference profiles.py:48-90) that runs real B200 steps.

    ``table``: a ``ProfileTable`` (ours or the reference's) holding the measured times.
    ``executor``: a ``B200Executor`` (or anything with its ``dit_step`` / ``vae`` protocol).
    """

    def __init__(self, table: Any, executor: Any, mode: str = "profiled"):
        if mode not in ("profiled", "measured"):
            raise ValueError(f"mode must be 'profiled' or 'measured', got {mode!r}")
        self._table = table
        self.executor = executor
        self.mode = mode
        # the frozen ProfileTable fields, so helpers that read them (derive_dop_table,
        # dump_profiles, solve_optimal) see the measured table
        self.resolutions = table.resolutions
        self.dop_candidates = table.dop_candidates
        self.dit_step_time = table.dit_step_time
        self.vae_time = table.vae_time
        self.executed: list[Executed] = []
        self._groups: dict[int, tuple[int, ...]] = {}

    # ---- the lookups (unchanged semantics, errors included)
    def resolution(self, name: str):
        return self._table.resolution(name)

    def has_resolution(self, name: str) -> bool:
        return self._table.has_resolution(name)

    def profiled_dops(self, resolution: str) -> tuple[int, ...]:
        return self._table.profiled_dops(resolution)

    # ---- the two call sites with work behind them
    def dit_step(self, resolution: str, dop: int) -> float:
        t = self._table.dit_step(resolution, dop)  # ProfileLookupError exactly as the reference
        frame = sys._getframe(1)
        site = _STEP_SITES.get(frame.f_code.co_name)
        req = frame.f_locals.get("request") if site else None
        if req is None or getattr(req, "gpus", None) is None:
            return t  # a starvation / planning lookup
        ids = tuple(req.gpus.gpu_ids)
        prev = self._groups.get(req.request_id)
        resharded = prev if (prev is not None and prev != ids) else None
        # start_dit runs step 0; at a step boundary cur_step is the index of the step to run
        step = 0 if site == "start" else req.cur_step
        secs = self.executor.dit_step(req, ids, step, resharded)
        self._groups[req.request_id] = ids
        kind = "promotion" if resharded is not None else site
        self.executed.append(Executed(kind, req.request_id, resolution, ids, step, t, secs))
        return secs if self.mode == "measured" else t

    def vae(self, resolution: str, dop: int = 1) -> float:
        t = self._table.vae(resolution, dop)
        frame = sys._getframe(1)
        if frame.f_code.co_name not in _VAE_SITES:
            return t
        req = frame.f_locals.get("request")
        retained = frame.f_locals.get("retained")
        if req is None or retained is None or req.request_id not in self._groups:
            return t
        dit_ids = self._groups.pop(req.request_id)
        secs = self.executor.vae(req, dit_ids, tuple(retained.gpu_ids))
        self.executed.append(Executed("vae", req.request_id, resolution, tuple(retained.gpu_ids),
                                      -1, t, secs))
        return secs if self.mode == "measured" else t

    # ---- summaries
    def measured_seconds(self) -> dict[str, float]:
        """Total measured device seconds per kind of call."""
        out: dict[str, float] = {}
        for e in self.executed:
            out[e.kind] = out.get(e.kind, 0.0) + e.measured_seconds
        return out
