"""One process per GPU: a DoP-P group of ranks running one request's step together.

torch.distributed is only the rendezvous (exchanging 64-byte CUDA IPC handles); the
sequence-parallel all-to-all itself runs inside libddit as peer stores over NVLink into
the other ranks' mapped buffers, closed by a flag barrier (csrc/exchange.cu). Reference
counterpart: the paper's NCCL data plane between engine units; the
reference simulator models it only as the dit_step(res, dop) curve (profiles.py:69-76).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ._lib import check, lib
from .stdit import STDiTModel, StepRequest


def ipc_export(ptr: int) -> tuple[bytes, int]:
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    check(lib().ddit_ipc_export(ptr, h, ctypes.byref(off)))
    return bytes(h.raw), off.value


def ipc_import(handle: bytes, offset: int) -> int:
    out = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(handle, 64)
    check(lib().ddit_ipc_import(buf, offset, ctypes.byref(out)))
    return out.value


def assemble_peer_table(rank: int, dop: int, local: tuple[int, int, int], gathered: list,
                        importer=None) -> tuple[list[list[int]], list[int]]:
    """Per-rank pointer table of the three exchange buffers (x_sp, x_tp, flags).

    ``gathered[q]`` = rank q's [(ipc_handle, offset)] * 3. Own buffers are used directly;
    every distinct peer allocation is mapped once (``importer(handle) -> base``) and the
    three pointers are base + offset. Returns (columns, imported bases)."""
    importer = importer or (lambda h: ipc_import(h, 0))
    imported: list[int] = []
    cols: list[list[int]] = [[], [], []]
    for q in range(dop):
        bases: dict[bytes, int] = {}
        for j in range(3):
            if q == rank:
                cols[j].append(local[j])
                continue
            h, off = gathered[q][j]
            if h not in bases:
                bases[h] = importer(h)
                imported.append(bases[h])
            cols[j].append(bases[h] + off)
    return cols, imported


class GroupStep:
    """This process's rank of a DoP-``world_size`` group (``group`` or the default group)."""

    def __init__(self, model: STDiTModel, shape, y_cond, group=None, **kw):
        self.rank = dist.get_rank(group)
        self.dop = dist.get_world_size(group)
        self.req = StepRequest(model, shape, y_cond, dop=self.dop, rank=self.rank, **kw)
        local = self.req.exchange_buffers()
        mine = [ipc_export(p) for p in local]
        allh: list = [None] * self.dop
        dist.all_gather_object(allh, mine, group=group)
        cols, self._imported = assemble_peer_table(self.rank, self.dop, local, allh)
        self.req.set_peers(cols[0], cols[1], cols[2])
        torch.cuda.synchronize()
        dist.barrier(group=group)

    @property
    def shard(self):
        return self.req.shard

    def step(self, z_local: torch.Tensor, step: int, stream=None) -> torch.Tensor:
        return self.req.step(z_local, step, stream)

    def close(self) -> None:
        for p in self._imported:
            lib().ddit_ipc_close(p, 0)
        self._imported = []
        self.req.close()


class NcclGroupStep:
    """The NCCL arm of the DSP exchange (the baseline the fused peer-store exchange must beat):
    this process's rank of a DoP-``world_size`` group whose all-to-all between the spatial and
    temporal layouts is ``ncclAllToAll`` (torch.distributed ``all_to_all_single`` with per-rank
    splits, backend "nccl") on packed fp32 rows: after every phase the rank packs its outgoing
    rows per destination (``ddit_request_xch_pack``), the collective moves them, and the rank
    unpacks the rows it received (``ddit_request_xch_unpack``). Reference counterpart: the
    paper's NCCL data plane; the reference simulator only charges a
    constant (engine.py:286-290). ``a2a_ms`` accumulates CUDA-event time of the collectives when
    ``timing`` is on."""

    def __init__(self, model: STDiTModel, shape, y_cond, group=None, timing: bool = False, **kw):
        from .stdit import DDIT_OPT_EXTERNAL_XCH

        self.group = group
        self.rank = dist.get_rank(group)
        self.dop = dist.get_world_size(group)
        self.req = StepRequest(model, shape, y_cond, dop=self.dop, rank=self.rank, **kw)
        self.req.set_option(DDIT_OPT_EXTERNAL_XCH, 1)
        self.depth = model.cfg.depth
        self.C = model.cfg.hidden
        self.counts = [self.req.xch_counts(d) for d in (0, 1)]
        rows = max(max(sum(c[0]), sum(c[1])) for c in self.counts)
        self.send = torch.empty((max(rows, 1), self.C), device=model.device)
        self.recv = torch.empty((max(rows, 1), self.C), device=model.device)
        self.timing = timing
        self.a2a_ms = 0.0
        self.a2a_bytes = 0
        self._ev = []

    @property
    def shard(self):
        return self.req.shard

    def bytes_per_step(self) -> int:
        """fp32 bytes this rank sends to other ranks in one step (own block excluded)."""
        tot = 0
        for d in (0, 1):
            snd = self.counts[d][0]
            tot += self.depth * (sum(snd) - snd[self.rank]) * self.C * 4
        return tot

    def step(self, z_local: torch.Tensor, step: int, stream=None) -> torch.Tensor:
        req = self.req
        req.begin(z_local, step, stream)
        for k in range(2 * self.depth):
            req.phase(k, stream)
            snd, rcv = self.counts[k & 1]
            req.xch_pack(k, self.send, stream)
            if self.timing:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
            dist.all_to_all_single(self.recv[:sum(rcv)], self.send[:sum(snd)],
                                   output_split_sizes=rcv, input_split_sizes=snd, group=self.group)
            if self.timing:
                b.record()
                self._ev.append((a, b))
            req.xch_unpack(k, self.recv, stream)
        req.end(z_local, step, stream)
        return z_local

    def read_timing(self) -> float:
        """ms of all-to-all collectives since the last read (synchronises)."""
        ms = 0.0
        for a, b in self._ev:
            b.synchronize()
            ms += a.elapsed_time(b)
        self._ev = []
        self.a2a_ms += ms
        return ms

    def close(self) -> None:
        self.req.close()
