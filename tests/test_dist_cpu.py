"""N>1 host logic on CPU with world_size-2 (and 4) gloo groups: shard assignment per rank,
the IPC-handle exchange / peer-table assembly, and a numpy re-enactment of the DSP
all-to-all (every rank's temporal shard assembled from the others' spatial shards)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import shard_ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_13497_b200 import shapes
        from paper_2506_13497_b200.dist import assemble_peer_table

        # 1) peer table from fake IPC handles: one allocation per rank at base 1000*(q+1)
        local = (1000 * (rank + 1) + 0, 1000 * (rank + 1) + 64, 1000 * (rank + 1) + 512)
        mine = [(bytes([rank]) * 64, off) for off in (0, 64, 512)]
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        fake_base = {bytes([r]) * 64: 1000 * (r + 1) for r in range(world)}
        cols, imported = assemble_peer_table(rank, world, local, allh, fake_base.__getitem__)
        ok_table = all(cols[j][qq] == 1000 * (qq + 1) + (0, 64, 512)[j]
                       for j in range(3) for qq in range(world)) and len(imported) == world - 1

        # 2) DSP exchange re-enacted with gloo: x_sp shard -> all ranks -> x_tp shard
        B, T, S, C = 2, 15, 37, 3
        sh_T = shapes.shard_range(T, world, rank)
        x_full = torch.arange(B * T * S * C, dtype=torch.float64).view(B, T, S, C)
        x_sp = x_full[:, sh_T[0]:sh_T[1]].contiguous()
        parts = [None] * world
        dist.all_gather_object(parts, x_sp)
        s_lo, s_hi = shapes.shard_range(S, world, rank)
        x_tp = torch.cat(parts, dim=1)[:, :, s_lo:s_hi]
        want_tokens = shard_ref.temporal_tokens(B, T, S, world, rank)
        got_tokens = (x_tp[..., 0] / C).reshape(-1).long().numpy()
        ok_x = np.array_equal(want_tokens, got_tokens)

        # 3) max-over-ranks timing as bench.py does it
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok_max = t.item() == world
        q.put((rank, ok_table, ok_x, ok_max))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_group_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, a, b, c in res:
        assert a and b and c, (rank, a, b, c)
