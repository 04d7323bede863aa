"""H9 plumbing on CPU: world_size-2 gloo process group, contiguous shards, all_gather of
makespans.  The per-shard solve here is the oracle (test scaffolding only — the product path
is far_solve_many on each rank's GPU, with NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_13601_b200 import dist as fdist
from paper_2507_13601_b200 import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    w = inputs.WORKLOADS["M3"]
    lo, hi = fdist.shard_range(total, rank, world)
    tab = w.table(count=hi - lo, start=lo)
    ms, _ = O.far_many(w.profile, w.costs(), tab)
    g = fdist.gather_makespans(torch.from_numpy(ms.astype(np.int32)), total)
    # packed schedules (8 B per task, the far_task_slot layout): node, size, pad, start
    sl = np.zeros((hi - lo, w.n, 8), np.uint8)
    for i in range(hi - lo):
        o = O.far(w.profile, w.costs(), tab[i])["slots"]
        sl[i, :, 0] = o["node"]
        sl[i, :, 1] = o["size_used"]
        sl[i, :, 4:] = o["start"].astype("<i4").view(np.uint8).reshape(-1, 4)
    gs = fdist.gather_schedules(torch.from_numpy(sl), total)
    if rank == 0:
        q.put((g.numpy().tolist(), gs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges():
    for total in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            rs = [fdist.shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(hi - lo <= fdist.padded_shard(total, world) for lo, hi in rs)


@pytest.mark.parametrize("total", [37, 64])
def test_gloo_allgather_world2(O, total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = inputs.WORKLOADS["M3"]
    tab = w.table(count=total)
    ref, _ = O.far_many(w.profile, w.costs(), tab)
    got_ms, got_sl = got
    assert got_ms == ref.tolist()
    assert got_sl.shape == (total, w.n, 8)
    for i in (0, total // 2, total - 1):  # the gathered schedules are the whole job's, in order
        o = O.far(w.profile, w.costs(), tab[i])["slots"]
        assert (got_sl[i, :, 0] == o["node"]).all() and (got_sl[i, :, 1] == o["size_used"]).all()
        assert (got_sl[i, :, 4:].copy().view("<i4")[:, 0] == o["start"]).all()
