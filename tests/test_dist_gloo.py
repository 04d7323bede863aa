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
    if rank == 0:
        q.put(g.numpy().tolist())
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
    ref, _ = O.far_many(w.profile, w.costs(), w.table(count=total))
    assert got == ref.tolist()
