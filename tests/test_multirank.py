"""CPU suite: the N>1 path (paper_2208_09151_b200/shard.py) with world_size 2
over gloo. Each rank runs its superbatches through the oracle (the device is
not needed to check the sharding logic); the union over ranks must equal the
single-process run and the reduced statistics must match."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _superbatch_edges(o, ip, ind, sbs, j, S):
    from paper_2208_09151_b200.shard import first_global_batch
    tot = 0
    for i, b in enumerate(sbs[j]):
        _, layers, _ = o.sample_batch(ip, ind, b, [4, 4], o.derive_seed(1, first_global_batch(j, S) + i))
        tot += sum(len(l) for l in layers)
    return tot


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2208_09151_b200.shard import assign_superbatches, reduce_stats
    o = oracle.C
    ip, ind = o.rmat_graph(4000, 6.0, 3)
    plan = o.plan_seed_batches(o.train_ids(4000, 1, 0.1), 20, o.epoch_seed(1, 0))
    S = 4
    sbs = [plan[k:k + S] for k in range(0, len(plan), S)]
    mine = assign_superbatches(len(sbs), rank, world, steps=2)
    edges = sum(_superbatch_edges(o, ip, ind, sbs, j, S) for j in mine)
    tot, mx = reduce_stats([edges, float(rank + 1)], ["sum", "max"])
    q.put((rank, mine, edges, tot, mx))
    dist.destroy_process_group()


def test_two_rank_sharding_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2208_09151_b200.shard import assign_superbatches
    o = oracle.C
    ip, ind = o.rmat_graph(4000, 6.0, 3)
    plan = o.plan_seed_batches(o.train_ids(4000, 1, 0.1), 20, o.epoch_seed(1, 0))
    S = 4
    sbs = [plan[k:k + S] for k in range(0, len(plan), S)]
    # disjoint assignment covering the first 2*world superbatches
    got = sorted(j for _, mine, *_ in res for j in mine)
    assert got == [0, 1, 2, 3]
    single = sum(_superbatch_edges(o, ip, ind, sbs, j, S) for j in range(4))
    assert res[0][3] == res[1][3] == single       # sum-reduced edges == single process
    assert res[0][4] == res[1][4] == 2.0          # max-reduced
    assert res[0][2] + res[1][2] == single


def test_assignment_validation():
    sys.path.insert(0, ROOT)
    from paper_2208_09151_b200.shard import assign_superbatches
    assert assign_superbatches(10, 1, 4, 3) == [1, 5, 9]
    with pytest.raises(ValueError):
        assign_superbatches(10, 4, 4, 1)
    with pytest.raises(ValueError):
        assign_superbatches(0, 0, 1, 1)
