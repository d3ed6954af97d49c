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


def _part_worker(rank, world, port, q):
    """Host-side model of the row-partitioned exchange (comm.cu part_fetch)
    over gloo: the product's partition bounds (gx_partition_bounds, a host
    function), owner grouping by a stable sort, counts / ids / rows as variable
    all-to-alls, rows scattered back to their requests."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2208_09151_b200 as gx
    o = oracle.C
    N, dim = 5000, 8
    table = np.random.default_rng(1).random((N, dim)).astype(np.float32)
    lo, hi = gx.partition_bounds(N, world, rank)
    local = table[lo:hi]
    bounds = np.array([gx.partition_bounds(N, world, r)[0] for r in range(world)] + [N], np.int64)
    ip, ind = o.rmat_graph(N, 6.0, 3)
    plan = o.plan_seed_batches(o.train_ids(N, 1, 0.2), 25, o.epoch_seed(1, 0))
    S = 6
    sb = plan[rank * S:(rank + 1) * S]                      # this rank's superbatch
    trace = [o.sample_batch(ip, ind, b, [4, 3], o.derive_seed(1, rank * S + i))[0] for i, b in enumerate(sb)]
    req = np.concatenate(trace).astype(np.int64)           # requests, repeats across iterations
    owner = np.searchsorted(bounds, req, side="right") - 1
    perm = np.argsort(owner, kind="stable")
    send_ids = torch.from_numpy(req[perm] - bounds[owner[perm]])
    scnt = torch.from_numpy(np.bincount(owner, minlength=world).astype(np.int64))
    rcnt = torch.empty(world, dtype=torch.int64)
    dist.all_to_all_single(rcnt, scnt)
    recv_ids = torch.empty(int(rcnt.sum()), dtype=torch.int64)
    dist.all_to_all_single(recv_ids, send_ids, rcnt.tolist(), scnt.tolist())
    served = torch.from_numpy(np.ascontiguousarray(local[recv_ids.numpy()])).reshape(-1)
    back = torch.empty(len(req) * dim, dtype=torch.float32)
    dist.all_to_all_single(back, served, (scnt * dim).tolist(), (rcnt * dim).tolist())
    out = np.empty((len(req), dim), np.float32)
    out[perm] = back.numpy().reshape(-1, dim)
    q.put((rank, bool(np.array_equal(out, table[req])), int(rcnt.sum()), len(req),
           int(len(req) - scnt[rank])))
    dist.destroy_process_group()


def test_partitioned_exchange_protocol_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_part_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _, _ in res)
    assert sum(r[2] for r in res) == sum(r[3] for r in res)   # every request served exactly once
    assert all(r[4] > 0 for r in res)                          # rows did cross ranks


def test_superbatch_jobs_multi_epoch():
    """TrainingRunner::run (pipeline.hpp:212-228): each epoch's plan is cut
    into superbatches (short last one kept) and first_global_batch counts every
    earlier job's batches -- 7 batches per epoch at S = 3 give jobs of
    3, 3, 1 batches per epoch."""
    from paper_2208_09151_b200.shard import first_global_batch, superbatch_jobs
    jobs = superbatch_jobs([7, 7], 3)
    assert [(j.epoch, j.lo, j.hi, j.first_global_batch) for j in jobs] == [
        (0, 0, 3, 0), (0, 3, 6, 3), (0, 6, 7, 6), (1, 0, 3, 7), (1, 3, 6, 10), (1, 6, 7, 13)]
    assert [j.seq for j in jobs] == list(range(6))
    assert first_global_batch(4, 3, [7, 7]) == 10   # not 4 * 3
    assert first_global_batch(4, 3) == 12           # epoch-0-only form
