"""GPU: the row-partitioned CSC (include/gx_b200.h
gx_graph_partition / gx_graph_attach_*). Rank r keeps the in-neighbour lists of
an edge-balanced node range; the sampler loads other ranks' lists from their
HBM (CUDA IPC peer mappings; NVLink on a multi-GPU box). Sampled batches must
be bit-identical to the whole-CSC sampler and the oracle (sample_batch,
sampler.hpp:69-117), with the superbatch's batches split by rank
(shard.batch_block; seeds by global batch index, sampler.hpp:216).

* in-process: P ranks as P graphs of one process on one GPU (attach_local);
* two processes sharing the GPU: the handles go through torch.distributed
  (gloo) and are opened with cudaIpcOpenMemHandle -- the same code path the
  ranks of an 8-GPU box take (shard.partition_graph)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAN = [5, 4, 3]


@pytest.fixture(scope="module")
def data(oracle):
    n = 30000
    ip, ind = oracle.rmat_graph(n, 9.0, 17)
    train = oracle.train_ids(n, 1, 0.2)
    plan = oracle.plan_seed_batches(train, 150, oracle.epoch_seed(1, 0))[:10]
    return n, ip, ind, plan


def _same_samples(a, b, n_batches):
    for i in range(n_batches):
        x, y = a.batch(i), b.batch(i)
        assert np.array_equal(x.ids, y.ids), i
        for l in range(len(FAN)):
            assert np.array_equal(x.layers[l], y.layers[l]), (i, l)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_partitioned_sampler_in_process(gx, oracle, data, P):
    from paper_2208_09151_b200.shard import batch_block
    n, ip, ind, plan = data
    whole = gx.GraphFile.from_csc(ip, ind)
    bounds = whole.partition_bounds(P)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds.astype(np.int64)) >= 0)
    eb = ip[bounds.astype(np.int64)].astype(np.int64)           # lists are never split
    max_deg = int(np.diff(ip.astype(np.int64)).max())
    assert np.all(np.abs(np.diff(eb) - len(ind) / P) <= max_deg + 1)   # edge-balanced up to one list
    parts = [gx.GraphFile.from_csc(ip, ind).partition(P, q) for q in range(P)]
    for q in range(P):
        assert parts[q].partition_info() == (P, q, P == 1)
        assert np.array_equal(parts[q].partition_bounds(P), bounds)
    for q in range(P):
        parts[q].attach_local(parts)
    ref = gx.sample_superbatch(whole, None, plan, FAN, 1, 40)
    for q in range(P):
        blk = batch_block(len(plan), q, P)
        io_p, io_w = gx.IoStats(), gx.IoStats()
        mine = gx.sample_superbatch(parts[q], None, plan[blk.start:blk.stop], FAN, 1, 40 + blk.start, io_p)
        full = gx.sample_superbatch(whole, None, plan[blk.start:blk.stop], FAN, 1, 40 + blk.start, io_w)
        _same_samples(mine, full, len(blk))
        assert io_p == io_w
        for i in range(len(blk)):            # and the oracle, batch by batch
            ids, layers, _ = oracle.sample_batch(ip, ind, plan[blk.start + i], FAN,
                                                 oracle.derive_seed(1, 40 + blk.start + i))
            assert np.array_equal(mine.batch(i).ids, ids)
            assert np.array_equal(mine.batch(i).ids, ref.batch(blk.start + i).ids)


def test_partitioned_graph_refuses_whole_csc_calls(gx, data):
    n, ip, ind, plan = data
    g = gx.GraphFile.from_csc(ip, ind).partition(2, 1)
    with pytest.raises(gx.LogicError):
        gx.sample_superbatch(g, None, plan[:2], FAN, 1, 0)      # peers not attached yet
    with pytest.raises(gx.LogicError):
        g.to_csc()
    with pytest.raises(gx.LogicError):
        g.partition(2, 0)
    with pytest.raises(gx.LogicError):
        gx.NeighborCache.build(g, n * 8 + 4096)
    with pytest.raises(ValueError):
        gx.GraphFile.from_csc(ip, ind).partition(2, 2)
    other = gx.GraphFile.from_csc(ip, ind).partition(3, 0)
    with pytest.raises(ValueError):
        g.attach_local([other, g])


def test_partitioned_pipeline_matches_oracle(gx, oracle, data):
    """The fused pipeline on rank q's partitioned graph with rank q's batch
    block: misses equal the oracle's Belady simulation of that block and the
    gathered rows are the block's feature rows."""
    from paper_2208_09151_b200.shard import batch_block
    n, ip, ind, plan = data
    P, K = 3, 2500
    rows = oracle.features(n, 16, 5)
    f = gx.FeatureFile.from_array(rows)
    parts = [gx.GraphFile.from_csc(ip, ind).partition(P, q) for q in range(P)]
    for q in range(P):
        parts[q].attach_local(parts)
    for q in range(P):
        blk = batch_block(len(plan), q, P)
        p = gx.Pipeline(parts[q], f, FAN, K, digest=True)
        st = p.run_superbatch(plan[blk.start:blk.stop], 1, blk.start)
        trace = [oracle.sample_batch(ip, ind, plan[blk.start + i], FAN, oracle.derive_seed(1, blk.start + i))[0]
                 for i in range(len(blk))]
        sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
        assert np.array_equal(st.misses, sim["misses"])
        for i in range(len(blk)):
            assert np.array_equal(p.batch(i), rows[trace[i].astype(np.int64)])


WORKER = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["GX_ROOT"])
import torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
import oracle
import paper_2208_09151_b200 as gx
from paper_2208_09151_b200.shard import batch_block, partition_graph
o = oracle.C
n = 30000
ip, ind = o.rmat_graph(n, 9.0, 17)
plan = o.plan_seed_batches(o.train_ids(n, 1, 0.2), 150, o.epoch_seed(1, 0))[:10]
g = gx.GraphFile.from_csc(ip, ind)
partition_graph(g, rank, world)
blk = batch_block(len(plan), rank, world)
s = gx.sample_superbatch(g, None, plan[blk.start:blk.stop], [5, 4, 3], 1, blk.start)
ok = True
for i in range(len(blk)):
    ids, layers, _ = o.sample_batch(ip, ind, plan[blk.start + i], [5, 4, 3], o.derive_seed(1, blk.start + i))
    b = s.batch(i)
    ok &= bool(np.array_equal(b.ids, ids)) and all(np.array_equal(b.layers[l], layers[l]) for l in range(3))
dist.barrier()   # peers keep their partitions mapped until everyone is done
print(json.dumps({"rank": rank, "ok": ok, "batches": len(blk), "info": list(g.partition_info())}))
dist.destroy_process_group()
"""


def test_partitioned_sampler_two_processes(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(2):
        env = dict(os.environ, GX_ROOT=ROOT, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, cwd=ROOT,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o + e
    res = sorted((json.loads(o.strip().splitlines()[-1]) for o, _ in outs), key=lambda r: r["rank"])
    assert [r["rank"] for r in res] == [0, 1]
    assert all(r["ok"] for r in res), res
    assert sum(r["batches"] for r in res) == 10
    assert all(r["info"] == [2, r["rank"], True] for r in res)
