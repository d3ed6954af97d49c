"""GPU parity of the row-partitioned feature table (comm.cu).

P ranks run on P host threads with the in-process transport (one B200 here),
each with its own context, pipeline and superbatches; the feature table is
split [N*r/P, N*(r+1)/P) across them and every row a rank's cache needs from
another rank crosses the variable all-to-all. Each rank's results must equal
the oracle on that rank's own trace (Belady changesets are per rank, §8e
"Inspector: replicas only") and its gathered bytes the table's rows. One world-1
NCCL communicator exercises the real NCCL send/recv path.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(P, fn):
    """fn(rank) on P threads; re-raise the first failure (with a timeout so a
    broken exchange cannot hang the suite)."""
    errs = [None] * P
    out = [None] * P

    def wrap(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=wrap, args=(r,), daemon=True) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for e in errs:   # a failing rank aborts the hub, so its error is the one to report
        if e is not None and "exchange aborted" not in str(e):
            raise e
    for e in errs:
        if e is not None:
            raise e
    assert all(not t.is_alive() for t in ts), "rank thread hung"
    return out


def test_partition_bounds(gx):
    for N, P in [(10, 3), (111_059_956, 8), (5, 8), (1, 1)]:
        b = [gx.partition_bounds(N, P, r) for r in range(P)]
        assert b[0][0] == 0 and b[-1][1] == N
        assert all(b[r][1] == b[r + 1][0] for r in range(P - 1))
        assert all(b[r] == (N * r // P, N * (r + 1) // P) for r in range(P))


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("K", [250, 4000])       # misses every iteration / all-fit
def test_partitioned_pipeline_matches_oracle(gx, oracle, P, K):
    n, dim = 5000, 40
    ip, ind = oracle.rmat_graph(n, 6.0, 31)
    rows = oracle.features(n, dim, 32)
    train = oracle.train_ids(n, 1, 0.3)
    plan = oracle.plan_seed_batches(train, 40, oracle.epoch_seed(1, 0))
    S = 6
    sbs = [plan[o:o + S] for o in range(0, len(plan), S)][:2 * P]
    ctxs = [gx.Context(0) for _ in range(P)]
    comms = gx.Comm.local(ctxs)

    def rank(r):
        lo, hi = gx.partition_bounds(n, P, r)
        g = gx.GraphFile.from_csc(ip, ind, ctx=ctxs[r])
        f = gx.FeatureFile.partitioned_from_array(rows[lo:hi], n, comms[r])
        p = gx.Pipeline(g, f, [5, 3], K, digest=True)
        res = []
        for k in range(2):  # superbatches r, r + P (shard.py assignment)
            j = r + k * P
            st = p.run_superbatch(sbs[j], 1, j * S)
            res.append((j, st, p.digests(), [p.batch(i) for i in range(len(sbs[j]))]))
        return res, f.exchange_stats()

    outs = _run_ranks(P, rank)
    for r, (res, xs) in enumerate(outs):
        for j, st, dig, batches in res:
            trace = [oracle.sample_batch(ip, ind, b, [5, 3], oracle.derive_seed(1, j * S + i))[0]
                     for i, b in enumerate(sbs[j])]
            sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
            assert np.array_equal(st.misses, sim["misses"]), (r, j)
            assert st.total_misses == st.predicted_misses
            assert st.storage_rows == st.init_size + st.total_misses
            for i, ids in enumerate(trace):
                want = rows[ids.astype(np.int64)]
                assert np.array_equal(batches[i], want), (r, j, i)
                assert int(dig[i]) == gx.batch_digest(want)
        assert xs.calls == 4                       # 2 superbatches x (init + misses)
        assert xs.rows_remote > 0 and xs.rows_remote <= xs.rows_requested
    # every requested row was served by exactly one owner
    assert sum(x.rows_requested for _, x in outs) == sum(x.rows_served for _, x in outs)


def test_partitioned_cache_api(gx, oracle):
    """FeatureCache ctor / gather / apply over a partitioned store (collective calls)."""
    P, n, dim, K = 2, 3000, 24, 400
    rows = np.random.default_rng(5).random((n, dim)).astype(np.float32)
    ctxs = [gx.Context(0) for _ in range(P)]
    comms = gx.Comm.local(ctxs)
    rng = np.random.default_rng(9)
    inits = [rng.choice(n, 300, replace=False).astype(np.uint64) for _ in range(P)]
    reqs = [[rng.choice(n, 500, replace=False).astype(np.uint64) for _ in range(3)] for _ in range(P)]
    reqs[1][1] = np.zeros(0, np.uint64)           # an empty request set still joins the exchange

    def rank(r):
        lo, hi = gx.partition_bounds(n, P, r)
        f = gx.FeatureFile.partitioned_from_array(rows[lo:hi], n, comms[r])
        io = gx.IoStats()
        c = gx.FeatureCache(f, inits[r], K, io)
        out = [io]
        for ids in reqs[r]:
            b, cnt = c.gather(f, ids, io)
            out.append((b.numpy(), cnt.hits, cnt.misses))
        return out

    outs = _run_ranks(P, rank)
    for r in range(P):
        oc = oracle.cache(rows, inits[r], K)
        io = outs[r][0]
        for k, ids in enumerate(reqs[r]):
            got, h, m = outs[r][1 + k]
            want, wh, wm, _ = oc.gather(ids)
            assert np.array_equal(got, want) and (h, m) == (wh, wm)
        assert io.rows_read == 300 + sum(outs[r][1 + k][2] for k in range(3))


def test_generate_partitioned_and_fp16(gx, oracle):
    n, dim = 1000, 12
    full = oracle.features(n, dim, 77)
    ctxs = [gx.Context(0) for _ in range(3)]
    comms = gx.Comm.local(ctxs)

    def rank(r):
        f = gx.FeatureFile.partitioned_generate(n, dim, 77, comms[r])
        c = gx.FeatureCache(f, np.arange(r * 100, r * 100 + 50, dtype=np.uint64), 64)
        b, cnt = c.gather(f, np.arange(n - 50, n, dtype=np.uint64))
        return b.numpy()

    outs = _run_ranks(3, rank)
    for r in range(3):
        assert np.array_equal(outs[r], full[n - 50:])
    f16 = gx.FeatureFile.generate(n, 768, 5, dtype=np.float16)
    assert f16.row_bytes() == 1536 and f16.dtype == np.float16
    want = oracle.features(n, 768, 5).astype(np.float16)  # numpy float32->float16 is round-to-nearest-even
    ids = np.array([0, 1, 999, 500], np.uint64)
    assert np.array_equal(f16.read_rows(ids), want[ids.astype(np.int64)])


def test_nccl_world1_matches_device_backing(gx, oracle):
    """The real NCCL transport (self send/recv) behind the pipeline."""
    n, dim, K = 4000, 32, 600
    ip, ind = oracle.rmat_graph(n, 6.0, 41)
    rows = oracle.features(n, dim, 42)
    ctx = gx.Context(0)
    comm = gx.Comm.nccl(ctx, gx.Comm.unique_id(), 1, 0)
    g = gx.GraphFile.from_csc(ip, ind, ctx=ctx)
    fp = gx.FeatureFile.partitioned_from_array(rows, n, comm)
    fd = gx.FeatureFile.from_array(rows, ctx=ctx)
    train = oracle.train_ids(n, 1, 0.3)
    plan = oracle.plan_seed_batches(train, 40, oracle.epoch_seed(1, 0))[:8]
    pp = gx.Pipeline(g, fp, [5, 3], K, digest=True)
    pd = gx.Pipeline(g, fd, [5, 3], K, digest=True)
    a = pp.run_superbatch(plan, 1, 0)
    da = pp.digests()
    b = pd.run_superbatch(plan, 1, 0)
    assert np.array_equal(a.misses, b.misses) and np.array_equal(da, pd.digests())
    assert a.gather_io == b.gather_io
    xs = fp.exchange_stats()
    assert xs.calls == 2 and xs.rows_remote == 0 and xs.rows_requested == a.init_size + a.total_misses


MP_WORKER = r"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["GX_ROOT"])
import torch.distributed as dist
rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
import oracle
import paper_2208_09151_b200 as gx
from paper_2208_09151_b200.shard import partition_graph
o = oracle.C
n, dim, K, S = 5000, 40, int(os.environ["GX_K"]), 6
ip, ind = o.rmat_graph(n, 6.0, 31)
rows = o.features(n, dim, 32)
plan = o.plan_seed_batches(o.train_ids(n, 1, 0.3), 40, o.epoch_seed(1, 0))
sbs = [plan[q:q + S] for q in range(0, len(plan), S)]
ctx = gx.Context(0)
comm = gx.Comm.host(ctx, P, rank)
lo, hi = gx.partition_bounds(n, P, rank)
g = partition_graph(gx.GraphFile.from_csc(ip, ind, ctx=ctx), rank, P)
f = gx.FeatureFile.partitioned_from_array(rows[lo:hi], n, comm)
p = gx.Pipeline(g, f, [5, 3], K, digest=True)
ok = True
for k in range(2):                      # superbatches rank, rank + P
    j = rank + k * P
    st = p.run_superbatch(sbs[j], 1, j * S)
    trace = [o.sample_batch(ip, ind, b, [5, 3], o.derive_seed(1, j * S + i))[0] for i, b in enumerate(sbs[j])]
    sim = o.simulate(trace, n, K, o.compute_init_set(trace, K, n))
    ok &= bool(np.array_equal(st.misses, sim["misses"])) and st.storage_rows == st.init_size + st.total_misses
    for i, ids in enumerate(trace):
        ok &= bool(np.array_equal(p.batch(i), rows[ids.astype(np.int64)]))
xs = f.exchange_stats()
dist.barrier()
print(json.dumps({"rank": rank, "ok": ok, "calls": xs.calls, "remote": xs.rows_remote,
                  "requested": xs.rows_requested, "served": xs.rows_served}))
dist.destroy_process_group()
"""


@pytest.mark.parametrize("K", [250, 4000])
def test_partitioned_table_two_processes_host_transport(K):
    """Two processes on the one GPU: row-partitioned table exchanged through
    the host-staged transport (gx_comm_init_host, gloo all_to_all_single) and
    the row-partitioned CSC mapped over CUDA IPC -- the product's grouping,
    owner gathers and scatters with real process separation."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [subprocess.Popen([sys.executable, "-c", MP_WORKER], cwd=root, text=True,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              env=dict(os.environ, GX_ROOT=root, RANK=str(r), WORLD_SIZE="2", GX_K=str(K),
                                       MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PYTHONPATH=root))
             for r in range(2)]
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o + e
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    assert all(r["ok"] for r in res), res
    assert all(r["calls"] == 4 and 0 < r["remote"] <= r["requested"] for r in res), res
    assert sum(r["requested"] for r in res) == sum(r["served"] for r in res)
