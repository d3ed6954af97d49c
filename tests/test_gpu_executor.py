"""GPU parity: the HBM feature cache (executor.cu) vs the C oracle restatement
of FeatureCache (feature_cache.hpp:19-130) and the reference's KATs
(test_feature_cache.cpp); plus the fused pipeline end to end."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _feat(n, dim, seed, dtype=np.float32):
    rng = np.random.default_rng(seed)
    return rng.random((n, dim)).astype(dtype)


def test_init_gather_kats(gx, oracle):
    rows = _feat(20, 8, 1)
    f = gx.FeatureFile.from_array(rows)
    io = gx.IoStats()
    c = gx.FeatureCache(f, [], 4, io)
    assert not any(c.contains(v) for v in range(20)) and io.rows_read == 0
    c = gx.FeatureCache(f, [4, 1, 2], 4, io)
    assert c.contains(4) and c.contains(1) and c.contains(2) and not c.contains(0)
    assert np.array_equal(c.cached_row(4), rows[4])
    with pytest.raises(ValueError):
        gx.FeatureCache(f, [0, 1, 2], 2)
    with pytest.raises(ValueError):
        gx.FeatureCache(f, [1, 1], 4)
    with pytest.raises(IndexError):
        gx.FeatureCache(f, [25], 4)
    # straddling rows: 1200-byte rows, prefetch pages = per-row page sum
    odd = gx.FeatureFile.from_array(_feat(40, 300, 2))
    io = gx.IoStats()
    gx.FeatureCache(odd, [0, 3, 17, 33, 39], 8, io)
    assert io.pages_read == sum(oracle.page_count_for_row(1200, v) for v in [0, 3, 17, 33, 39])
    assert io.rows_read == 5


def test_gather_apply_kats(gx):
    rows = _feat(10, 6, 3)
    f = gx.FeatureFile.from_array(rows)
    c = gx.FeatureCache(f, [0, 1, 4, 6, 7], 5)
    ids = [0, 2, 5, 7]
    io = gx.IoStats()
    b, cnt = c.gather(f, ids, io)
    assert (cnt.hits, cnt.misses, io.rows_read) == (2, 2, 2)
    assert np.array_equal(b.numpy(), rows[ids])
    b2, cnt2 = c.gather(f, [7, 4, 0], gx.IoStats())
    assert cnt2.misses == 0
    with pytest.raises(IndexError):
        c.gather(f, [11])
    # error paths (test_feature_cache.cpp:153-173), before any mutation
    with pytest.raises(gx.LogicError):
        c.apply_changeset(b, ids, gx.Changeset([0], [], [0]))
    with pytest.raises(gx.LogicError):
        c.apply_changeset(b, ids, gx.Changeset([], [5], []))
    with pytest.raises(gx.LogicError):
        c.apply_changeset(b, ids, gx.Changeset([5], [], [1]))
    with pytest.raises(gx.LogicError):
        c.apply_changeset(b, ids, gx.Changeset([2], [], [1]))
    c.apply_changeset(b, ids, gx.Changeset([2, 5], [0, 6], [1, 2]))
    assert not c.contains(0) and not c.contains(6)
    assert np.array_equal(c.cached_row(2), rows[2]) and np.array_equal(c.cached_row(5), rows[5])
    assert list(c.resident_set()) == [1, 2, 4, 5, 7]
    # under-full cache draws slots from the free list
    small = gx.FeatureCache(f, [], 3)
    b3, _ = small.gather(f, [9, 3])
    small.apply_changeset(b3, [9, 3], gx.Changeset([9], [], [0]))
    assert small.contains(9) and np.array_equal(small.cached_row(9), rows[9])


@pytest.mark.parametrize("dim,dtype", [(5, np.float32), (128, np.float32), (300, np.float32),
                                       (64, np.float16), (768, np.float16)])
def test_replay_matches_oracle(gx, oracle, dim, dtype):
    """Live replay of simulated changesets (test_feature_cache.cpp:176-221,
    acceptance c9): gathered bytes, counts, IoStats and slot layout all match."""
    n = 400
    rows = _feat(n, dim, 9, dtype)
    f = gx.FeatureFile.from_array(rows)
    rng = np.random.default_rng(41)
    trace = [np.sort(rng.choice(n, size=int(rng.integers(1, 60)), replace=False)).astype(np.uint64)
             for _ in range(25)]
    for K in (2, 7, 20, 150):
        init = oracle.compute_init_set(trace, K, n)
        sim = oracle.simulate(trace, n, K, init)
        c = gx.FeatureCache(f, init, K)
        oc = oracle.cache(rows, init, K)
        for i, ids in enumerate(trace):
            io = gx.IoStats()
            b, cnt = c.gather(f, ids, io)
            ob, oh, om, oio = oc.gather(ids)
            got = b.numpy()
            assert got.tobytes() == ob.tobytes()
            assert (cnt.hits, cnt.misses) == (oh, om) and om == int(sim["misses"][i])
            assert (io.pages_read, io.rows_read, io.bytes_read) == (int(oio[0]), int(oio[1]), int(oio[3]))
            a, z = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
            p, q = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
            cs = gx.Changeset(sim["in_ids"][a:z], sim["out_ids"][p:q], sim["in_pos"][a:z])
            c.apply_changeset(b, ids, cs)
            oc.apply(ob, ids, cs.in_ids, cs.in_positions, cs.out_ids)
            assert np.array_equal(c.resident_set(), oc.resident())
        for v in oc.resident():
            assert c.cached_row(int(v)).tobytes() == rows[int(v)].tobytes()


def test_host_backing_store(gx, oracle):
    rows = _feat(1000, 64, 4)
    f = gx.FeatureFile.from_array(rows, backing="host")
    c = gx.FeatureCache(f, [1, 2, 3], 10)
    b, cnt = c.gather(f, [5, 1, 999, 3])
    assert np.array_equal(b.numpy(), rows[[5, 1, 999, 3]]) and cnt.misses == 2


def test_pipeline_end_to_end(gx, oracle):
    """sample -> inspect -> gather/apply on the device == oracle stages composed."""
    n, dim = 30000, 32
    ip, ind = oracle.rmat_graph(n, 8.0, 17)
    g = gx.GraphFile.from_csc(ip, ind)
    rows = oracle.features(n, dim, 99)
    f = gx.FeatureFile.from_array(rows)
    train = oracle.train_ids(n, 2, 0.1)
    plan = oracle.plan_seed_batches(train, 100, oracle.epoch_seed(2, 0))[:12]
    K = 3000
    p = gx.Pipeline(g, f, [5, 5, 5], K, digest=True)
    st = p.run_superbatch(plan, 2, 0)
    trace = [oracle.sample_batch(ip, ind, b, [5, 5, 5], oracle.derive_seed(2, i))[0]
             for i, b in enumerate(plan)]
    init = oracle.compute_init_set(trace, K, n)
    sim = oracle.simulate(trace, n, K, init)
    assert np.array_equal(st.misses, sim["misses"])
    assert st.total_misses == st.predicted_misses == int(sim["misses"].sum())
    assert st.gathered_rows == sum(len(t) for t in trace)
    # gathered bytes of every iteration, via the digest
    dig = p.digests()
    for i, ids in enumerate(trace):
        assert int(dig[i]) == gx.batch_digest(rows[ids.astype(np.int64)])
    # second superbatch on the same pipeline (buffers reused, tables clean)
    plan2 = oracle.plan_seed_batches(train, 100, oracle.epoch_seed(2, 0))[12:20]
    st2 = p.run_superbatch(plan2, 2, 12)
    trace2 = [oracle.sample_batch(ip, ind, b, [5, 5, 5], oracle.derive_seed(2, 12 + i))[0]
              for i, b in enumerate(plan2)]
    init2 = oracle.compute_init_set(trace2, K, n)
    assert np.array_equal(st2.misses, oracle.simulate(trace2, n, K, init2)["misses"])


def test_pipeline_all_distinct_nodes_fit(gx, oracle):
    """K >= distinct nodes of the superbatch: init = every node, no misses, empty
    changesets (the inspector's all-fit shortcut) -- bytes still exact."""
    n, dim = 8000, 16
    ip, ind = oracle.rmat_graph(n, 6.0, 5)
    g = gx.GraphFile.from_csc(ip, ind)
    rows = oracle.features(n, dim, 4)
    f = gx.FeatureFile.from_array(rows)
    plan = oracle.plan_seed_batches(oracle.train_ids(n, 3, 0.2), 50, oracle.epoch_seed(3, 0))[:10]
    trace = [oracle.sample_batch(ip, ind, b, [4, 4], oracle.derive_seed(3, i))[0] for i, b in enumerate(plan)]
    for K in (n, len(np.unique(np.concatenate(trace)))):
        p = gx.Pipeline(g, f, [4, 4], K, digest=True)
        st = p.run_superbatch(plan, 3, 0)
        sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
        assert np.array_equal(st.misses, sim["misses"]) and st.total_misses == 0
        assert st.total_in == 0 and st.total_out == 0
        dig = p.digests()
        for i, ids in enumerate(trace):
            assert int(dig[i]) == gx.batch_digest(rows[ids.astype(np.int64)])
    # one node short of all-fit: the general path, still exact
    K = len(np.unique(np.concatenate(trace))) - 1
    st = gx.Pipeline(g, f, [4, 4], K).run_superbatch(plan, 3, 0)
    sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
    assert np.array_equal(st.misses, sim["misses"])


def test_pipeline_async_overlap_matches_sync(gx, oracle):
    """submit/wait with two superbatches in flight gives the same per-superbatch
    results (misses, digests) as running them one at a time."""
    n, dim = 20000, 32
    ip, ind = oracle.rmat_graph(n, 8.0, 23)
    g = gx.GraphFile.from_csc(ip, ind)
    rows = oracle.features(n, dim, 7)
    f = gx.FeatureFile.from_array(rows)
    plan = oracle.plan_seed_batches(oracle.train_ids(n, 4, 0.2), 64, oracle.epoch_seed(4, 0))
    sbs = [plan[o:o + 6] for o in range(0, 36, 6)]
    K = 2500
    sync = gx.Pipeline(g, f, [5, 5], K, digest=True)
    want = []
    for j, sb in enumerate(sbs):
        st = sync.run_superbatch(sb, 4, 6 * j)
        want.append((st.misses.copy(), sync.digests().copy()))
    asyn = gx.Pipeline(g, f, [5, 5], K, digest=True)
    got, prev = [], None
    for j, sb in enumerate(sbs):
        t = asyn.submit(sb, 4, 6 * j)
        if prev is not None:
            st = asyn.wait(prev)
            got.append((st.misses.copy(), asyn.digests().copy()))
        prev = t
    st = asyn.wait(prev)
    got.append((st.misses.copy(), asyn.digests().copy()))
    for (m1, d1), (m2, d2) in zip(want, got):
        assert np.array_equal(m1, m2) and np.array_equal(d1, d2)
    with pytest.raises(gx.LogicError):
        t0 = asyn.submit(sbs[0], 4, 0)
        t1 = asyn.submit(sbs[1], 4, 6)
        asyn.submit(sbs[2], 4, 12)  # a third in flight is refused
    asyn.wait(t0)
    asyn.wait(t1)


@pytest.mark.parametrize("K", [40, 400, 2500])
def test_pipeline_segments_resident_batches(gx, oracle, K):
    """Iterations without cache mutation are gathered by one launch (segment):
    misses are still charged to their own iteration (some miss without being
    inserted at small K), IoStats match a live oracle replay, and every
    iteration's batch stays readable in HBM after wait (gx_pipeline_batch)."""
    n, dim = 6000, 24
    ip, ind = oracle.rmat_graph(n, 5.0, 31)
    g = gx.GraphFile.from_csc(ip, ind)
    rows = oracle.features(n, dim, 12)
    f = gx.FeatureFile.from_array(rows)
    plan = oracle.plan_seed_batches(oracle.train_ids(n, 5, 0.3), 20, oracle.epoch_seed(5, 0))[:14]
    trace = [oracle.sample_batch(ip, ind, b, [3, 2], oracle.derive_seed(5, i))[0] for i, b in enumerate(plan)]
    init = oracle.compute_init_set(trace, K, n)
    sim = oracle.simulate(trace, n, K, init)
    p = gx.Pipeline(g, f, [3, 2], K)
    st = p.run_superbatch(plan, 5, 0)
    assert np.array_equal(st.misses, sim["misses"])
    empty = [int(sim["in_off"][i + 1] - sim["in_off"][i]) == 0 and int(sim["out_off"][i + 1] - sim["out_off"][i]) == 0
             for i in range(len(trace))]
    if K == 40:  # the case this test exists for: misses inside merged segments
        assert any(e and int(m) > 0 for e, m in zip(empty, sim["misses"]))
    oc = oracle.cache(rows, init, K)
    pages = rr = 0
    for i, ids in enumerate(trace):
        ob, oh, om, oio = oc.gather(ids)
        pages, rr = pages + int(oio[0]), rr + int(oio[1])
        a, z = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
        q, w = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
        oc.apply(ob, ids, sim["in_ids"][a:z], sim["in_pos"][a:z], sim["out_ids"][q:w])
        assert p.batch(i).tobytes() == ob.tobytes(), f"iteration {i} rows"
    assert (st.gather_io.pages_read, st.gather_io.rows_read, st.gather_io.bytes_read) == (pages, rr, rr * 4 * dim)
    with pytest.raises(IndexError):
        p.batch(len(trace))


@pytest.mark.parametrize("K,window", [(300, 16), (5000, 16), (5000, 3)])
def test_pipeline_batch_budget_fallback(oracle, K, window):
    """GX_BATCH_BUDGET_MB=0: the superbatch is not resident; a window of up to
    GX_BATCH_WINDOW iterations' rows is reused (runs of iterations without
    changesets -- all of them when everything fits, K = 5000 -- gather in one
    launch per window); results identical, only the last iteration stays
    readable."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent("""
        import numpy as np
        import paper_2208_09151_b200 as gx
        import oracle
        o = oracle.C
        n = 5000
        ip, ind = o.rmat_graph(n, 6.0, 3)
        rows = o.features(n, 16, 2)
        g, f = gx.GraphFile.from_csc(ip, ind), gx.FeatureFile.from_array(rows)
        plan = o.plan_seed_batches(o.train_ids(n, 2, 0.3), 30, o.epoch_seed(2, 0))[:8]
        trace = [o.sample_batch(ip, ind, b, [4, 3], o.derive_seed(2, i))[0] for i, b in enumerate(plan)]
        K = %d
        sim = o.simulate(trace, n, K, o.compute_init_set(trace, K, n))
        p = gx.Pipeline(g, f, [4, 3], K, digest=True)
        st = p.run_superbatch(plan, 2, 0)
        assert np.array_equal(st.misses, sim["misses"])
        for i, ids in enumerate(trace):
            assert int(p.digests()[i]) == gx.batch_digest(rows[ids.astype(np.int64)])
        assert np.array_equal(p.batch(len(trace) - 1), rows[trace[-1].astype(np.int64)])
        try:
            p.batch(0)
            raise SystemExit("expected LogicError")
        except gx.LogicError:
            pass
        print("OK")
    """) % K
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GX_BATCH_BUDGET_MB="0", GX_BATCH_WINDOW=str(window), PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("K", [200, 3000])       # changesets every iteration / all-fit (fused fill)
def test_pipeline_fp16_768(gx, oracle, K):
    """scalar_width 2 extension (configs[3], MAG240M shape: 768-d fp16 rows of
    1536 bytes) through the whole pipeline: batches byte-identical to the rows."""
    n, dim = 4000, 768
    ip, ind = oracle.rmat_graph(n, 6.0, 23)
    rows = oracle.features(n, dim, 24).astype(np.float16)
    g = gx.GraphFile.from_csc(ip, ind)
    f = gx.FeatureFile.from_array(rows)
    assert f.row_bytes() == 1536
    train = oracle.train_ids(n, 1, 0.3)
    plan = oracle.plan_seed_batches(train, 40, oracle.epoch_seed(1, 0))[:8]
    p = gx.Pipeline(g, f, [5, 3], K, digest=True)
    st = p.run_superbatch(plan, 1, 0)
    trace = [oracle.sample_batch(ip, ind, b, [5, 3], oracle.derive_seed(1, i))[0] for i, b in enumerate(plan)]
    sim = oracle.simulate(trace, n, K, oracle.compute_init_set(trace, K, n))
    assert np.array_equal(st.misses, sim["misses"])
    for i, ids in enumerate(trace):
        assert np.array_equal(p.batch(i), rows[ids.astype(np.int64)])
    assert st.fused_fill == (K >= len(np.unique(np.concatenate(trace))))


@pytest.mark.parametrize("fanout,S", [(1, 64), (0, 64), (1, 1), (1, 2)])
def test_allfit_fan_out_forms(gx, oracle, fanout, S):
    """All-fit superbatch through both fused executors: the fan-out form (each
    init row read once, written to its slot and to every batch row of its node;
    64 iterations over a 500-node graph, so hub slots own more than 32 batch rows
    and the per-warp list spans more than one 32-entry window) and the older
    fill-first + rest-gather form (GX_FANOUT=0, in a subprocess). Batches must
    be byte-identical to the rows of the oracle's trace."""
    import json
    import os
    import subprocess
    import sys
    import textwrap
    n, dim = 500, 32
    code = textwrap.dedent(f"""
        import json, numpy as np
        import paper_2208_09151_b200 as gx
        from oracle import C as oracle
        ip, ind = oracle.rmat_graph({n}, 8.0, 31)
        rows = oracle.features({n}, {dim}, 32)
        g = gx.GraphFile.from_csc(ip, ind)
        f = gx.FeatureFile.from_array(rows)
        train = oracle.train_ids({n}, 1, 0.9)
        plan = [train[(7 * i) % (len(train) - 20):][:20] for i in range({S})]
        p = gx.Pipeline(g, f, [6, 4], {n}, digest=True)
        st = p.run_superbatch(plan, 3, 0)
        trace = [oracle.sample_batch(ip, ind, b, [6, 4], oracle.derive_seed(3, i))[0] for i, b in enumerate(plan)]
        flat = np.concatenate(trace)
        hub = int(np.bincount(flat.astype(np.int64)).max())
        ok = all(np.array_equal(p.batch(i), rows[ids.astype(np.int64)]) for i, ids in enumerate(trace))
        dig = p.digests()
        ok = ok and all(int(dig[i]) == gx.batch_digest(rows[trace[i].astype(np.int64)]) for i in range(0, {S}, 9))
        print(json.dumps({{"ok": bool(ok), "fused": bool(st.fused_fill), "fan": bool(st.fan_out), "hub": hub,
                          "misses": int(st.total_misses), "init": int(st.init_size),
                          "distinct": int(len(np.unique(flat)))}}))
    """)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GX_FANOUT=str(fanout), PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["fused"] and res["fan"] == bool(fanout), res
    assert res["misses"] == 0 and res["init"] == res["distinct"], res
    assert res["hub"] > 32 or S < 64, res                      # S = 1: no access besides the first uses


def test_apply_duplicate_ids_match_reference(gx, ref, tmp_path):
    """apply_changeset with duplicate ids (feature_cache.hpp:103-129): the
    reference accepts them -- a duplicated out id frees its slot twice (two
    inserted nodes then share it, the later row wins), a duplicated in id is
    rewritten by its later entry. The device path replays exactly that."""
    dim = 8
    rows = _feat(12, dim, 5)
    path = str(tmp_path / "features.bin")
    ref.write_features(path, rows)
    rf = ref.open_features(path)
    f = gx.FeatureFile.from_array(rows)
    cases = [
        ([2, 5], [0, 0], [1, 2]),        # duplicated out: 2 and 5 share slot(0)
        ([2, 2], [0], [1, 1]),           # duplicated in: 2 written twice
        ([2, 5, 2], [0, 6, 6], [1, 2, 1]),
        ([2], [0, 0, 6], [1]),           # surplus freed slots pushed twice
    ]
    for in_ids, out_ids, in_pos in cases:
        init = [0, 1, 4, 6, 7]
        c = gx.FeatureCache(f, init, 6)
        rc = rf.cache(init, 6)
        ids = [0, 2, 5, 7]
        b, _ = c.gather(f, ids)
        rb, _, _, _ = rc.gather(ids, dim)
        assert b.numpy().tobytes() == rb.tobytes()
        c.apply_changeset(b, ids, gx.Changeset(in_ids, out_ids, in_pos))
        rc.apply(rb, ids, in_ids, in_pos, out_ids)
        res = rc.resident(12)
        assert list(c.resident_set()) == list(res)
        for v in res:
            assert c.cached_row(int(v)).tobytes() == rc.row(int(v), dim).tobytes()
        # later traffic goes through the same (shared / re-pushed) slots
        ids2 = [3, 8, 9, 10]
        b2, _ = c.gather(f, ids2)
        rb2, _, _, _ = rc.gather(ids2, dim)
        assert b2.numpy().tobytes() == rb2.tobytes()
        # two inserts with no evictions: fits only where the free list grew
        # (re-pushed surplus slots); otherwise both sides raise logic_error
        # "changeset overflows cache capacity" (feature_cache.hpp:110-111)
        from oracle.bind import OracleLogicError
        from paper_2208_09151_b200._lib import LogicError
        got = want = None
        try:
            c.apply_changeset(b2, ids2, gx.Changeset([3, 8], [], [0, 1]))
        except LogicError:
            got = "logic_error"
        try:
            rc.apply(rb2, ids2, [3, 8], [0, 1], [])
        except OracleLogicError:
            want = "logic_error"
        assert got == want, (in_ids, out_ids, got, want)
        assert list(c.resident_set()) == list(rc.resident(12))
        for v in rc.resident(12):
            assert c.cached_row(int(v)).tobytes() == rc.row(int(v), dim).tobytes()


def test_pipeline_rejects_duplicate_seeds(gx, oracle):
    """superbatch_sample rethrows sample_batch's duplicate-seed
    invalid_argument as runtime_error (sampler.hpp:83, 236); the fused
    pipeline reports the same, and stays usable afterwards."""
    ip, ind = oracle.rmat_graph(3000, 5.0, 21)
    g = gx.GraphFile.from_csc(ip, ind)
    f = gx.FeatureFile.from_array(_feat(3000, 16, 2))
    p = gx.Pipeline(g, f, [4, 4], 500)
    good = [np.arange(10, 40, dtype=np.uint64), np.arange(100, 130, dtype=np.uint64)]
    bad = [good[0], np.array([7, 8, 9, 8], np.uint64)]
    with pytest.raises(RuntimeError) as e1:
        p.run_superbatch(bad, 1, 0)
    with pytest.raises(RuntimeError) as e2:
        gx.sample_superbatch(g, None, bad, [4, 4], 1, 0)
    assert type(e1.value) is RuntimeError and type(e2.value) is RuntimeError  # not a CudaError
    st = p.run_superbatch(good, 1, 0)
    ref_edges = sum(sum(len(l) for l in oracle.sample_batch(ip, ind, b, [4, 4], oracle.derive_seed(1, i))[1])
                    for i, b in enumerate(good))
    assert st.sampled_edges == ref_edges


@pytest.mark.parametrize("one_gather,init_fan", [(1, 2), (1, 0), (0, 0)])
def test_pipeline_cache_state_matches_reference_replay(gx, oracle, one_gather, init_fan):
    """The fused pipeline's executor leaves the feature cache in the state the
    reference's FeatureCache reaches after S x (gather, apply_changeset)
    (feature_cache.hpp:58-130): every occupied slot holds its node's row, and
    every iteration's batch holds the rows of its ids. Run with the one-launch
    executor (GX_ONE_GATHER=1: one gather, changesets applied at once, last
    insert per slot) with and without the init fan-out (GX_INIT_FAN=2 forces
    it: the switch writes each init row to every access it serves, the gather
    copies the rest), and with the per-segment one."""
    import json
    import os
    import subprocess
    import sys
    code = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import oracle, paper_2208_09151_b200 as gx
o = oracle.C
n, dim, K = 4000, 16, 300
ip, ind = o.rmat_graph(n, 7.0, 44)
rows = o.features(n, dim, 45)
plan = o.plan_seed_batches(o.train_ids(n, 1, 0.3), 40, o.epoch_seed(1, 0))[:9]
p = gx.Pipeline(gx.GraphFile.from_csc(ip, ind), gx.FeatureFile.from_array(rows), [4, 3], K)
st = p.run_superbatch(plan, 1, 0)
trace = [o.sample_batch(ip, ind, b, [4, 3], o.derive_seed(1, i))[0] for i, b in enumerate(plan)]
init = o.compute_init_set(trace, K, n)
sim = o.simulate(trace, n, K, init)
c = o.cache(rows, init, K)
for i, ids in enumerate(trace):
    b, _, _, _ = c.gather(ids)
    a, e = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
    q, w = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
    c.apply(b, ids, sim["in_ids"][a:e], sim["in_pos"][a:e], sim["out_ids"][q:w])
got = p.cache_rows()
ok, occ = True, 0
for i, ids in enumerate(trace):
    ok &= bool(np.array_equal(p.batch(i), rows[ids.astype(np.int64)]))
ok &= bool(st.init_fan) == (%d == 1 and %d == 2)
for v in c.resident():
    s = c.slot(int(v))
    occ += 1
    ok &= bool(np.array_equal(got[s], rows[int(v)]))
print(json.dumps({"ok": ok, "occupied": occ, "inserts": int(st.total_in), "misses": int(st.total_misses)}))
""" % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), one_gather, init_fan)
    env = dict(os.environ, GX_ONE_GATHER=str(one_gather), GX_INIT_FAN=str(init_fan))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["occupied"] == 300 and res["inserts"] > 0, res
