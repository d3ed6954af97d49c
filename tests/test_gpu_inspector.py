"""GPU parity: the persistent Belady inspector (inspector.cu) vs the C oracle
restatement of compute_init_set / simulate_changesets (changeset.hpp:137-295),
plus the reference's own KATs (test_changeset.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def make_trace(num_nodes, iterations, max_ids, seed):
    """test_changeset.cpp:17-32 make_trace (same RNG, same semantics)."""
    from paper_2208_09151_b200 import SplitMix64
    rng = SplitMix64(seed)
    pool = list(range(num_nodes))
    t = []
    for _ in range(iterations):
        want = 1 + rng.bounded(min(max_ids, num_nodes))
        ids = []
        for i in range(want):
            j = i + rng.bounded(num_nodes - i)
            pool[i], pool[j] = pool[j], pool[i]
            ids.append(pool[i])
        t.append(ids)
    return t


def _check(oracle, gx, trace, N, K, init=None):
    if init is None:
        init = oracle.compute_init_set(trace, K, N)
        cs = gx.precompute_trace(trace, N, K)
        assert np.array_equal(cs.init_set(), init), "init set differs"
    else:
        cs = gx.precompute_trace(trace, N, K, init=init)
    want = oracle.simulate(trace, N, K, init)
    assert np.array_equal(cs.misses(), want["misses"]), "misses differ"
    for i in range(len(trace)):
        c = cs.changeset(i)
        a, b = int(want["in_off"][i]), int(want["in_off"][i + 1])
        assert np.array_equal(c.in_ids, want["in_ids"][a:b]), f"in_ids differ at {i}"
        assert np.array_equal(c.in_positions, want["in_pos"][a:b]), f"in_pos differ at {i}"
        a, b = int(want["out_off"][i]), int(want["out_off"][i + 1])
        assert np.array_equal(c.out_ids, want["out_ids"][a:b]), f"out_ids differ at {i}"
    return cs


def test_fig11_kat(gx):
    # test_changeset.cpp:150-171
    t = [[0, 2, 5, 7], [1, 2, 4, 5, 7], [6]]
    cs = gx.precompute_trace(t, 10, 5, init=[0, 1, 4, 6, 7])
    c = cs.changeset(0)
    assert list(c.in_ids) == [2, 5] and list(c.in_positions) == [1, 2] and list(c.out_ids) == [0, 6]
    states = []
    gx.simulate_changesets(None, t, 5, [0, 1, 4, 6, 7], lambda i, c, st: states.append(list(st)),
                           num_nodes=10)
    assert states[0] == [1, 2, 4, 5, 7]


def test_elementary_kats(gx, oracle):
    # test_changeset.cpp:174-232
    r = gx.simulate_changesets(None, [[7], [8], [7]], 1, [], num_nodes=9)
    assert list(r.misses) == [1, 1, 0] and r.total_misses() == 2
    t = make_trace(10, 5, 4, 3)
    r = gx.simulate_changesets(None, t, 0, [], num_nodes=10)
    assert r.total_misses() == r.total_accesses
    with pytest.raises(gx.LogicError):
        gx.precompute_trace([[1], [2]], 5, 2, init=[4])
    with pytest.raises(ValueError):
        gx.precompute_trace([[1, 2]], 5, 1, init=[1, 2])
    with pytest.raises(gx.LogicError):
        gx.precompute_trace([[1, 1]], 3, 1)
    with pytest.raises(IndexError):
        gx.precompute_trace([[9]], 3, 1)
    assert list(gx.compute_init_set([[4, 1], [2, 4, 9]], 3, 10)) == [4, 1, 2]
    assert list(gx.compute_init_set([[4, 1], [2, 4, 9]], 100, 10)) == [4, 1, 2, 9]


def test_access_index_kat(gx, oracle):
    # test_changeset.cpp:92-112 (tracking fixture)
    t = [[3, 4], [2, 4], [3, 0], [0, 4], [3, 1]]
    ix = gx.build_access_index(t, 5)
    assert len(ix.iters) == 11
    assert int(ix.ptr[3]) == 4 and int(ix.ptr[4]) == 7
    assert [int(x) & gx.api.ITER_MASK for x in ix.iters[4:7]] == [0, 2, 4]
    assert int(ix.iters[10]) == gx.api.ITER_DUMMY
    for seed in range(10):
        tr = make_trace(30, 12, 8, 500 + seed)
        a = gx.build_access_index(tr, 30)
        i2, p2 = oracle.access_index(tr, 30)
        assert np.array_equal(a.iters, i2) and np.array_equal(a.ptr, p2)


@pytest.mark.parametrize("seed", range(20))
def test_random_traces_vs_oracle(oracle, gx, seed):
    # the acceptance c1 shape (simulator == naive oracle) against the restatement
    n = 10 + 7 * seed
    t = make_trace(n, 3 + (seed % 24), 9, 900 + seed)
    for K in (0, 1, 3, 8, 40):
        _check(oracle, gx, t, n, K)


def test_wide_traces_vs_oracle(oracle, gx):
    rng = np.random.default_rng(7)
    for t_i in range(12):
        n = int(16 << rng.integers(0, 9))
        n = min(n + int(rng.integers(0, n)), 5000)
        iters = int(2 << rng.integers(0, 7))
        width = 1 + int(rng.integers(0, min(512, n)))
        tr = make_trace(n, iters, width, 10_000 + t_i)
        for K in (16, 64, 256, 1024):
            _check(oracle, gx, tr, n, K)


def test_explicit_init_and_big_selection(oracle, gx):
    # large cut buckets: all ids accessed once -> everything NEVER after first use
    tr = [list(range(i * 3000, i * 3000 + 3000)) for i in range(6)]
    _check(oracle, gx, tr, 18000, 5000)
    # many distinct keys, out-set larger than the smem sort path (> 4096)
    rng = np.random.default_rng(3)
    N = 200000
    tr = [rng.choice(N, size=20000, replace=False) for _ in range(8)]
    _check(oracle, gx, tr, N, 30000)
    init = oracle.compute_init_set(tr, 30000, N)[::-1].copy()
    _check(oracle, gx, tr, N, 30000, init=init)


@pytest.mark.slow
def test_sampled_trace_cfg_like(oracle, gx):
    """A trace produced by the sampler itself (100K-node R-MAT, 32 x 512 seeds)."""
    ip, ind = oracle.rmat_graph(100_000, 15.0, 71)
    g = gx.GraphFile.from_csc(ip, ind)
    rng = np.random.default_rng(0)
    batches = [rng.choice(100_000, size=512, replace=False) for _ in range(32)]
    s = gx.sample_superbatch(g, None, batches, [10, 10, 10], 5, 0)
    tr = [s.batch(i).ids for i in range(len(s))]
    for K in (1000, 10000, 50000):
        _check(oracle, gx, tr, 100_000, K)
