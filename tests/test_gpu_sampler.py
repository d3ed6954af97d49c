"""GPU parity: the sm_100a sampler (sampler.cu) vs the C oracle restatement of
sample_batch / superbatch_sample (sampler.hpp:69-117, 197-243). Bit-exact ids,
per-layer edges and IoStats on the same inputs."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_graph(oracle, n, m, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, size=m).astype(np.uint64)
    dst = rng.integers(0, n, size=m).astype(np.uint64)
    return oracle.build_csc(n, src, dst)


def _same(a, b):
    ids_a, layers_a, io_a = a
    assert np.array_equal(ids_a, b.ids), "ids differ"
    assert len(layers_a) == len(b.layers)
    for l, (x, y) in enumerate(zip(layers_a, b.layers)):
        assert np.array_equal(x, y), f"layer {l} edges differ"


def test_sample_batch_random_graphs(oracle, gx):
    rng = np.random.default_rng(1)
    for t in range(40):
        n = int(rng.integers(2, 3000))
        ip, ind = _rand_graph(oracle, n, int(rng.integers(0, 12 * n)), 100 + t)
        g = gx.GraphFile.from_csc(ip, ind)
        ns = int(rng.integers(1, min(n, 200) + 1))
        seeds = rng.choice(n, size=ns, replace=False).astype(np.uint64)
        fan = [int(x) for x in rng.integers(1, 26, size=int(rng.integers(1, 4)))]
        bs = int(rng.integers(0, 2**63))
        io = gx.IoStats()
        got = gx.sample_batch(g, None, seeds, fan, bs, io)
        want = oracle.sample_batch(ip, ind, seeds, fan, bs)
        _same(want, got)
        assert (io.pages_read, io.rows_read, io.neighbor_lists_read, io.bytes_read) == tuple(
            int(x) for x in want[2]), "IoStats differ"


def test_fanout_above_degree_and_big_fanouts(oracle, gx):
    # test_sampler.cpp:52-71 plus fanouts beyond the 32-entry pick cache
    ip, ind = oracle.build_csc(3, [1, 2], [0, 0])
    g = gx.GraphFile.from_csc(ip, ind)
    out = gx.sample_batch(g, None, [0], [3], 9)
    assert len(out.layers[0]) == 2
    assert sorted(int(out.ids[s]) for s, d in out.layers[0]) == [1, 2]
    ip, ind = _rand_graph(oracle, 500, 40000, 5)  # avg in-degree ~80
    g = gx.GraphFile.from_csc(ip, ind)
    for fan in ([40, 3], [70], [33, 33]):
        seeds = np.arange(0, 500, 7, dtype=np.uint64)
        _same(oracle.sample_batch(ip, ind, seeds, fan, 77), gx.sample_batch(g, None, seeds, fan, 77))


def test_edgeless_and_errors(oracle, gx):
    ip = np.zeros(6, np.uint64)
    g = gx.GraphFile.from_csc(ip, np.zeros(0, np.uint64))
    out = gx.sample_batch(g, None, [3, 1], [4, 4], 1)
    assert list(out.ids) == [3, 1]
    assert all(len(l) == 0 for l in out.layers)
    with pytest.raises(IndexError):
        gx.sample_batch(g, None, [7], [2], 1)
    with pytest.raises(ValueError):
        gx.sample_batch(g, None, [1, 1], [2], 1)
    with pytest.raises(ValueError):
        gx.sample_batch(g, None, [], [2], 1)
    # duplicate before out-of-range -> invalid_argument (reference seed order)
    with pytest.raises(ValueError):
        gx.sample_batch(g, None, [1, 1, 9], [2], 1)
    with pytest.raises(IndexError):
        gx.sample_batch(g, None, [1, 9, 1], [2], 1)
    # superbatch_sample wraps per-batch failures into runtime_error (sampler.hpp:236)
    with pytest.raises(RuntimeError):
        gx.sample_superbatch(g, None, [[1], [9]], [2], 1, 0)


def test_superbatch_matches_per_batch_oracle(oracle, gx):
    ip, ind = oracle.rmat_graph(20000, 9.0, 71)
    g = gx.GraphFile.from_csc(ip, ind)
    train = oracle.train_ids(20000, 3, 0.2)
    plan = oracle.plan_seed_batches(train, 128, oracle.epoch_seed(3, 0))
    batches = plan[:24]
    io = gx.IoStats()
    s = gx.sample_superbatch(g, None, batches, [10, 10, 10], 3, 40, io)
    tot = np.zeros(4, np.uint64)
    for i, b in enumerate(batches):
        want = oracle.sample_batch(ip, ind, b, [10, 10, 10], oracle.derive_seed(3, 40 + i))
        _same(want, s.batch(i))
        tot += want[2]
    assert (io.pages_read, io.neighbor_lists_read, io.bytes_read) == (int(tot[0]), int(tot[2]), int(tot[3]))


def test_superbatch_files_roundtrip(oracle, gx):
    ip, ind = oracle.rmat_graph(3000, 6.0, 5)
    g = gx.GraphFile.from_csc(ip, ind)
    batches = [np.arange(i * 30, i * 30 + 30, dtype=np.uint64) for i in range(4)]
    with tempfile.TemporaryDirectory() as d:
        r = gx.superbatch_sample(g, None, batches, [4, 4], 123, 0, 7, d)
        assert r.files_written == 8 and len(os.listdir(d)) == 8
        for i, b in enumerate(batches):
            ids, layers, _ = oracle.sample_batch(ip, ind, b, [4, 4], oracle.derive_seed(123, i))
            assert np.array_equal(gx.read_ids_file(gx.api.ids_file_path(d, 7, i)), ids)
            adj = gx.read_adj_file(gx.api.adj_file_path(d, 7, i))
            assert all(np.array_equal(x, y) for x, y in zip(adj, layers))


@pytest.mark.slow
def test_cfg1_shape_batches(oracle, gx):
    """cfg1 shape (1M nodes, avg degree 10, B=1000, fanout 10,10,10): first 8 batches."""
    ip, ind = oracle.rmat_graph(1_000_000, 10.0, oracle.derive_seed(7, 0xED6E5))
    assert len(ind) == 9_711_781  # SURVEY §8d cfg1 edge count after dedup
    g = gx.GraphFile.from_csc(ip, ind)
    train = oracle.train_ids(1_000_000, 1, 0.1)
    plan = oracle.plan_seed_batches(train, 1000, oracle.epoch_seed(1, 0))
    s = gx.sample_superbatch(g, None, plan[:8], [10, 10, 10], 1, 0)
    for i in range(8):
        _same(oracle.sample_batch(ip, ind, plan[i], [10, 10, 10], oracle.derive_seed(1, i)), s.batch(i))


def test_device_generator_matches_reference_generator(oracle, gx):
    for (n, deg, seed) in [(1000, 8.0, 61), (4097, 3.5, 9), (1, 4.0, 2), (50, 0.0, 3)]:
        ip, ind = oracle.rmat_graph(n, deg, seed)
        g = gx.GraphFile.generate_rmat(n, deg, seed)
        gip, gind = g.to_csc()
        assert np.array_equal(ip, gip) and np.array_equal(ind, gind)


def test_superbatch_spanning_several_launches(oracle, gx):
    """> 128 batches run as consecutive sampler launches into one output."""
    ip, ind = oracle.rmat_graph(5000, 6.0, 21)
    g = gx.GraphFile.from_csc(ip, ind)
    rng = np.random.default_rng(9)
    batches = [rng.choice(5000, size=int(rng.integers(1, 12)), replace=False).astype(np.uint64)
               for _ in range(300)]
    io = gx.IoStats()
    s = gx.sample_superbatch(g, None, batches, [3, 3], 17, 1000, io)
    tot = np.zeros(4, np.uint64)
    for i in range(0, 300, 7):
        want = oracle.sample_batch(ip, ind, batches[i], [3, 3], oracle.derive_seed(17, 1000 + i))
        _same(want, s.batch(i))
    for i in range(300):
        tot += oracle.sample_batch(ip, ind, batches[i], [3, 3], oracle.derive_seed(17, 1000 + i))[2]
    assert (io.pages_read, io.neighbor_lists_read) == (int(tot[0]), int(tot[2]))
