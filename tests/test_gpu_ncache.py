"""GPU parity of the static neighbor cache (ncache.cu) against the reference
(neighbor_cache.hpp, compiled from its headers in oracle/_ref): the built
ncache.bin is byte-identical, the builder's IoStats match, and sampling with
the cache gives the same ids/edges and the same (reduced) IoStats as the
reference's sample_batch with that cache (sampler.hpp:91-97)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dataset(ref, tmp_path_factory):
    d = str(tmp_path_factory.mktemp("ncache"))
    ref.generate_dataset(d, 6000, 7.0, 8, 101, 102)
    return d


def _io_list(io):
    return [io.pages_read, io.rows_read, io.neighbor_lists_read, io.bytes_read]


@pytest.mark.parametrize("extra", [0, 16, 4000, 40_000, 10_000_000])
def test_build_matches_reference_bytes(gx, ref, dataset, tmp_path, extra):
    gpath = os.path.join(dataset, "graph.bin")
    rg = ref.open_graph(gpath)
    budget = rg.num_nodes * 8 + extra
    rpath = str(tmp_path / "ref_ncache.bin")
    rio, rk = rg.ncache_build(budget, rpath)
    g = gx.GraphFile.open(gpath)
    io = gx.IoStats()
    nc = gx.NeighborCache.build(g, budget, io)
    gpath2 = str(tmp_path / "gx_ncache.bin")
    nc.write(gpath2)
    assert open(gpath2, "rb").read() == open(rpath, "rb").read()
    assert nc.cached_node_count() == rk
    assert _io_list(io) == list(map(int, rio))
    assert nc.bytes_used() <= budget


def test_sampling_with_cache_matches_reference(gx, ref, dataset, tmp_path):
    gpath = os.path.join(dataset, "graph.bin")
    rg = ref.open_graph(gpath)
    budget = rg.num_nodes * 8 + 60_000
    rpath = str(tmp_path / "ncache.bin")
    rg.ncache_build(budget, rpath)
    g = gx.GraphFile.open(gpath)
    lio = gx.IoStats()
    nc = gx.NeighborCache.open(g, rpath, lio)       # the reference's file
    size = os.path.getsize(rpath)
    assert (lio.bytes_read, lio.pages_read) == (size, gx.pages_touched(0, size))
    rng = np.random.default_rng(4)
    total_with = gx.IoStats()
    for trial in range(6):
        seeds = rng.choice(rg.num_nodes, 64, replace=False).astype(np.uint64)
        want_ids, want_layers, want_io = rg.sample_batch(seeds, [5, 4, 3], 1000 + trial, rpath)
        _, _, plain_io = rg.sample_batch(seeds, [5, 4, 3], 1000 + trial)
        io = gx.IoStats()
        got = gx.sample_batch(g, nc, seeds, [5, 4, 3], 1000 + trial, io)
        assert np.array_equal(got.ids, want_ids)
        for l in range(3):
            assert np.array_equal(got.layers[l], want_layers[l])
        assert _io_list(io) == list(map(int, want_io))
        assert io.neighbor_lists_read <= int(plain_io[2])
        total_with += io
        io0 = gx.IoStats()                        # the cache is installed per call only
        gx.sample_batch(g, None, seeds, [5, 4, 3], 1000 + trial, io0)
        assert _io_list(io0) == list(map(int, plain_io))
    # superbatch form: IoStats = sum over its batches
    batches = [rng.choice(rg.num_nodes, 50, replace=False).astype(np.uint64) for _ in range(5)]
    sio = gx.IoStats()
    gx.sample_superbatch(g, nc, batches, [5, 4], 9, 3, sio)
    want = np.zeros(4, np.uint64)
    for i, b in enumerate(batches):
        want += rg.sample_batch(b, [5, 4], gx.derive_seed(9, 3 + i), rpath)[2]
    assert _io_list(sio) == list(map(int, want))


def test_ncache_errors(gx, ref, dataset, tmp_path):
    g = gx.GraphFile.open(os.path.join(dataset, "graph.bin"))
    with pytest.raises(ValueError):
        gx.NeighborCache.build(g, g.num_nodes() * 8 - 1)
    nc = gx.NeighborCache.build(g, g.num_nodes() * 8 + 1000)
    assert nc.contains(int(np.argmax([nc.contains(v) for v in range(50)]))) in (True, False)
    with pytest.raises(IndexError):
        nc.contains(g.num_nodes())
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTNCACH" + b"\0" * 40)
    with pytest.raises(RuntimeError):
        gx.NeighborCache.open(g, str(bad))
    small = gx.GraphFile.from_csc(np.array([0, 1, 1], np.uint64), np.array([1], np.uint64))
    with pytest.raises(ValueError):
        gx.sample_batch(small, nc, [0], [1], 1)


# ---------------------------------------------------------------------------
# comparison policies of `gx simulate` (baselines.hpp) vs the reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("K", [0, 50, 700, 6000])
def test_policies_match_reference(gx, ref, dataset, K):
    gpath = os.path.join(dataset, "graph.bin")
    rg = ref.open_graph(gpath)
    g = gx.GraphFile.open(gpath)
    rng = np.random.default_rng(K)
    trace = [rg.sample_batch(rng.choice(rg.num_nodes, 40, replace=False).astype(np.uint64), [4, 3], 50 + i)[0]
             for i in range(8)]
    for pol in ["none", "static_degree", "belady", "lru"]:
        want, tot = rg.simulate_policy(trace, K, pol)
        got = gx.simulate_policy(trace, rg.num_nodes, K, pol, graph=g)
        assert np.array_equal(got.misses, want), pol
        assert got.total_accesses == tot and got.policy == pol and got.capacity == K
    with pytest.raises(ValueError):
        gx.simulate_policy(trace, rg.num_nodes, K, "fifo")
    with pytest.raises(ValueError):
        gx.static_degree_set(g, rg.num_nodes + 1)
    s = gx.static_degree_set(g, 10)
    assert len(s) == 10 and len(set(s.tolist())) == 10


@pytest.mark.parametrize("K", [0, 1, 7, 64, 300, 5000])
def test_lru_matches_reference(gx, ref, dataset, K):
    """LRU (baselines.hpp:104-128) by device stack distances vs the reference's
    list+map simulation: sampled traces, random lists with repeats inside one
    iteration (the reference counts the repeat as a hit), and skewed ids."""
    gpath = os.path.join(dataset, "graph.bin")
    rg = ref.open_graph(gpath)
    n = rg.num_nodes
    rng = np.random.default_rng(100 + K)
    traces = [
        [rg.sample_batch(rng.choice(n, 30, replace=False).astype(np.uint64), [5, 4], 7 + i)[0] for i in range(12)],
        [rng.integers(0, 200, rng.integers(1, 80)).astype(np.uint64) for _ in range(40)],   # repeats
        [(rng.zipf(1.3, 150) % n).astype(np.uint64) for _ in range(25)],
        [np.zeros(0, np.uint64), np.array([5], np.uint64), np.zeros(0, np.uint64)],
    ]
    for t in traces:
        want, tot = rg.simulate_policy(t, K, "lru")
        got = gx.simulate_policy(t, n, K, "lru")
        assert np.array_equal(got.misses, want), (K, [len(x) for x in t][:5])
        assert got.total_accesses == tot
    with pytest.raises(IndexError):
        gx.simulate_policy([np.array([n], np.uint64)], n, K, "lru")
