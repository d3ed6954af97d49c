"""CPU suite: pin the C restatement (oracle/gx_oracle.c) before trusting it.

1. against golden fixtures generated from the UNMODIFIED reference
   (tests/golden/make_golden.py -> reference_golden.npz);
2. against the reference's own recorded acceptance numbers
   (tests/golden/acceptance_kats.json <- proj/test_output.txt);
3. against the reference unit-test KATs (test_changeset.cpp, test_sampler.cpp,
   test_feature_cache.cpp), restated;
4. live against oracle/_ref/libgx_ref.so when it is built (this container).
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
KATS = json.load(open(os.path.join(HERE, "golden", "acceptance_kats.json")))


def _unflat(flat, off):
    return [flat[int(off[i]):int(off[i + 1])] for i in range(len(off) - 1)]


def test_dataset_matches_reference_generator(oracle):
    ip, ind = oracle.rmat_graph(2000, 8.0, 61)
    assert np.array_equal(ip, G["g_indptr"]) and np.array_equal(ind, G["g_indices"])
    assert len(ind) == int(G["g_num_edges"])
    assert np.array_equal(oracle.features(2000, 16, 62), G["g_features"])


def test_sample_batch_golden(oracle):
    ip, ind = G["g_indptr"], G["g_indices"]
    for t in G["sample_cases"]:
        fan = [int(x) for x in G[f"s{t}_fan"]]
        ids, layers, io = oracle.sample_batch(ip, ind, G[f"s{t}_seeds"], fan, int(G[f"s{t}_bs"]))
        assert np.array_equal(ids, G[f"s{t}_ids"])
        for l in range(len(fan)):
            assert np.array_equal(layers[l], G[f"s{t}_l{l}"])
        assert np.array_equal(io, G[f"s{t}_io"])


def test_changesets_golden(oracle):
    for t in G["cs_cases"]:
        tr = _unflat(G[f"c{t}_flat"], G[f"c{t}_off"])
        n = int(G[f"c{t}_n"])
        iters, ptr = oracle.access_index(tr, n)
        assert np.array_equal(iters, G[f"c{t}_iters"]) and np.array_equal(ptr, G[f"c{t}_ptr"])
        for K in G[f"c{t}_caps"]:
            K = int(K)
            init = oracle.compute_init_set(tr, K, n)
            assert np.array_equal(init, G[f"c{t}_K{K}_init"])
            r = oracle.simulate(tr, n, K, init)
            for k in ("misses", "in_ids", "in_pos", "in_off", "out_ids", "out_off"):
                assert np.array_equal(r[k], G[f"c{t}_K{K}_{k}"]), (t, K, k)


def _dp_optimal_misses(trace, cap):
    """changeset.hpp:363-403 restated (exhaustive DP over cache subsets)."""
    labels = []
    masks = []
    for ids in trace:
        m = 0
        for v in ids:
            if v not in labels:
                labels.append(v)
            m |= 1 << labels.index(v)
        masks.append(m)
    INF = float("inf")
    dp = {0: 0}
    for a in masks:
        nd = {}
        for mask, c in dp.items():
            cost = c + bin(a & ~mask).count("1")
            u = mask | a
            s = u
            while True:
                if bin(s).count("1") <= cap and cost < nd.get(s, INF):
                    nd[s] = cost
                if s == 0:
                    break
                s = (s - 1) & u
        dp = nd
    return min(dp.values())


def test_dp_optimum_golden_and_simulator_optimality(oracle):
    from tests.golden.make_golden import make_trace
    for t, K, want in G["dp"]:
        t, K, want = int(t), int(K), int(want)
        tr = make_trace(2 + t % 7, 1 + t % 6, 4, 4000 + t)
        assert _dp_optimal_misses(tr, K) == want
        n = 2 + t % 7
        assert int(oracle.simulate(tr, n, K, []) ["misses"].sum()) == want  # acceptance c2


def test_changeset_kats(oracle):
    # test_changeset.cpp:52-171 restated against the oracle
    t = [[3, 4], [2, 4], [3, 0], [0, 4], [3, 1]]
    iters, ptr = oracle.access_index(t, 5)
    assert int(ptr[3]) == 4 and int(ptr[4]) == 7 and len(iters) == 11
    assert [int(x) & ((1 << 63) - 1) for x in iters[4:7]] == [0, 2, 4]
    assert list(oracle.compute_init_set([[4, 1], [2, 4, 9]], 3, 10)) == [4, 1, 2]
    r = oracle.simulate([[0, 2, 5, 7], [1, 2, 4, 5, 7], [6]], 10, 5, [0, 1, 4, 6, 7], states=True)
    a, b = int(r["in_off"][0]), int(r["in_off"][1])
    assert list(r["in_ids"][a:b]) == [2, 5] and list(r["in_pos"][a:b]) == [1, 2]
    assert list(r["out_ids"][:int(r["out_off"][1])]) == [0, 6]
    assert list(r["state"][:int(r["state_off"][1])]) == [1, 2, 4, 5, 7]
    assert list(oracle.simulate([[7], [8], [7]], 9, 1, [])["misses"]) == [1, 1, 0]
    with pytest.raises(Exception):
        oracle.simulate([[1, 1]], 3, 1, [])


def test_sampler_kats(oracle):
    ip, ind = oracle.build_csc(3, [1, 2], [0, 0])
    ids, layers, _ = oracle.sample_batch(ip, ind, [0], [3], 9)
    assert len(layers[0]) == 2 and sorted(int(ids[s]) for s, d in layers[0]) == [1, 2]
    ip = np.zeros(6, np.uint64)
    ids, layers, _ = oracle.sample_batch(ip, np.zeros(0, np.uint64), [3, 1], [4, 4], 1)
    assert list(ids) == [3, 1] and all(len(l) == 0 for l in layers)
    with pytest.raises(IndexError):
        oracle.sample_batch(ip, np.zeros(0, np.uint64), [7], [2], 1)
    with pytest.raises(ValueError):
        oracle.sample_batch(ip, np.zeros(0, np.uint64), [1, 1], [2], 1)


def test_page_accounting(oracle):
    # test_graph_store.cpp:6-21, common.hpp:48-61
    assert oracle.page_count_for_row(4096, 0) == 1 and oracle.page_count_for_row(3072, 1) == 2
    rng = np.random.default_rng(13)
    for _ in range(200):
        w, r = int(rng.integers(1, 10000)), int(rng.integers(0, 50))
        walk = len({b // 4096 for b in range(r * w, (r + 1) * w)})
        assert oracle.page_count_for_row(w, r) == walk


def test_acceptance_c3_miss_ratios(oracle):
    """The reference's recorded Belady miss ratios (test_output.txt:17), from the oracle."""
    from paper_2208_09151_b200 import SplitMix64
    k = KATS["c3_belady_miss_ratio"]
    n = k["num_nodes"]
    ip, ind = oracle.rmat_graph(n, k["avg_degree"], k["edge_seed"])
    sums = np.zeros(4)
    for seed in (1, 2, 3):
        rng = SplitMix64(oracle.derive_seed(seed, 0x7261))
        pool = list(range(n))
        train = []
        for i in range(64 * 512):
            j = i + rng.bounded(n - i)
            pool[i], pool[j] = pool[j], pool[i]
            train.append(pool[i])
        plan = oracle.plan_seed_batches(train, 512, oracle.derive_seed(seed, 1))
        trace = [oracle.sample_batch(ip, ind, b, [10, 10, 10], oracle.derive_seed(seed, 100 + i))[0]
                 for i, b in enumerate(plan)]
        acc = sum(len(t) for t in trace)
        for c, K in enumerate(k["capacities"]):
            init = oracle.compute_init_set(trace, K, n)
            sums[c] += oracle.simulate(trace, n, K, init)["misses"].sum() / acc
    assert [f"{x / 3:.6f}" for x in sums] == k["miss_ratio"]


def test_oracle_vs_reference_live(oracle, ref):
    rng = np.random.default_rng(5)
    ip, ind = oracle.rmat_graph(3000, 7.0, 9)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        ref.write_graph_csc(os.path.join(d, "g.bin"), ip, ind)
        g = ref.open_graph(os.path.join(d, "g.bin"))
        for t in range(20):
            seeds = rng.choice(3000, size=int(rng.integers(1, 100)), replace=False)
            fan = [int(x) for x in rng.integers(1, 30, size=int(rng.integers(1, 4)))]
            bs = int(rng.integers(0, 2**63))
            a, b = oracle.sample_batch(ip, ind, seeds, fan, bs), g.sample_batch(seeds, fan, bs)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
            assert all(np.array_equal(x, y) for x, y in zip(a[1], b[1]))
        g.close()
    from tests.golden.make_golden import make_trace
    for t in range(10):
        n = int(rng.integers(10, 400))
        tr = make_trace(n, int(rng.integers(1, 30)), int(rng.integers(1, 50)), 77 + t)
        for K in (0, 1, 5, 30, n):
            init = oracle.compute_init_set(tr, K, n)
            assert np.array_equal(init, ref.compute_init_set(tr, K, n))
            x, y = oracle.simulate(tr, n, K, init), ref.simulate(tr, n, K, init)
            for k in ("misses", "in_ids", "in_pos", "out_ids", "in_off", "out_off"):
                assert np.array_equal(x[k], y[k])
            z = ref.simulate(tr, n, K, init, naive=True)  # acceptance c1: simulator == naive oracle
            assert np.array_equal(z["misses"], y["misses"]) and np.array_equal(z["in_ids"], y["in_ids"])


def test_feature_cache_oracle_vs_reference(oracle, ref):
    import tempfile
    rng = np.random.default_rng(3)
    rows = rng.random((60, 5)).astype(np.float32)
    with tempfile.TemporaryDirectory() as d:
        ref.write_features(os.path.join(d, "f.bin"), rows)
        f = ref.open_features(os.path.join(d, "f.bin"))
        trace = [np.sort(rng.choice(60, size=int(rng.integers(1, 12)), replace=False)) for _ in range(25)]
        for K in (2, 7, 20):
            init = oracle.compute_init_set(trace, K, 60)
            sim = oracle.simulate(trace, 60, K, init)
            rc, oc = f.cache(init, K), oracle.cache(rows, init, K)
            assert np.array_equal(rc.io, oc.io)
            for i, ids in enumerate(trace):
                rb, rh, rm, rio = rc.gather(ids, 5)
                ob, oh, om, oio = oc.gather(ids)
                assert rb.tobytes() == ob.tobytes() and (rh, rm) == (oh, om) and np.array_equal(rio, oio)
                a, z = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
                p, q = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
                args = (ids, sim["in_ids"][a:z], sim["in_pos"][a:z], sim["out_ids"][p:q])
                rc.apply(rb, *args)
                oc.apply(ob, *args)
                assert np.array_equal(rc.resident(60), oc.resident())
        f.close()


@pytest.mark.parametrize("n,avg,dim,threads", [(1, 3.0, 4, 2), (2000, 8.0, 16, 3), (70_000, 10.0, 8, 8),
                                               (5000, 0.0, 4, 4), (33_333, 14.67, 3, 5)])
def test_threaded_generator_matches_reference(ref, tmp_path, n, avg, dim, threads):
    """oracle/gen_dataset.cpp (the bench reference arm's input writer) is
    byte-identical to the reference's generate_dataset (graphgen.hpp:82-108)
    at any thread count."""
    import oracle as o
    es, vs = o.C.derive_seed(7, 0xED6E5), o.C.derive_seed(7, 0xFEA7)
    rd = tmp_path / "ref"
    rd.mkdir()
    e_ref = ref.generate_dataset(str(rd), n, avg, dim, es, vs)
    e = o.GEN.graph_file(tmp_path / "graph.bin", n, avg, es, threads)
    o.GEN.features_file(tmp_path / "features.bin", n, dim, vs, threads)
    assert e == e_ref
    for name in ("graph.bin", "features.bin"):
        assert (tmp_path / name).read_bytes() == (rd / name).read_bytes(), name


def test_compute_stub_matches_reference(oracle, ref):
    """compute_stub (pipeline.hpp:35-57) restated in oracle/gx_oracle.c equals the
    reference's on random batches and adjacency (incl. empty layers/batches)."""
    rng = np.random.default_rng(3)
    for rows_n, dim, layers in [(5, 4, [3, 0, 7]), (0, 8, [0]), (40, 16, [12, 90]), (1, 1, [])]:
        rows = rng.random((rows_n, dim)).astype(np.float32)
        adj = [rng.integers(0, 1 << 20, (c, 2)).astype(np.uint32) for c in layers]
        assert oracle.compute_stub(rows, adj) == ref.compute_stub(rows, adj)
