"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only where oracle/_ref/libgx_ref.so exists (built by oracle/Makefile from
/root/reference/proj/include). Every array here is produced by a reference
function (listed per fixture); the tests compare the C oracle (CPU suite) and
the CUDA path (GPU suite) against them.

    python tests/golden/make_golden.py
"""
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import REF  # noqa: E402


def make_trace(num_nodes, iterations, max_ids, seed):
    """test_changeset.cpp:17-32 (same SplitMix64 stream)."""
    M = (1 << 64) - 1

    class R:
        def __init__(s, x):
            s.s = x

        def next(s):
            s.s = (s.s + 0x9E3779B97F4A7C15) & M
            z = s.s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
            return z ^ (z >> 31)

        def bounded(s, n):
            return (s.next() * n) >> 64

    r = R(seed)
    pool = list(range(num_nodes))
    t = []
    for _ in range(iterations):
        want = 1 + r.bounded(min(max_ids, num_nodes))
        ids = []
        for i in range(want):
            j = i + r.bounded(num_nodes - i)
            pool[i], pool[j] = pool[j], pool[i]
            ids.append(pool[i])
        t.append(ids)
    return t


def flat(trace):
    off = np.zeros(len(trace) + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in trace])
    return np.concatenate([np.asarray(x, np.uint64) for x in trace]), off


def main():
    assert REF.available(), "build oracle/_ref first (make -C oracle ref)"
    out = {}
    with tempfile.TemporaryDirectory() as d:
        # 1. dataset: generate_dataset (graphgen.hpp:87-108), N=2000, deg 8, dim 16
        E = REF.generate_dataset(d, 2000, 8.0, 16, 61, 62)
        g = REF.open_graph(os.path.join(d, "graph.bin"))
        ip, ind = g.read_all()
        with open(os.path.join(d, "features.bin"), "rb") as fh:
            feat = np.frombuffer(fh.read()[4096:], dtype="<f4").reshape(2000, 16)
        out.update(g_indptr=ip, g_indices=ind, g_features=feat.copy(), g_num_edges=np.uint64(E))
        # 2. sample_batch (sampler.hpp:69-117) on that graph
        rng = np.random.default_rng(2024)
        cases = []
        for t in range(12):
            ns = int(rng.integers(1, 80))
            seeds = rng.choice(2000, size=ns, replace=False).astype(np.uint64)
            fan = [int(x) for x in rng.integers(1, 16, size=int(rng.integers(1, 4)))]
            bs = int(rng.integers(0, 2**63))
            ids, layers, io = g.sample_batch(seeds, fan, bs)
            out[f"s{t}_seeds"] = seeds
            out[f"s{t}_fan"] = np.asarray(fan, np.uint32)
            out[f"s{t}_bs"] = np.uint64(bs)
            out[f"s{t}_ids"] = ids
            out[f"s{t}_io"] = io
            for l, e in enumerate(layers):
                out[f"s{t}_l{l}"] = e
            cases.append(t)
        out["sample_cases"] = np.asarray(cases)
        # 3. superbatch_sample files (sampler.hpp:197-243): byte images
        batches = [np.arange(i * 40, i * 40 + 40, dtype=np.uint64) for i in range(3)]
        rt = os.path.join(d, "rt")
        os.makedirs(rt)
        g.superbatch_sample(batches, [4, 4], 123, 5, 9, rt, 2)
        for i in range(3):
            for stem in ("ids", "adj"):
                with open(os.path.join(rt, f"{stem}_9_{i}.bin"), "rb") as fh:
                    out[f"file_{stem}_{i}"] = np.frombuffer(fh.read(), np.uint8).copy()
        g.close()
    # 4. changesets: compute_init_set + simulate_changesets (changeset.hpp:137-295)
    ccases = []
    for t, (n, it, w, seed, caps) in enumerate([(30, 12, 8, 500, (1, 3, 8)), (97, 24, 20, 901, (4, 16, 40)),
                                                 (400, 40, 60, 95000, (4, 32, 200)),
                                                 (5000, 64, 512, 10000, (16, 256, 1024))]):
        tr = make_trace(n, it, w, seed)
        fl, off = flat(tr)
        out[f"c{t}_flat"], out[f"c{t}_off"], out[f"c{t}_n"] = fl, off, np.uint64(n)
        iters, ptr = REF.access_index(tr, n)
        out[f"c{t}_iters"], out[f"c{t}_ptr"] = iters, ptr
        for K in caps:
            init = REF.compute_init_set(tr, K, n)
            r = REF.simulate(tr, n, K, init)
            for k in ("misses", "in_ids", "in_pos", "in_off", "out_ids", "out_off"):
                out[f"c{t}_K{K}_{k}"] = r[k]
            out[f"c{t}_K{K}_init"] = init
        out[f"c{t}_caps"] = np.asarray(caps, np.uint64)
        ccases.append(t)
    out["cs_cases"] = np.asarray(ccases)
    # 5. DP optimum (changeset.hpp:363-403) on tiny instances
    dp = []
    for t in range(40):
        tr = make_trace(2 + t % 7, 1 + t % 6, 4, 4000 + t)
        for K in range(4):
            dp.append((t, K, REF.dp_optimal_misses(tr, K)))
    out["dp"] = np.asarray(dp, np.uint64)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
