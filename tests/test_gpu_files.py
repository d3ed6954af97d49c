"""GPU: the precompute file stage (changeset.hpp:409-484) and the runtime-file
writers, byte-compared with the reference's own writers (oracle/_ref).

* test_changeset.cpp:333-352 ("precompute stage emits S+1 files consistent
  with the simulation") restated for gx.precompute_changesets;
* init_{sb}.bin / update_{sb}_{i}.bin written by the device path are
  byte-identical to the files the reference's precompute_changesets writes
  from the same ids files (write_init_file / write_update_file,
  changeset.hpp:417-442);
* the same for a sampler-produced superbatch: device sampler -> ids/adj files,
  device inspector (the pipeline's trusted-trace path) -> init/update files,
  against the reference's superbatch_sample + precompute_changesets."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def make_trace(num_nodes, iterations, max_ids, seed, gx):
    """make_trace (test_changeset.cpp:17-32): per iteration 1 + bounded(min(max_ids, n))
    distinct ids by a partial Fisher-Yates over a persistent pool."""
    rng = gx.SplitMix64(seed)
    pool = list(range(num_nodes))
    t = []
    for _ in range(iterations):
        want = 1 + rng.bounded(min(max_ids, num_nodes))
        ids = []
        for i in range(want):
            j = i + rng.bounded(num_nodes - i)
            pool[i], pool[j] = pool[j], pool[i]
            ids.append(pool[i])
        t.append(np.array(ids, np.uint64))
    return t


def _files(d, sb, S):
    names = [f"init_{sb}.bin"] + [f"update_{sb}_{i}.bin" for i in range(S)]
    return {n: open(os.path.join(d, n), "rb").read() for n in names}


def _write_trace(gx, d, sb, trace):
    os.makedirs(d, exist_ok=True)
    paths = []
    for i, ids in enumerate(trace):
        p = gx.ids_file_path(d, sb, i)
        gx.write_ids_file(p, ids)
        paths.append(p)
    return paths


def test_precompute_stage_emits_files(gx, oracle, ref, tmp_path):
    """test_changeset.cpp:333-352, plus the file bytes vs the reference."""
    t = make_trace(30, 6, 8, 123, gx)
    d = str(tmp_path / "gx")
    ft = gx.FileTrace(_write_trace(gx, d, 0, t))
    pr = gx.precompute_changesets(ft, 30, 5, d, 0)
    assert pr.files_written == 7
    assert pr.init_size == 5
    init = gx.read_init_file(gx.init_file_path(d, 0))
    assert np.array_equal(init, oracle.compute_init_set(t, 5, 30))
    sim = oracle.simulate(t, 30, 5, init)
    for i in range(len(t)):
        cs = gx.read_update_file(gx.update_file_path(d, 0, i))
        a, b = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
        c, e = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
        assert cs == gx.Changeset(sim["in_ids"][a:b], sim["out_ids"][c:e], sim["in_pos"][a:b]), i
    assert np.array_equal(pr.sim.misses, sim["misses"])
    # the reference's precompute_changesets over the same ids files
    r = str(tmp_path / "ref")
    _write_trace(gx, r, 0, t)
    m, n_init = ref.precompute_changesets(r, 0, len(t), 30, 5)
    assert n_init == pr.init_size and np.array_equal(m, pr.sim.misses)
    assert _files(d, 0, len(t)) == _files(r, 0, len(t))


@pytest.mark.parametrize("n,S,width,K,seed", [
    (200, 40, 60, 50, 1),        # steady eviction: changesets in every iteration
    (5000, 25, 900, 700, 2),     # wide iterations, out lists sorted in smem
    (40000, 12, 9000, 6000, 3),  # out lists > 4096 (bitmap compaction)
    (3000, 30, 100, 4000, 4),    # all-fit: empty changesets
    (100, 20, 30, 0, 5),         # K = 0: no init, everything misses
])
def test_precompute_files_match_reference(gx, ref, tmp_path, n, S, width, K, seed):
    t = make_trace(n, S, width, seed, gx)
    d, r = str(tmp_path / "gx"), str(tmp_path / "ref")
    pr = gx.precompute_changesets(gx.FileTrace(_write_trace(gx, d, 7, t)), n, K, d, 7)
    _write_trace(gx, r, 7, t)
    m, n_init = ref.precompute_changesets(r, 7, S, n, K)
    assert pr.files_written == S + 1
    assert n_init == pr.init_size and np.array_equal(m, pr.sim.misses)
    assert _files(d, 7, S) == _files(r, 7, S)


def test_sampled_superbatch_files_match_reference(gx, oracle, ref, tmp_path):
    """Sampler + inspector on the device (the fused pipeline's trusted-trace
    inspector path) write ids/adj/init/update files byte-identical to the
    reference's superbatch_sample + precompute_changesets."""
    n = 20000
    ip, ind = oracle.rmat_graph(n, 8.0, 31)
    gpath = str(tmp_path / "graph.bin")
    ref.write_graph_csc(gpath, ip, ind)
    rg = ref.open_graph(gpath)
    g = gx.GraphFile.from_csc(ip, ind)
    train = oracle.train_ids(n, 1, 0.2)
    plan = oracle.plan_seed_batches(train, 100, oracle.epoch_seed(1, 0))[:12]
    fan = [6, 4, 3]
    for K in (1500, 20000):      # changesets every iteration / all-fit
        d, r = str(tmp_path / f"gx{K}"), str(tmp_path / f"ref{K}")
        os.makedirs(d)
        os.makedirs(r)
        s = gx.sample_superbatch(g, None, plan, fan, 1, 3)
        s.write_files(d, 2)
        cs = s.precompute(n, K)
        cs.write_files(d, 2)
        rg.superbatch_sample(plan, fan, 1, 3, 2, r, 4)
        m, n_init = ref.precompute_changesets(r, 2, len(plan), n, K)
        assert np.array_equal(cs.misses(), m) and len(cs.init_set()) == n_init
        for stem in ("ids", "adj"):
            for i in range(len(plan)):
                a = open(os.path.join(d, f"{stem}_2_{i}.bin"), "rb").read()
                b = open(os.path.join(r, f"{stem}_2_{i}.bin"), "rb").read()
                assert a == b, (stem, i)
        assert _files(d, 2, len(plan)) == _files(r, 2, len(plan))
        if K == 1500:
            assert sum(len(cs.changeset(i).in_ids) for i in range(len(plan))) > 0
