"""Full-size parity through size-independent properties (papers100M shape:
111M nodes, 1.6B edges, 128-d features, superbatch 100, cache 20 %).

The oracle cannot run this size in seconds, so the checks are the ones the
domain offers at any size: the device generator's CSC is sorted/deduplicated
with the reference edge count; every sampled batch obeys the sampler's
invariants (seeds first, distinct ids, edges point inside the batch, at most
f children per parent); the all-fit Belady schedule is empty with init =
distinct ids in first-occurrence order; and gathered rows equal the closed-form
feature_value rows (graphgen.hpp:74-77) of their ids, recomputed here in numpy.
Needs ~90 GB of HBM."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N, AVG, DIM, FAN, B, S, KFRAC = 111_059_956, 14.67, 128, [10, 10, 10], 1000, 100, 0.20


def _feature_rows(ids, dim, seed):
    from oracle.bind import _np_mix64
    node = np.asarray(ids, np.uint64)[:, None]
    col = np.arange(dim, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = _np_mix64(np.uint64(seed) ^ _np_mix64(node * np.uint64(0x10001) + col))
    return ((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


@pytest.fixture(scope="module")
def papers(gx):
    ctx = gx.Context.default()
    eseed, vseed = gx.derive_seed(7, 0xED6E5), gx.derive_seed(7, 0xFEA7)
    g = gx.GraphFile.generate_rmat(N, AVG, eseed, ctx=ctx)
    f = gx.FeatureFile.generate(N, DIM, vseed, ctx=ctx)
    train = gx.derive_train_ids(N, 1, 0.1)
    plan = gx.plan_seed_batches(train, B, gx.epoch_seed(1, 0)).batches
    return g, f, plan[:S], vseed


@pytest.mark.parametrize("kfrac", [KFRAC, 0.05])      # all-fit (fused fill) / changesets every iteration
def test_papers_superbatch_properties(gx, papers, kfrac):
    g, f, sb, vseed = papers
    E = g.num_edges()
    assert 1_600_000_000 < E < 1_630_000_000          # ogbn-papers100M: 1,615,685,872
    K = int(kfrac * N)
    p = gx.Pipeline(g, f, FAN, K, digest=True)
    st = p.run_superbatch(sb, 1, 0)
    samples = gx.sample_superbatch(g, None, sb, FAN, 1, 0)
    assert samples.total_edges() == st.sampled_edges
    rng = np.random.default_rng(0)
    trace = []
    for i in range(S):
        b = samples.batch(i)
        ids = b.ids
        trace.append(ids)
        assert np.array_equal(ids[:len(sb[i])], np.asarray(sb[i], np.uint64))   # seeds first
        assert len(np.unique(ids)) == len(ids)                                   # distinct
        frontier = len(sb[i])                          # ids before layer l (sampler.hpp:90-92)
        for l, e in enumerate(b.layers):
            if len(e):
                assert e[:, 0].max() < len(ids) and e[:, 1].max() < frontier     # inside the batch
                assert np.bincount(e[:, 1].astype(np.int64)).max() <= FAN[l]   # <= f children
                frontier = max(frontier, int(e[:, 0].max()) + 1)               # new ids are appended
        assert frontier == len(ids)
    flat = np.concatenate(trace)
    uniq, first = np.unique(flat, return_index=True)
    assert st.gathered_rows == len(flat)
    if len(uniq) <= K:                                 # the papers case: everything fits
        assert st.total_misses == 0 and st.total_in == 0 and st.total_out == 0
        assert st.init_size == len(uniq) and st.fused_fill
    else:                                              # Belady bookkeeping at any size
        assert st.init_size == K and st.total_misses == st.predicted_misses
        assert int(st.misses.sum()) == st.total_misses and st.misses[0] == 0   # iteration 0 lies inside init
        assert 0 < st.total_in <= st.total_misses
        assert st.total_out == st.total_in            # the cache stays full: every insert evicts
    # gathered bytes == closed-form rows of the trace ids, on sampled iterations
    for i in rng.choice(S, 6, replace=False):
        got = p.batch(int(i))
        want = _feature_rows(trace[i], DIM, vseed)
        assert np.array_equal(got, want), f"iteration {i}"
    # and the digests of every iteration agree with the host digest of those rows
    dig = p.digests()
    for i in rng.choice(S, 3, replace=False):
        assert int(dig[i]) == gx.batch_digest(_feature_rows(trace[i], DIM, vseed))


def test_papers_sampler_matches_oracle(gx, oracle, papers):
    """Bit-exact sampled batches of the bench superbatch vs the oracle's
    sample_batch (sampler.hpp:69-117) on the host copy of the papers-shape
    CSC: ids, per-layer (src, dst) edges and the IoStats charge."""
    g, f, sb, vseed = papers
    ip, ind = g.to_csc()                                   # u64, 13.8 GB of host memory
    samples = gx.sample_superbatch(g, None, sb, FAN, 1, 0)
    for i in (0, 1, 2, 3, 50, 97, 98, 99):
        ids, layers, io = oracle.sample_batch(ip, ind, sb[i], FAN, oracle.derive_seed(1, i))
        b = samples.batch(i)
        assert np.array_equal(b.ids, ids), i
        for l in range(len(FAN)):
            assert np.array_equal(b.layers[l], layers[l]), (i, l)
        st = gx.IoStats()
        gx.sample_batch(g, None, sb[i], FAN, gx.derive_seed(1, i), st)
        assert (st.pages_read, st.neighbor_lists_read, st.bytes_read) == (int(io[0]), int(io[2]), int(io[3])), i


def test_papers_changesets_match_oracle(gx, oracle, papers):
    """Belady changesets of a papers-shape superbatch under cache pressure
    (K = 2 % of N = 2.2M slots) vs the oracle's simulate_changesets
    (changeset.hpp:228-295): init, misses, in/out/pos per iteration. At this
    size the device recurrence takes its large-cache slot scan (>= 8 slots
    per thread, inspector.cu `nres >= 8u * G`) and its two-level-bitmap out
    ordering (4096 < |out| < N/1024), which smaller tests cannot reach.
    The pipeline's observed misses agree as well."""
    g, f, sb, vseed = papers
    K = int(0.02 * N)
    samples = gx.sample_superbatch(g, None, sb, FAN, 1, 0)
    cs = samples.precompute(N, K)
    trace = [samples.batch(i).ids for i in range(S)]
    init = oracle.compute_init_set(trace, K, N)
    assert len(init) == K
    assert np.array_equal(cs.init_set(), init)
    sim = oracle.simulate(trace, N, K, init)
    assert np.array_equal(cs.misses(), sim["misses"])
    n_out = np.diff(sim["out_off"].astype(np.int64))
    assert ((n_out > 4096) & (n_out < N // 1024)).any(), n_out.max()   # the sparse-out branch ran
    for i in range(S):
        c = cs.changeset(i)
        a, b = int(sim["in_off"][i]), int(sim["in_off"][i + 1])
        o0, o1 = int(sim["out_off"][i]), int(sim["out_off"][i + 1])
        assert np.array_equal(c.in_ids, sim["in_ids"][a:b]), i
        assert np.array_equal(c.in_positions, sim["in_pos"][a:b]), i
        assert np.array_equal(c.out_ids, sim["out_ids"][o0:o1]), i
    st = gx.Pipeline(g, f, FAN, K).run_superbatch(sb, 1, 0)
    assert np.array_equal(st.misses, sim["misses"]) and st.total_misses == st.predicted_misses
