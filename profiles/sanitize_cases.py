"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck) over the
hot-path kernels: the persistent grid-barrier sampler (k_sample), the inspector
with the Belady recurrence cutting every iteration (k_inspect, k_inspect_rec),
the changeset executor (k_gather_tma2, k_apply_slots, k_gather_rows), the
all-fit fan-out executor (k_fan_rows; the per-slot lists are built in
k_inspect), the deferred-ordering post-pass (k_sort_outs, k_finish_changesets)
and the LRU policy kernels. Each case checks its result against the oracle, so a
run that passes the sanitizer also passed parity.

    compute-sanitizer --tool memcheck python profiles/sanitize_cases.py
    GX_INSPECT_CTAS=8 GX_INSPECT_NEVER=2 compute-sanitizer ...   # the multi-CTA
        recurrence (eviction pool, ticket spins, NEVER fast path) on the same
        small traces, which otherwise run on one CTA
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2208_09151_b200 as gx  # noqa: E402

o = oracle.C
n, dim = 3000, 16
ip, ind = o.rmat_graph(n, 6.0, 11)
rows = o.features(n, dim, 12)
g = gx.GraphFile.from_csc(ip, ind)
f = gx.FeatureFile.from_array(rows)
plan = o.plan_seed_batches(o.train_ids(n, 1, 0.2), 48, o.epoch_seed(1, 0))[:6]
fan = [4, 3]
trace = [o.sample_batch(ip, ind, b, fan, o.derive_seed(1, i))[0] for i, b in enumerate(plan)]

# sampler + inspector (cut every iteration) + changeset executor
K = 150
p = gx.Pipeline(g, f, fan, K, digest=True)
st = p.run_superbatch(plan, 1, 0)
sim = o.simulate(trace, n, K, o.compute_init_set(trace, K, n))
assert np.array_equal(st.misses, sim["misses"]) and st.total_in > 0
for i, ids in enumerate(trace):
    assert np.array_equal(p.batch(i), rows[ids.astype(np.int64)])

# all-fit: fan-out executor
pf = gx.Pipeline(g, f, fan, n, digest=True)
sf = pf.run_superbatch(plan, 1, 0)
assert sf.fan_out and sf.total_misses == 0
for i, ids in enumerate(trace):
    assert np.array_equal(pf.batch(i), rows[ids.astype(np.int64)])

# FeatureCache API path: gather + apply_changeset with the precomputed changesets
cs = gx.precompute_trace(trace, n, K)
c = gx.FeatureCache(f, cs.init_set(), K)
for i, ids in enumerate(trace):
    b, _ = c.gather(f, ids)
    assert np.array_equal(b.numpy(), rows[ids.astype(np.int64)])
    c.apply_changeset(b, ids, cs.changeset(i))

# LRU policy
lru = gx.simulate_policy(trace, n, 64, "lru")
assert lru.total_accesses == sum(len(t) for t in trace)
print("sanitize cases ok:", st.sampled_edges, "edges,", st.total_in, "inserts,", int(lru.misses.sum()), "LRU misses")
