"""Belady-recurrence timing sweep (one B200): acceptance c8's traces
(acceptance.cpp:544-602: S = 512 / 1024 iterations of 64 fresh ids, K = 256)
through gx.precompute_trace, and the cfg1 pipeline's inspector stage (1M
nodes, K = 10 %: a cut every iteration), for several recurrence grid sizes
(GX_INSPECT_CTAS / GX_INSPECT_CLUSTER; each setting in a fresh process since
the knobs are read once).

    python profiles/inspect_sweep.py [ctas ...]  -> one JSON line per setting
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.environ["GX_ROOT"])
import paper_2208_09151_b200 as gx
out = {"setting": os.environ.get("GX_SWEEP_SETTING", "default")}
def c8(S):
    t = [np.arange(i * 64, (i + 1) * 64, dtype=np.uint64) for i in range(S)]
    best = 1e9
    for rep in range(6):
        t0 = time.perf_counter()
        cs = gx.precompute_trace(t, S * 64, 256)
        best = min(best, time.perf_counter() - t0)
    assert int(cs.misses().sum()) == S * 64 - 256
    return best
out["c8_s512_ms"] = 1e3 * c8(512)
out["c8_s1024_ms"] = 1e3 * c8(1024)
out["c8_ratio"] = out["c8_s1024_ms"] / out["c8_s512_ms"]
# cfg1 pipeline (configs[0]): inspector stage per superbatch
N, K = 1_000_000, 100_000
g = gx.GraphFile.generate_rmat(N, 10.0, gx.derive_seed(7, 0xED6E5))
f = gx.FeatureFile.generate(N, 128, gx.derive_seed(7, 0xFEA7))
plan = gx.plan_seed_batches(gx.derive_train_ids(N, 1, 0.1), 1000, gx.epoch_seed(1, 0)).batches
p = gx.Pipeline(g, f, [10, 10, 10], K)
for _ in range(3):
    st = p.run_superbatch(plan, 1, 0)
ins = []
for _ in range(5):
    st = p.run_superbatch(plan, 1, 0)
    ins.append(st.ms_inspect)
out["cfg1_inspect_ms"] = float(np.median(ins))
out["cfg1_inspect_us_per_iter"] = 1e3 * out["cfg1_inspect_ms"] / len(plan)
out["cfg1_misses"] = int(st.total_misses)
print(json.dumps(out))
"""

if __name__ == "__main__":
    # a setting is "default" or comma-separated ENV=VALUE pairs (GX_INSPECT_CTAS=16,GX_INSPECT_CLUSTER=16)
    settings = sys.argv[1:] or ["default", "GX_INSPECT_CTAS=1", "GX_INSPECT_CLUSTER=8", "GX_INSPECT_CLUSTER=16"]
    for c in settings:
        env = dict(os.environ, GX_ROOT=ROOT, GX_SWEEP_SETTING=c)
        if c != "default":
            env.update(kv.split("=", 1) for kv in c.split(","))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else json.dumps(
            {"setting": c, "error": r.stderr[-2000:]})
        print(line, flush=True)
