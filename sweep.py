#!/usr/bin/env python
"""sweep.py -- BASELINE.json configs[4]: changeset/gather stress sweep, superbatch
1-500 batches x cache 5-50 % on the papers100M-shape graph (one GPU; the
multi-GPU version of each point is bench.py's weak-scaling run).

Every point runs the fused device pipeline for `--steps` timed superbatches after
one warm-up and prints one JSON line (and appends it to --out)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers", choices=sorted(bench.CONFIGS))
    ap.add_argument("--superbatches", default="1,10,50,100,250,500")
    ap.add_argument("--cache", default="5,10,20,35,50")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=4,
                    help="untimed superbatches per point: each of the pipeline's two buffer slots grows to "
                         "the point's sizes (device buffers are grow-only) before the timed steps")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2208_09151_b200 as gx
    cfg = dict(bench.CONFIGS[args.config])
    ctx = gx.Context(0)
    g, f = bench.build_dataset(gx, cfg, ctx, lambda m: print(f"[sweep] {m}", file=sys.stderr))
    train = gx.derive_train_ids(cfg["N"], bench.SEED_RUN, cfg["train_fraction"])
    plan = gx.plan_seed_batches(train, cfg["batch"], gx.epoch_seed(bench.SEED_RUN, 0)).batches
    out = open(args.out, "a") if args.out else None
    for pct in [float(x) for x in args.cache.split(",")]:
        K = int(pct / 100 * cfg["N"])
        pipe = gx.Pipeline(g, f, cfg["fanouts"], K)
        for S in [int(x) for x in args.superbatches.split(",")]:
            sts = []
            for k in range(args.warmup + args.steps):
                o = (k * S) % max(len(plan) - S, 1)
                st = pipe.run_superbatch(plan[o:o + S], bench.SEED_RUN, o)
                if k >= args.warmup:
                    sts.append(st)
            ms = sum(s.ms_sample + s.ms_inspect + s.ms_switch + s.ms_gather for s in sts) / len(sts)
            edges = sum(s.sampled_edges for s in sts) / len(sts)
            rows = sum(s.gathered_rows for s in sts) / len(sts)
            rec = {"config": args.config, "superbatch": S, "cache_pct": pct, "cache_entries": K,
                   "ms_per_superbatch": ms, "sampled_edges_per_s": edges / (ms / 1e3),
                   "ms_sample": sum(s.ms_sample for s in sts) / len(sts),
                   "ms_inspect": sum(s.ms_inspect for s in sts) / len(sts),
                   "ms_switch": sum(s.ms_switch for s in sts) / len(sts),
                   "ms_gather_apply": sum(s.ms_gather for s in sts) / len(sts),
                   # feature bytes assembled per second of executor time (switch + gather + apply)
                   "gathered_GBps": rows * 4 * cfg["dim"] / (sum(s.ms_switch + s.ms_gather for s in sts) / len(sts) / 1e3) / 1e9,
                   "fused_fill": any(s.fused_fill for s in sts),
                   "miss_ratio": sum(s.total_misses for s in sts) / max(sum(s.gathered_rows for s in sts), 1),
                   "changeset_in_per_iter": sum(s.total_in for s in sts) / (len(sts) * S),
                   "observed_eq_predicted": all(s.total_misses == s.predicted_misses for s in sts)}
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
                out.flush()
        del pipe


if __name__ == "__main__":
    main()
