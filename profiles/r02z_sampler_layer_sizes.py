import sys, numpy as np
sys.path.insert(0, '.')
import bench
import paper_2208_09151_b200 as gx
cfg = bench.CONFIGS["papers"]
ctx = gx.Context(0)
g, f = bench.build_dataset(gx, cfg, ctx, print)
train = gx.derive_train_ids(cfg["N"], bench.SEED_RUN, cfg["train_fraction"])
plan = gx.plan_seed_batches(train, cfg["batch"], gx.epoch_seed(bench.SEED_RUN, 0)).batches
s = gx.sample_superbatch(g, None, plan[:100], cfg["fanouts"], bench.SEED_RUN, 0)
F = np.zeros((100, 4)); E = np.zeros((100, 3))
for b in range(100):
    o = s.batch(b)
    Fl = o.num_seeds
    F[b, 0] = Fl
    for l, e in enumerate(o.layers):
        E[b, l] = len(e)
        Fl = max(Fl, int(e[:, 0].max()) + 1 if len(e) else Fl)
        F[b, l + 1] = Fl
print("F per layer (mean, max):", F.mean(0), F.max(0))
print("draws per layer (mean, max):", E.mean(0), E.max(0))
for l in range(3):
    m = F[:, l].max() * (1 + cfg["fanouts"][l]) * 2
    h = 1024
    while h < m: h <<= 1
    print(f"layer {l}: H = {h} slots = {h*8/2**20:.1f} MiB per batch, {h*8*100/2**30:.2f} GiB per 100")
