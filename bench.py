#!/usr/bin/env python
"""bench.py -- the Ginex data-preparation hot path on B200 (BASELINE.json metric).

One step = one superbatch of S batches through the whole hot path on one GPU:
    sample (S x batch seeds, fanout 10,10,10) -> Belady inspector (init set +
    S changesets) -> cache init ("switch") -> S x (gather batch rows, apply
    changeset)
on the papers100M-shape synthetic graph (configs[1]): 111,059,956 nodes,
~1.6B edges (R-MAT a/b/c/d = .57/.19/.19/.05, `gx gen --seed 7` seeds), 128-d
fp32 features, batch 1000, superbatch 100, cache 20% of the nodes. Graph and
feature table are generated on the device, bit-identical to the reference's
generator (tests/test_gpu_sampler.py::test_device_generator_matches_reference_generator).

value  = sampled edges / device time of the K timed steps (CUDA events on the
         pipeline's stream; max over ranks; whole-job edges over all ranks).
e2e    = the same through the public API call (host seeds uploaded per
         superbatch, per-iteration statistics read back), timed by the wall
         clock around the calls.
Extra keys: `cache_pressure` (the same superbatches with a 5 % cache: Belady
recurrence + changeset executor), `ssd_tier` (cfg1 with features.bin on the
box's storage, O_DIRECT reads vs the storage's sequential rate), `exchange`
(row-partitioned table, N > 1).
Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) unless a
launcher already did; the CSC is row-partitioned over the ranks (the sampler
reads remote lists over NVLink through CUDA IPC mappings); rank r runs
superbatches r, r+N, ... ("scaling": "weak"), or `--split batches` splits
every superbatch's batches into rank blocks ("strong").

--impl reference runs the UNMODIFIED reference (oracle/_ref/libgx_ref.so, the
reference headers compiled in this container) on the host cores, one full
superbatch (S = 100, K = 20 %) per step, on graph.bin/features.bin written to
/dev/shm by oracle/gen_dataset.cpp (byte-identical to generate_dataset); the
reference process loads neither torch nor the CUDA library.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED_GEN = 7    # `gx gen --seed 7` (gx.cpp:159-160)
SEED_RUN = 1    # run seed (pipeline.hpp:380-399)

CONFIGS = {
    # configs[1] of BASELINE.json: the bench workload
    # avg_degree 14.67 pre-dedup -> 1.615B edges after dedup (ogbn-papers100M: 1,615,685,872)
    "papers": dict(N=111_059_956, avg_degree=14.67, dim=128, fanouts=[10, 10, 10], batch=1000,
                   S=100, cache_frac=0.20, train_fraction=0.1,
                   workload="ogbn-papers100M-shape synthetic R-MAT: 111M nodes, ~1.6B edges, "
                            "128-d fp32, fanout (10,10,10), batch 1000, superbatch 100, cache 20%"),
    # configs[2]: com-friendster shape, 256-d features (1 KB rows, 67 GB table); K unspecified -> 10 %
    "friendster": dict(N=65_608_366, avg_degree=27.9, dim=256, fanouts=[10, 10, 10], batch=1000,
                       S=100, cache_frac=0.10, train_fraction=0.1,
                       workload="com-friendster-shape synthetic R-MAT: 65.6M nodes, ~1.8B edges, "
                                "256-d fp32, fanout (10,10,10), batch 1000, superbatch 100, cache 10%"),
    # configs[3]: MAG240M paper-subgraph shape, 768-d fp16 (scalar_width 2 extension): the
    # 187 GB table exceeds one B200, so it runs row-partitioned over >= 2 GPUs (--features
    # partitioned) -- 1.30B edges after dedup at avg_degree 10.75 pre-dedup
    "mag240m": dict(N=121_751_666, avg_degree=10.75, dim=768, dtype="fp16", fanouts=[10, 10, 10],
                    batch=1000, S=100, cache_frac=0.10, train_fraction=0.1, min_gpus_partitioned=2,
                    workload="MAG240M-shape paper subgraph synthetic R-MAT: 122M nodes, ~1.3B edges, "
                             "768-d fp16, fanout (10,10,10), batch 1000, superbatch 100, cache 10%"),
    # configs[0]: the reference's own CPU-runnable case
    "cfg1": dict(N=1_000_000, avg_degree=10.0, dim=128, fanouts=[10, 10, 10], batch=1000, S=100,
                 cache_frac=0.10, train_fraction=0.1,
                 workload="synthetic R-MAT 1M nodes / 9.7M edges, 128-d fp32, fanout (10,10,10), "
                          "batch 1000, superbatch 100, cache 10%"),
}


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """SM clock + throttle-reason sampling during the timed region
    (B200_PROFILING.md recipe). NVML every 5 ms (the timed region of a few
    superbatches lasts tens of ms); nvidia-smi polling when NVML is absent."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason* (HwSlowdown, HwThermal, SwThermal, SwPowerCap)

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, [4 bools])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device]) if vis and vis.split(",")[0].isdigit() else device
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
        try:
            r = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = n.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return (float(sm), float(mx), [bool(r & b) for b in self.BITS])

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        v = [x.strip() for x in out.split(",")]
        num = lambda x: float(x) if x.replace(".", "").isdigit() else None  # noqa: E731
        return (num(v[0]), num(v[1]), [x.lower() == "active" for x in v[2:6]])

    def _run(self):
        period = 0.005 if self._nvml else 0.2
        while True:
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            if self._stop.wait(period):
                break

    def __enter__(self):
        if self._nvml or shutil.which("nvidia-smi"):
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples if x[0] is not None]
        mx = [x[1] for x in self.samples if x[1] is not None]
        reasons = sorted({self.NAMES[k] for x in self.samples for k in range(4) if x[2][k]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml 5 ms" if self._nvml else "nvidia-smi"}


def build_dataset(gx, cfg, ctx, log, backing="device", ssd_dir=None, comm=None):
    edge_seed = gx.derive_seed(SEED_GEN, 0xED6E5)
    value_seed = gx.derive_seed(SEED_GEN, 0xFEA7)
    dtype = np.float16 if cfg.get("dtype") == "fp16" else np.float32
    t0 = time.time()
    g = gx.GraphFile.generate_rmat(cfg["N"], cfg["avg_degree"], edge_seed, ctx=ctx)
    t1 = time.time()
    if comm is not None:   # row-partitioned: this rank generates only its own rows
        f = gx.FeatureFile.partitioned_generate(cfg["N"], cfg["dim"], value_seed, comm, ctx, dtype=dtype)
    else:
        f = gx.FeatureFile.generate(cfg["N"], cfg["dim"], value_seed, ctx=ctx, dtype=dtype)
    ctx.synchronize()
    t2 = time.time()
    log(f"dataset: N={g.num_nodes()} E={g.num_edges()} (graph {t1 - t0:.1f}s, features {t2 - t1:.1f}s)")
    if backing == "file":
        # the SSD tier: features.bin on storage, the table leaves HBM
        path = os.path.join(ssd_dir, f"gx_bench_features_{os.getpid()}.bin")
        f.write(path)
        del f
        f = gx.FeatureFile.open(path, "file", ctx=ctx)
        os.unlink(path)  # the open descriptor keeps the inode readable
        log(f"features.bin written to {ssd_dir} ({time.time() - t2:.1f}s), "
            f"O_DIRECT={f.storage_stats().direct}")
    return g, f


def storage_seq_read_GBps(path, threads=16, chunk=8 << 20, limit=4 << 30):
    """The box's storage roofline for the SSD tier: sequential O_DIRECT reads of
    `path` (page-aligned buffers, `threads` readers on disjoint chunks), GB/s."""
    import mmap
    from concurrent.futures import ThreadPoolExecutor
    size = min(os.path.getsize(path), limit) // chunk * chunk
    if size == 0:
        return None
    try:
        fd = os.open(path, os.O_RDONLY | getattr(os, "O_DIRECT", 0))
    except OSError:
        fd = os.open(path, os.O_RDONLY)
    bufs = [mmap.mmap(-1, chunk) for _ in range(threads)]

    def work(t):
        n = 0
        for off in range(t * chunk, size, threads * chunk):
            n += os.preadv(fd, [bufs[t]], off)
        return n

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        got = sum(ex.map(work, range(threads)))
    dt = time.perf_counter() - t0
    os.close(fd)
    return got / dt / 1e9


def ssd_tier_line(gx, ctx, args, log):
    """The SSD tier in the driver's bench: configs[0] (cfg1, 1M nodes, K = 10 %)
    with features.bin on the box's storage (GX_BACKING_FILE: the init set and
    the misses are read with pread/O_DIRECT into pinned staging, storage.cu),
    against the storage's own sequential O_DIRECT read rate on the same file."""
    import torch
    cfg = dict(CONFIGS["cfg1"])
    g = gx.GraphFile.generate_rmat(cfg["N"], cfg["avg_degree"], gx.derive_seed(SEED_GEN, 0xED6E5), ctx=ctx)
    f = gx.FeatureFile.generate(cfg["N"], cfg["dim"], gx.derive_seed(SEED_GEN, 0xFEA7), ctx=ctx)
    path = os.path.join(args.ssd_dir, f"gx_bench_ssd_{os.getpid()}.bin")
    try:
        f.write(path)
        del f
        os.sync()
        peak = storage_seq_read_GBps(path)
        fb = gx.FeatureFile.open(path, "file", ctx=ctx)
    finally:
        if os.path.exists(path):
            os.unlink(path)  # an open descriptor keeps the inode readable
    sbs = make_plan(gx, cfg)
    K = int(cfg["cache_frac"] * cfg["N"])
    p = gx.Pipeline(g, fb, cfg["fanouts"], K)
    p.run_superbatch(sbs[0], SEED_RUN, 0)             # warm-up (staging buffers)
    fb_before = fb.storage_stats()
    stats = []
    xs = torch.cuda.ExternalStream(p.exec_stream, device=torch.device("cuda", ctx.device))
    st0 = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", ctx.device))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    e0.record(st0)
    for _ in range(2):
        stats.append(p.run_superbatch(sbs[0], SEED_RUN, 0))
    e1.record(xs)
    ctx.synchronize()
    torch.cuda.synchronize(ctx.device)
    secs = e0.elapsed_time(e1) / 1e3
    fs = fb.storage_stats()
    rows = sum(s.storage_rows for s in stats)
    byts = sum(s.storage_bytes for s in stats)
    ms_read = sum(s.ms_storage for s in stats)
    preads = fs.preads - fb_before.preads
    achieved = byts / (ms_read / 1e3) / 1e9 if ms_read else None
    for s in stats:
        assert s.total_misses == s.predicted_misses
    out = {
        "workload": cfg["workload"] + ", features.bin on storage (O_DIRECT)",
        "ms_per_superbatch": 1e3 * secs / len(stats),
        "sampled_edges_per_s": sum(s.sampled_edges for s in stats) / secs,
        "rows_read_per_superbatch": rows / len(stats),
        "storage_bytes_per_superbatch": byts / len(stats),
        "storage_read_ms_per_superbatch": ms_read / len(stats),
        "storage_GBps": achieved,
        "storage_MBps": achieved * 1e3 if achieved else None,
        "preads_per_s": preads / (ms_read / 1e3) if ms_read else None,
        "o_direct": fs.direct, "reader_threads": fs.threads, "dir": args.ssd_dir,
        "roofline": {"bound": "storage", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved and peak else None,
                     "peak_source": "measured here: sequential O_DIRECT reads of the same features.bin, 16 threads"},
        "page_accounting": {"gather_pages_read": sum(s.gather_io.pages_read for s in stats),
                            "note": "IoStats charged per missed row as the reference's FeatureFile does"},
    }
    log(f"ssd tier: {out['ms_per_superbatch']:.1f} ms/superbatch, {achieved} GB/s read vs {peak} GB/s sequential")
    return out


def make_plan(gx, cfg):
    train = gx.derive_train_ids(cfg["N"], SEED_RUN, cfg["train_fraction"])
    plan = gx.plan_seed_batches(train, cfg["batch"], gx.epoch_seed(SEED_RUN, 0)).batches
    S = cfg["S"]
    sbs = [plan[o:o + S] for o in range(0, len(plan), S)]
    return sbs


# ---------------------------------------------------------------------------
# the reference on the host cores (oracle/_ref) -- cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def ref_prepare(gx, g, f, cfg, samples, workdir, log):
    """graph.bin (persist_graph bytes) + a sparse features.bin holding the rows
    the sample touches, both in tmpfs, so the reference reads page-cache-warm.
    samples = [(batches, first_global_batch), ...] exactly as the reference runs them."""
    os.makedirs(workdir, exist_ok=True)
    gpath = os.path.join(workdir, "graph.bin")
    fpath = os.path.join(workdir, "features.bin")
    t0 = time.time()
    g.write(gpath)
    # features.bin header (FeatureWriter, graph_store.hpp:237-250), payload at 4096
    N, dim = cfg["N"], cfg["dim"]
    hdr = (b"GXFEAT01" + (1).to_bytes(4, "little") + N.to_bytes(8, "little") +
           dim.to_bytes(4, "little") + (4).to_bytes(4, "little") + (4096).to_bytes(8, "little"))
    with open(fpath, "wb") as fh:
        fh.write(hdr + b"\0" * (4096 - len(hdr)))
        fh.truncate(4096 + N * dim * 4)
    touched = []
    for batches, first in samples:
        s = gx.sample_superbatch(g, None, batches, cfg["fanouts"], SEED_RUN, first)
        touched += [s.batch(i).ids for i in range(len(s))]
    ids = np.unique(np.concatenate(touched))
    rows = f.read_rows(ids)
    mm = np.memmap(fpath, dtype=np.float32, mode="r+", offset=4096, shape=(N, dim))
    mm[ids.astype(np.int64)] = rows
    mm.flush()
    del mm
    log(f"reference inputs in {workdir}: {len(ids)} feature rows materialised ({time.time() - t0:.1f}s)")
    return gpath, fpath


def dropin_run(gx, ctx, g, cfg, batches, fpath, workdir, K, first_batch=0):
    """The reference's stage sequence (TrainingRunner::run_superbatch,
    pipeline.hpp:338-377) through this library's drop-in API: superbatch_sample
    writing the ids/adj runtime files -> precompute_changesets (init/update
    files) -> FeatureCache ctor on features.bin through the file tier (pread, as
    the reference's FeatureFile) -> per iteration read the ids/update files,
    gather into a host RowMatrix (pinned) and apply_changeset. Same inputs and
    files as the reference arm; the graph is the bench's (graph.bin was written
    from it) and the feature file is opened before the clock starts."""
    import torch
    f2 = gx.FeatureFile.open(fpath, "file", ctx=ctx)
    rt = os.path.join(workdir, "rt_dropin")
    shutil.rmtree(rt, ignore_errors=True)
    os.makedirs(rt)
    S = len(batches)
    t = [time.perf_counter()]
    res = gx.superbatch_sample(g, None, batches, cfg["fanouts"], SEED_RUN, first_batch, 0, rt)
    t.append(time.perf_counter())
    trace = gx.FileTrace([gx.api.ids_file_path(rt, 0, i) for i in range(S)])
    gx.precompute_changesets(trace, cfg["N"], K, rt, 0, ctx=ctx)
    t.append(time.perf_counter())
    cache = gx.FeatureCache(f2, gx.read_init_file(gx.api.init_file_path(rt, 0)), K)
    t.append(time.perf_counter())
    host = None
    rows = d2h = 0
    b = gx.Batch(ctx, f2.dim(), f2.dtype)  # one RowMatrix reused by every gather (as the reference's loop)
    loop = np.zeros(4)  # read files, gather, rows to host, apply
    for i in range(S):
        c0 = time.perf_counter()
        ids = gx.read_ids_file(gx.api.ids_file_path(rt, 0, i))
        cs = gx.read_update_file(gx.api.update_file_path(rt, 0, i))
        c1 = time.perf_counter()
        b, _ = cache.gather(f2, ids, out=b)
        n = b.rows
        c2 = time.perf_counter()
        if host is None or host.shape[0] < n:
            host = torch.empty((max(n, 1) * 5 // 4, f2.dim()), dtype=torch.float32, pin_memory=True).numpy()
        gx.api.check(gx.api.lib.gx_batch_copy_to_host(b.h, host.ctypes.data))
        c3 = time.perf_counter()
        rows += n
        d2h += n * f2.row_bytes()
        cache.apply_changeset(b, ids, cs)
        loop += np.diff([c0, c1, c2, c3, time.perf_counter()])
    ctx.synchronize()
    t.append(time.perf_counter())
    edges = sum(res_edges(gx.read_adj_file(gx.api.adj_file_path(rt, 0, i))) for i in range(S))
    shutil.rmtree(rt, ignore_errors=True)
    return dict(edges=edges, seconds=t[-1] - t[0], rows=rows, d2h=d2h,
                stages={"sample_files_s": t[1] - t[0], "precompute_files_s": t[2] - t[1],
                        "cache_ctor_s": t[3] - t[2], "main_loop_s": t[4] - t[3],
                        "loop_read_files_s": loop[0], "loop_gather_s": loop[1], "loop_rows_to_host_s": loop[2],
                        "loop_apply_s": loop[3]})


def res_edges(layers):
    return sum(len(e) for e in layers)


def ref_run(batches, cfg, gpath, fpath, workdir, workers, global_seed=SEED_RUN, first_batch=0):
    """One superbatch through the reference's own stages (oracle/_ref,
    gxr_run_superbatch): superbatch_sample with `workers` threads writing the
    ids/adj files -> precompute_changesets (init/update files) -> FeatureCache
    ctor -> per iteration read files, gather, apply_changeset. The files are
    opened before the clock starts; `seconds` is the sum of the four stages."""
    import oracle
    L = oracle.REF.lib
    import ctypes as C
    flat = np.concatenate([np.asarray(b, np.uint64) for b in batches])
    off = np.zeros(len(batches) + 1, np.uint64)
    off[1:] = np.cumsum([len(b) for b in batches])
    fan = np.asarray(cfg["fanouts"], np.uint32)
    rt = os.path.join(workdir, "rt")
    shutil.rmtree(rt, ignore_errors=True)
    os.makedirs(rt)
    times = np.zeros(4, np.float64)
    e, r, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
    K = int(cfg["cache_frac"] * cfg["N"])
    oracle.REF._chk(L.gxr_run_superbatch(gpath.encode(), fpath.encode(), rt.encode(), flat, off,
                                         len(batches), fan, len(fan), global_seed, first_batch, K,
                                         workers, times, C.byref(e), C.byref(r), C.byref(m)))
    shutil.rmtree(rt, ignore_errors=True)
    return dict(edges=e.value, rows=r.value, misses=m.value, seconds=float(times.sum()),
                stages={"sample_s": times[0], "precompute_s": times[1], "switch_s": times[2],
                        "main_loop_s": times[3]})


def ref_inputs(cfg, workdir, log):
    """graph.bin + features.bin of the bench workload, written on the host
    cores by oracle/gen_dataset.cpp -- byte-identical to the reference's
    generate_dataset (tests/test_oracle.py::test_threaded_generator_matches_reference)
    -- into tmpfs, so the reference reads page-cache-warm files. No CUDA."""
    import oracle
    os.makedirs(workdir, exist_ok=True)
    gpath = os.path.join(workdir, "graph.bin")
    fpath = os.path.join(workdir, "features.bin")
    es = oracle.C.derive_seed(SEED_GEN, 0xED6E5)
    vs = oracle.C.derive_seed(SEED_GEN, 0xFEA7)
    t0 = time.time()
    E = oracle.GEN.graph_file(gpath, cfg["N"], cfg["avg_degree"], es, cpu_cores())
    t1 = time.time()
    oracle.GEN.features_file(fpath, cfg["N"], cfg["dim"], vs, cpu_cores())
    t2 = time.time()
    log(f"reference inputs in {workdir}: N={cfg['N']} E={E} (graph.bin {t1 - t0:.1f}s, "
        f"features.bin {t2 - t1:.1f}s, {cpu_cores()} threads)")
    train = oracle.REF.train_ids(gpath, fpath, SEED_RUN, cfg["train_fraction"])
    plan = oracle.REF.plan_seed_batches(train, cfg["batch"], oracle.C.epoch_seed(SEED_RUN, 0))
    S = cfg["S"]
    sbs = [plan[o:o + S] for o in range(0, len(plan), S)]
    return gpath, fpath, sbs, E


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference_arm(args, cfg, log):
    """--impl reference: the UNMODIFIED reference (oracle/_ref/libgx_ref.so, its
    headers compiled in this container) on the host cores, on the same workload
    and config as the GPU arm. Neither torch nor the CUDA library is loaded:
    inputs come from the host-side writer, the seed plan from the reference's
    own TrainingRunner / plan_seed_batches. One step = one full superbatch
    (S batches, cache K) through the reference's stages."""
    rank, world, local = env_rank()
    if rank != 0:
        return
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgx_ref.so was not built"}))
        return
    workdir = f"/dev/shm/gx_bench_ref_{os.getpid()}"
    cores = cpu_cores()
    nb = args.ref_batches or cfg["S"]
    try:
        gpath, fpath, sbs, E = ref_inputs(cfg, workdir, log)
        res = []
        for k in range(args.warmup + args.steps):
            j = k % len(sbs)
            r = ref_run(sbs[j][:nb], cfg, gpath, fpath, workdir, cores, SEED_RUN, j * cfg["S"])
            if k >= args.warmup:
                res.append(r)
            log(f"reference step {k}: {r['edges']} edges in {r['seconds']:.2f}s {r['stages']}")
    finally:
        shutil.rmtree(workdir, ignore_errors=True)
    edges = sum(r["edges"] for r in res)
    secs = sum(r["seconds"] for r in res)
    v = edges / secs
    K = int(cfg["cache_frac"] * cfg["N"])
    sample = (f"{'every' if nb == cfg['S'] else f'first {nb} of the'} {cfg['S']} batches of superbatch k per "
              f"step through the reference's stages (superbatch_sample with {cores} workers + files, "
              f"precompute_changesets, FeatureCache init with K={K}, gather+apply); files opened "
              "outside the timed stages")
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "sampled_edges/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(len(res), 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 ids / f32 rows (byte copies)",
        "data": "synthetic (reference generator output, written by oracle/gen_dataset.cpp)",
        "config": bench_config(args, cfg, 1, K, E),   # one superbatch per step on the host
        "cpu_baseline": {"value": v, "unit": "sampled_edges/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "sampled_edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "stages": {k: sum(r["stages"][k] for r in res) / len(res) for k in res[0]["stages"]},
    }))


def bench_config(args, cfg, world, K, E):
    """The `config` object both arms print (same workload keys)."""
    S = cfg["S"]
    sb_per_step = world if args.split == "superbatch" else 1   # superbatches all ranks run per step
    return {"workload": cfg["workload"], "global_batch": cfg["batch"] * S * sb_per_step,
            "superbatch": S, "cache_entries": K, "num_edges": E,
            "features": args.features, "backing": args.backing,
            "l2": "inputs larger than L2 (57 GB table, 6.6 GB CSC)" if args.config == "papers"
            else "inputs larger than L2"}


METRIC = ("sampled edges/s through the full data-prep step (sample + Belady inspect + feature "
          "gather/cache update); gathered feature GB/s and HBM fraction in `stages`/`roofline`")


def relaunch(n):
    """`bench.py --gpus N` without a launcher: start N ranks on this node with
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gx", choices=["gx", "reference"])
    ap.add_argument("--config", default="papers", choices=sorted(CONFIGS))
    ap.add_argument("--avg-degree", type=float, default=None)
    ap.add_argument("--superbatch", type=int, default=None)
    ap.add_argument("--cache-frac", type=float, default=None, help="cache entries as a fraction of the nodes")
    ap.add_argument("--ref-batches", type=int, default=0,
                    help="batches per step for the reference / cpu_baseline sample (default: the whole superbatch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tiers", action="store_true",
                    help="skip the SSD-tier line (cfg1 with features.bin on storage, O_DIRECT)")
    ap.add_argument("--overlap", action="store_true",
                    help="two superbatches in flight: superbatch k's executor overlaps k+1's sampler/"
                         "inspector (slower on B200 at papers shape: the HBM-bound gather stretches the "
                         "barrier-bound inspector, DESIGN.md §6); default runs them back to back")
    ap.add_argument("--sync", action="store_true", help="(default) back-to-back superbatches")
    ap.add_argument("--backing", default="device", choices=["device", "file"],
                    help="feature backing store: HBM-resident table (default) or the SSD tier "
                         "(features.bin on storage, misses read with O_DIRECT into pinned staging)")
    ap.add_argument("--ssd-dir", default=os.environ.get("GX_SSD_DIR", "/tmp"))
    ap.add_argument("--features", default="replicated", choices=["replicated", "partitioned"],
                    help="replicated: every rank holds the whole table (no data-path collective); "
                         "partitioned: rows split over the ranks, cache init + misses fetched from "
                         "their owners by NCCL all-to-all (SURVEY.md 8e)")
    ap.add_argument("--graph", default="auto", choices=["auto", "replicated", "partitioned"],
                    help="CSC layout: replicated on every rank, or row-partitioned with the sampler "
                         "loading remote lists from their owner's HBM over NVLink (CUDA IPC); auto = "
                         "partitioned when N > 1")
    ap.add_argument("--pressure-frac", type=float, default=0.05,
                    help="also time the same superbatches with a cache of this fraction of the nodes "
                         "(the Belady recurrence + changeset executor regime; 0 = skip)")
    ap.add_argument("--split", default="superbatch", choices=["superbatch", "batches"],
                    help="superbatch: rank r runs superbatches r, r+N, ... (weak scaling); batches: every "
                         "superbatch's batches are split into N contiguous rank blocks (strong scaling)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "gx":
        return relaunch(args.gpus)
    cfg = dict(CONFIGS[args.config])
    if args.avg_degree is not None:
        cfg["avg_degree"] = args.avg_degree
    if args.superbatch is not None:
        cfg["S"] = args.superbatch
    if args.cache_frac is not None:
        cfg["cache_frac"] = args.cache_frac
    rank, world, local = env_rank()

    def log(m):
        if rank == 0:
            print(f"[bench] {m}", file=sys.stderr, flush=True)

    if args.impl == "reference":
        return run_reference_arm(args, cfg, log)

    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    import torch
    # GX_BENCH_SHARE_GPU=1 (tests on a one-GPU box): ranks share the visible
    # GPUs and talk over gloo, since NCCL refuses two ranks on one device
    share = os.environ.get("GX_BENCH_SHARE_GPU") == "1"
    local = local % torch.cuda.device_count() if share else local
    red_dev = "cpu" if share else f"cuda:{local}"
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        log(f"world {world}: torch.distributed {dist.get_backend()}"
            f"{' NCCL ' + '.'.join(map(str, torch.cuda.nccl.version())) if not share else ''}, "
            f"rank 0 on cuda:{local}")
    import paper_2208_09151_b200 as gx
    ctx = gx.Context(local)
    comm = None
    if args.features == "partitioned":
        uid = [gx.Comm.unique_id() if rank == 0 else None]
        if world > 1:
            torch.distributed.broadcast_object_list(uid, src=0)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)  # NCCL's version banner goes to stderr: stdout carries only the JSON line
        try:
            comm = gx.Comm.nccl(ctx, uid[0], world, rank)
        finally:
            os.dup2(saved, 1)
            os.close(saved)
    elif cfg.get("min_gpus_partitioned"):
        msg = (f"config {args.config} needs its table row-partitioned over >= "
               f"{cfg['min_gpus_partitioned']} GPUs (--features partitioned)")
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unavailable": msg}))
        return
    g, f = build_dataset(gx, cfg, ctx, log, args.backing, args.ssd_dir, comm)
    from paper_2208_09151_b200.shard import assign_superbatches, batch_block, partition_graph
    graph_layout = args.graph if args.graph != "auto" else ("partitioned" if world > 1 else "replicated")
    if graph_layout == "partitioned":
        try:
            partition_graph(g, rank, world)
            log(f"CSC row-partitioned over {world} ranks: this rank holds nodes "
                f"{g.partition_bounds(world)[rank:rank + 2].tolist()}, peers mapped over CUDA IPC")
        except Exception as e:   # e.g. no peer access between the GPUs: keep the whole CSC
            if g.partition_info()[0]:
                raise
            graph_layout = f"replicated (partitioning failed: {e})"
            log(f"CSC partitioning failed ({e}); every rank keeps the whole CSC")
    sbs = make_plan(gx, cfg)
    K_entries = int(cfg["cache_frac"] * cfg["N"])
    pipe = gx.Pipeline(g, f, cfg["fanouts"], K_entries, overlap=args.overlap)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    def sb_index(k):  # rank r takes superbatches r, r+world, ... of the epoch plan (split=superbatch)
        if args.split == "batches":
            return k % len(sbs)
        return assign_superbatches(len(sbs), rank, world, 1, start=k)[0]

    def rank_batches(j):
        """-> (this rank's batches of superbatch j, their first global batch index)"""
        if args.split == "batches":
            blk = batch_block(len(sbs[j]), rank, world)
            return sbs[j][blk.start:blk.stop], j * cfg["S"] + blk.start
        return sbs[j], j * cfg["S"]

    exec_stream = torch.cuda.ExternalStream(pipe.exec_stream, device=torch.device("cuda", local))

    def run_steps(k0, n, on_stats, ev_start=None, ev_end=None, pp=None, xs=None):
        """Two superbatches in flight: superbatch k+1 is submitted before k is
        waited for, so the host prepares k+1 while the GPU runs k. The GPU
        stages run back to back (default) or, with --overlap, k+1's
        sampler/inspector concurrently with k's executor."""
        pp = pp or pipe
        if ev_start is not None:
            ev_start.record(stream)
        prev = None
        for k in range(k0, k0 + n):
            b, first = rank_batches(sb_index(k))
            t = pp.submit(b, SEED_RUN, first)
            if prev is not None:
                on_stats(pp.wait(prev))
            prev = t
        if ev_end is not None:
            ev_end.record(xs or exec_stream)
        if prev is not None:
            on_stats(pp.wait(prev))

    def log_warm(st):
        log(f"warmup: {st.sampled_edges} edges, sample {st.ms_sample:.2f} ms inspect "
            f"{st.ms_inspect:.2f} ms switch {st.ms_switch:.2f} ms gather {st.ms_gather:.2f} ms")

    run_steps(0, args.warmup, log_warm)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        ctx.synchronize()
        torch.cuda.synchronize(local)

    stats = []
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        t_wall = time.perf_counter()
        run_steps(args.warmup, args.steps, stats.append, ev0, ev1)
        wall_s = time.perf_counter() - t_wall
        barrier()
    dev_s = ev0.elapsed_time(ev1) / 1e3
    edges = sum(s.sampled_edges for s in stats)
    if world > 1:
        t = torch.tensor([dev_s, wall_s], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_s, wall_s = t.tolist()
        e = torch.tensor([edges], device=red_dev, dtype=torch.float64)
        torch.distributed.all_reduce(e)
        edges_all = int(e.item())
    else:
        edges_all = edges
    for s in stats:
        assert s.total_misses == s.predicted_misses, "observed misses != inspector prediction"

    # --- e2e with the gathered rows returned to the host: a caller that consumes
    # batches on the CPU (the reference's RowMatrix) gets every iteration's rows
    # in pinned memory; submit + wait + one D2H per superbatch, wall clock
    e2e_rows = None
    if rank == 0 and world == 1 and not args.no_tiers:
        try:
            k0 = args.warmup + args.steps
            b0, f0 = rank_batches(sb_index(k0))
            pipe.wait(pipe.submit(b0, SEED_RUN, f0))
            nbytes = pipe.copy_superbatch(0, 0)
            host = torch.empty(int(nbytes * 1.25) + (1 << 20), dtype=torch.uint8, pin_memory=True)
            t0 = time.perf_counter()
            e_sum, b_sum = 0, 0
            for k in range(k0 + 1, k0 + 3):
                bk, fk = rank_batches(sb_index(k))
                stk = pipe.wait(pipe.submit(bk, SEED_RUN, fk))
                b_sum += pipe.copy_superbatch(host.data_ptr(), host.numel())
                e_sum += stk.sampled_edges
            dt = time.perf_counter() - t0
            e2e_rows = {"value": e_sum / dt, "unit": "sampled_edges/s", "d2h_GBps": b_sum / dt / 1e9,
                        "d2h_bytes_per_step": b_sum // 2, "h2d_bytes_per_step": int(8 * sum(len(b) for b in bk)),
                        "note": "2 superbatches, each: seeds in, sample + inspect + gather, then every "
                                "iteration's gathered rows copied to pinned host memory (one D2H); wall clock"}
            del host
        except Exception as e:
            e2e_rows = {"error": repr(e)}

    # --- cache-pressure line: the same superbatches through a small cache, so
    # the Belady recurrence and the changeset executor (not the all-fit path)
    # run inside the driver's bench (same graph and table, same timing rules)
    pressure = None
    if args.pressure_frac > 0:
        Kp = int(args.pressure_frac * cfg["N"])
        del pipe
        pp = gx.Pipeline(g, f, cfg["fanouts"], Kp, overlap=args.overlap)
        xs_p = torch.cuda.ExternalStream(pp.exec_stream, device=torch.device("cuda", local))
        run_steps(0, args.warmup, lambda st: None, pp=pp)
        pst = []
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run_steps(args.warmup, args.steps, pst.append, e0, e1, pp=pp, xs=xs_p)
        barrier()
        p_s = e0.elapsed_time(e1) / 1e3
        if world > 1:
            t = torch.tensor([p_s], device=red_dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            p_s = float(t.item())
        for s in pst:
            assert s.total_misses == s.predicted_misses, "observed misses != inspector prediction"
        n_p = len(pst)
        acc = sum(s.gathered_rows for s in pst)
        pressure = {
            "cache_entries": Kp, "cache_frac": args.pressure_frac,
            "ms_per_step": 1e3 * p_s / args.steps,
            "sampled_edges_per_s_rank0": sum(s.sampled_edges for s in pst) / p_s,
            "miss_ratio": sum(s.total_misses for s in pst) / max(acc, 1),
            "changeset_in_per_iter": sum(s.total_in for s in pst) / (n_p * cfg["S"]),
            "stages_ms": {"sample": sum(s.ms_sample for s in pst) / n_p,
                          "inspect (incl. Belady recurrence)": sum(s.ms_inspect for s in pst) / n_p,
                          ("switch (init rows fanned out to the accesses they serve)"
                           if any(s.init_fan for s in pst) else "switch (cache init)"):
                              sum(s.ms_switch for s in pst) / n_p,
                          "gather + apply": sum(s.ms_gather for s in pst) / n_p},
            "inspect_us_per_iteration": 1e3 * sum(s.ms_inspect for s in pst) / (n_p * cfg["S"]),
            "gather_GBps": (f.row_bytes() * sum(s.gather_kernel_rows for s in pst) /
                            (sum(s.ms_gather_kernels for s in pst) / 1e3) / 1e9
                            if sum(s.ms_gather_kernels for s in pst) else None),
            "note": "same superbatches as the headline with the cache at cache_frac of the nodes: misses and "
                    "changesets in every iteration (timed with CUDA events like the headline)"}
        del pp

    # --- rooflines: the gather (the north star's bandwidth kernel) and every stage --
    w = f.row_bytes()
    n = len(stats)
    rows = sum(s.gathered_rows for s in stats)                # accesses A
    rows_g = sum(s.gather_kernel_rows for s in stats)         # rows the gather launches moved
    gk_ms = sum(s.ms_gather_kernels for s in stats)
    g_row = 2 * w + 8                                         # read row + write row + u32 id + u32 slot
    alg_bytes = g_row * rows_g
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (gk_ms / 1e3) / 1e9 if gk_ms and alg_bytes else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("k_gather_dram_bytes_per_launch")
    step_ms = 1e3 * dev_s / args.steps

    def line(kernel, ms_tot, bytes_tot, bytes_formula, bound="hbm"):
        ms = ms_tot / n
        a = bytes_tot / (ms_tot / 1e3) / 1e9 if ms_tot else None
        return {"kernel": kernel, "ms_per_superbatch": ms, "share_of_step": ms / step_ms, "bound": bound,
                "achieved_GBps": a, "peak_GBps": peak, "frac": a / peak if a else None,
                "alg_bytes_per_superbatch": bytes_tot / n, "alg_bytes": bytes_formula}

    fused = any(s.fused_fill for s in stats)
    fan = any(s.fan_out for s in stats)
    ifan = any(getattr(s, "init_fan", False) for s in stats)
    staged = args.backing == "file" or comm is not None
    lists = sum(s.sample_io.neighbor_lists_read for s in stats)
    C = sum(s.total_in + s.total_out for s in stats)
    fills = sum(s.fill_rows for s in stats)
    samp = line("k_sample (stage: sampler)", sum(s.ms_sample for s in stats),
                24 * lists + 16 * edges + 8 * rows, "24*P + 16*E + 8*U (SURVEY 8d; P = parents expanded)",
                "random accesses (one scattered index read + one dedup-table probe/claim per draw)")
    # the sampler's own ceiling is a rate of scattered accesses, not bytes: one
    # draw = a random 4-byte index read + a dependent 8-byte table load/CAS,
    # measured alone at 21.4 G draws/s (profiles/random_sectors.cu ->
    # r02z_random_sectors.txt; 36.6 G/s for the index reads alone)
    ceil_dps = 21.4e9
    dps = edges / (sum(s.ms_sample for s in stats) / 1e3) if edges else None
    samp["random_access"] = {"achieved_draws_per_s": dps, "ceiling_draws_per_s": ceil_dps,
                             "frac": dps / ceil_dps if dps else None,
                             "ceiling_source": "profiles/r02z_random_sectors.txt (draw: idx4 -> probe8)",
                             "note": "whole sampler (every phase and layer) per draw; the draw loop alone "
                                     "(last-layer phase E) runs at ~1.2x the ceiling (hub repeats hit L2)"}
    rooflines = [
        samp,
        line("k_flatten + k_inspect (stage: inspector)", sum(s.ms_inspect for s in stats),
             24 * rows + 16 * C + 8 * fills, "24*A + 16*C + 8*|init| (SURVEY 8d)",
             "latency (random node-array atomics, grid barriers)"),
    ]
    fan_kernel = fan_bytes = fan_ms = None
    if fan and not staged:      # switch + every access in one kernel
        fan_kernel = "k_fan_rows (switch fanned out to every access)"
        fan_ms = sum(s.ms_switch for s in stats)
        fan_bytes = (3 * w + 12) * fills + (w + 4) * (rows - fills)
        rooflines.append(line(fan_kernel, fan_ms, fan_bytes,
                              "(3w + 12) per init row (read row, write slot + first-use row, id + first + range "
                              "end) + (w + 4) per other access (write batch row, list entry)"))
    elif fan:                   # staged tiers: the filled cache fans out
        rooflines.append(line("switch (storage / exchange scatter into slots)", sum(s.ms_switch for s in stats),
                              (2 * w + 8) * fills, "(2w + 8) per init row: write slot + first-use row, 2 ids "
                              "(device side)"))
        fan_kernel = "k_fan_rows (cache rows fanned out to the other accesses)"
        fan_ms = gk_ms
        fan_bytes = (w + 4) * fills + (w + 4) * (rows - fills)
        rooflines.append(line(fan_kernel, fan_ms, fan_bytes,
                              "<= (w + 4) per init row (read slot row if it has other accesses, range end) + "
                              "(w + 4) per other access (write batch row, list entry)"))
    elif ifan:                  # changesets: the init rows fanned out in the switch
        served = rows - rows_g  # accesses the init rows served
        fan_kernel = "switch: init rows fanned out (k_ifan_count + scan + k_ifan_place + k_fan_rows)"
        fan_ms = sum(s.ms_switch for s in stats)
        fan_bytes = (2 * w + 12) * fills + (w + 4) * served + 16 * rows
        rooflines += [
            line(fan_kernel, fan_ms, fan_bytes,
                 "(2w + 12) per init row (read row, write slot, id, count, range end) + (w + 4) per served "
                 "access (write batch row, list entry) + 16 per access (trace + slot, two passes)"),
            line("k_gather_rest (accesses the init rows do not serve) + miss counts", gk_ms,
                 (2 * w + 4) * rows_g + 8 * rows, "(2w + 4) per copied row + 8 per access (trace + slot)"),
        ]
    else:
        rooflines += [
            line("k_fill_first (switch fused with first uses)" if fused else "k_gather_rows<16,8> (switch: cache init)",
                 sum(s.ms_switch for s in stats), (3 * w + 8 if fused else 2 * w + 4) * fills,
                 "(3w + 8) per init row: read row, write slot + first batch row, 2 ids" if fused
                 else "(2w + 4) per init row: read row, write slot, id"),
            line("k_gather_tma2 (bulk-copy row gather)", gk_ms, alg_bytes,
                 "(2w + 8) per row: read row, write row, u32 id + u32 slot"),
        ]
    if fan or ifan:             # the headline roofline is the fan-out kernel
        achieved = fan_bytes / (fan_ms / 1e3) / 1e9
        traffic = None
        if os.path.exists(tp) and not staged and not ifan:   # captured on the device-backed all-fit fan-out
            with open(tp) as fh:
                traffic = json.load(fh).get("k_fan_dram_bytes_per_launch")
    S = cfg["S"]
    stages = {
        "sample_ms": sum(s.ms_sample for s in stats) / n,
        "inspect_ms": sum(s.ms_inspect for s in stats) / n,
        "switch_ms": sum(s.ms_switch for s in stats) / n,
        "gather_apply_ms": sum(s.ms_gather for s in stats) / n,
        "gather_kernels_ms": gk_ms / n,
        "apply_kernels_ms": sum(s.ms_apply_kernels for s in stats) / n,
        "sampler_edges_per_s": sum(s.sampled_edges for s in stats) / (sum(s.ms_sample for s in stats) / 1e3),
        # feature bytes assembled into batches per second of executor time (switch + gather + apply)
        "gathered_feature_GBps": w * rows / (sum(s.ms_switch + s.ms_gather for s in stats) / 1e3) / 1e9,
        "gather_kernel_rows_per_superbatch": rows_g / n,
        "fused_fill": fused,
        "fan_out": fan,
        "accesses_per_superbatch": rows / n,
        "miss_ratio": sum(s.total_misses for s in stats) / max(rows, 1),
        "init_size": stats[-1].init_size,
        "changeset_in_per_iter": sum(s.total_in for s in stats) / (n * S),
        "edges_per_superbatch": edges / n,
    }
    if comm is not None:
        xs = f.exchange_stats()
        stages.update({
            "exchange_ms": sum(s.ms_storage for s in stats) / n,
            "exchange_rows_per_superbatch": sum(s.storage_rows for s in stats) / n,
            "exchange_bytes_sent_total": xs.bytes_sent, "exchange_rows_remote_total": xs.rows_remote,
            "exchange_calls": xs.calls})
    if args.backing == "file":
        sm = sum(s.ms_storage for s in stats)
        sb = sum(s.storage_bytes for s in stats)
        srows = sum(s.storage_rows for s in stats)
        fs = f.storage_stats()
        stages.update({
            "storage_ms": sm / n, "storage_rows_per_superbatch": srows / n,
            "storage_bytes_per_superbatch": sb / n,
            "storage_GBps": sb / (sm / 1e3) / 1e9 if sm else None,
            "storage_row_GBps": srows * w / (sm / 1e3) / 1e9 if sm else None,
            "storage_preads_per_s": fs.preads / (fs.read_ms / 1e3) if fs.read_ms else None,
            "storage_direct": fs.direct, "storage_threads": fs.threads,
            "storage_dir": args.ssd_dir})
    out = {
        "metric": METRIC, "value": edges_all / dev_s, "unit": "sampled_edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.split == "batches" else "weak",
        "vs_baseline": None,
        "dtype": "u32 ids / f32 rows (byte copies)", "data": "synthetic (device R-MAT, bit-exact to the "
        "reference generator; feature_value table)",
        "config": bench_config(args, cfg, world, K_entries, g.num_edges()),
        "pipeline": ("2 superbatches in flight, GPU stages concurrent" if args.overlap else
                     "2 superbatches in flight, GPU stages back to back"),
        "parallelism": {
            "ranks": world,
            "split": ("superbatches r, r+N, ... per rank (weak scaling)" if args.split == "superbatch" else
                      "each superbatch's batches split into N contiguous rank blocks (strong scaling)"),
            "graph": graph_layout + (" (sampler loads remote lists over NVLink, CUDA IPC)"
                                     if graph_layout == "partitioned" and world > 1 else ""),
            "features": ("replicated (no data-path collective)" if comm is None else
                         f"{world}-way row-partitioned (NCCL all-to-all for cache init + misses)")},
        "e2e": {"value": edges_all / wall_s, "unit": "sampled_edges/s",
                "h2d_bytes_per_step": int(8 * sum(len(b) for b in sbs[0]) + 8 * (S + 1)),
                "d2h_bytes_per_step": int(8 * S + 8 * 16)},
        "gpu_launches": int(sum(s.kernel_launches for s in stats)),
        "roofline": ({"kernel": fan_kernel, "bound": "hbm", "achieved": achieved,
                      "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                      "peak_source": peak_src,
                      "init_rows_per_launch": fills / n, "accesses_per_launch": rows / n,
                      "alg_bytes_per_launch": fan_bytes / n,
                      "note": ("changeset superbatches: each init row is read once and written to its cache "
                               "slot and to every access it serves; the other accesses are copied from the table"
                               if ifan else
                               "all-fit superbatches: one launch per superbatch reads each init row once and "
                               "writes it to its cache slot and to the batch row of every access of its node"
                               if not staged else "staged tier: the scatter filled slots + first-use rows; the "
                               "cache rows fan out to the other accesses")}
                     if fan or ifan else
                     {"kernel": "k_gather_tma2 (bulk-copy row gather)", "bound": "hbm", "achieved": achieved,
                      "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                      "peak_source": peak_src,
                      "bytes_per_row": g_row,
                      "rows_per_launch": rows_g / max(1, sum(s.gather_launches for s in stats)),
                      "alg_bytes_per_launch": alg_bytes / max(1, sum(s.gather_launches for s in stats)),
                      "note": ("all-fit superbatches: the switch kernel also writes each init node's first-use "
                               "batch row, the gather moves the other accesses" if fused else None)}),
        "rooflines": rooflines,
        "stages": stages,
        "cache_pressure": pressure,
        "e2e_host_rows": e2e_rows,
        "clocks": clk.summary(),
    }
    if comm is not None:   # the NVLink tier: the row-partitioned table's all-to-all
        xms = stages["exchange_ms"] * n
        xb = stages["exchange_bytes_sent_total"]
        out["exchange"] = {
            "bound": "nvlink", "achieved": xb / (xms / 1e3) / 1e9 if xms else None, "peak": 900.0,
            "unit": "GB/s", "frac": (xb / (xms / 1e3) / 1e9) / 900.0 if xms else None,
            "note": "rows sent by this rank's exchanges over the timed steps / their wall time "
                    "(init + misses per superbatch); 900 GB/s = NVLink 5 per direction per GPU"}
    if rank == 0 and world == 1 and not args.no_tiers and args.backing == "device" and comm is None:
        try:
            out["ssd_tier"] = ssd_tier_line(gx, ctx, args, log)
        except Exception as e:  # the tier line never blocks the headline
            out["ssd_tier"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and comm is None:
        try:
            import oracle
            if oracle.ref_available():
                nb = args.ref_batches or cfg["S"]
                workdir = f"/dev/shm/gx_bench_cpu_{os.getpid()}"
                try:
                    gpath, fpath = ref_prepare(gx, g, f, cfg, [(sbs[0][:nb], 0)], workdir, log)
                    cores = cpu_cores()
                    r = ref_run(sbs[0][:nb], cfg, gpath, fpath, workdir, cores)
                    # the same superbatch and files through the drop-in API (host rows out)
                    try:
                        dropin_run(gx, ctx, g, cfg, sbs[0][:nb], fpath, workdir, K_entries)  # warm-up
                        dr = dropin_run(gx, ctx, g, cfg, sbs[0][:nb], fpath, workdir, K_entries)
                        out["e2e_dropin"] = {
                            "value": dr["edges"] / dr["seconds"], "unit": "sampled_edges/s",
                            "seconds_per_superbatch": dr["seconds"], "stages": dr["stages"],
                            "d2h_bytes_per_step": dr["d2h"], "rows": dr["rows"],
                            "vs_reference_same_sample": r["seconds"] / dr["seconds"],
                            "note": "the reference's stage sequence through the drop-in API on the same "
                                    "superbatch and files as cpu_baseline: superbatch_sample -> ids/adj files -> "
                                    "precompute_changesets -> init/update files -> FeatureCache on features.bin "
                                    "(file tier, pread) -> per iteration gather into pinned host rows + "
                                    "apply_changeset; wall clock, one superbatch after one untimed pass"}
                        log(f"drop-in API: {dr['edges']} edges in {dr['seconds']:.2f}s {dr['stages']}")
                    except Exception as e:  # never blocks the headline
                        out["e2e_dropin"] = {"error": repr(e)}
                finally:
                    shutil.rmtree(workdir, ignore_errors=True)
                out["cpu_baseline"] = {
                    "value": r["edges"] / r["seconds"], "unit": "sampled_edges/s", "cores": cores,
                    "kind": "reference",
                    "sample": f"{'all' if nb == cfg['S'] else f'the first {nb} of the'} {cfg['S']} batches of "
                              "superbatch 0 through the reference's stages "
                              f"(superbatch_sample {cores} workers, precompute_changesets, FeatureCache "
                              f"K={K_entries}, gather+apply); {r['edges']} edges in {r['seconds']:.2f}s",
                    "stages": r["stages"]}
            else:
                out["cpu_baseline"] = None
        except Exception as e:  # the baseline never blocks the GPU number
            out["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
