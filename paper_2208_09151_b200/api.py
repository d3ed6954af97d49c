"""Python mirror of the reference's host API for the data-preparation hot path.

Names, argument meaning and error behaviour follow the reference (Ginex "gx",
/root/reference/proj/include/gx): every call lands in libgx_b200.so's C-ABI
(include/gx_b200.h) and from there in sm_100a kernels. There is no CPU path:
without a B200 the first call that needs the device raises CudaError.

Exception mapping: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::logic_error -> LogicError, std::runtime_error -> RuntimeError,
std::overflow_error -> OverflowError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Callable, List, Optional, Sequence

import numpy as np

from ._lib import (ExchangeStatsC, IoStatsC, LogicError, PipelineStatsC, StorageStatsC, CudaError, check,  # noqa: F401
                   lib)

# ---------------------------------------------------------------------------
# primitives (common.hpp)
# ---------------------------------------------------------------------------
PAGE_SIZE = 4096
ITER_FLAG = 1 << 63
ITER_MASK = ITER_FLAG - 1
ITER_DUMMY = (1 << 64) - 1


def mix64(z: int) -> int:
    """common.hpp:90-95"""
    return lib.gx_mix64(z & 0xFFFFFFFFFFFFFFFF)


def derive_seed(base: int, index: int) -> int:
    """common.hpp:99-101"""
    return lib.gx_derive_seed(base & 0xFFFFFFFFFFFFFFFF, index & 0xFFFFFFFFFFFFFFFF)


def pages_touched(lo: int, hi: int) -> int:
    """common.hpp:48-52"""
    return lib.gx_pages_touched(lo, hi)


def page_count_for_row(row_bytes: int, row_index: int) -> int:
    """common.hpp:56-61"""
    out = C.c_uint64()
    check(lib.gx_page_count_for_row(row_bytes, row_index, C.byref(out)))
    return out.value


class SplitMix64:
    """common.hpp:68-87 (host-side; used for seed plans, as in the reference)."""

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def bounded(self, n: int) -> int:
        return (self.next() * n) >> 64


@dataclasses.dataclass
class IoStats:
    """common.hpp:32-45"""
    pages_read: int = 0
    rows_read: int = 0
    neighbor_lists_read: int = 0
    bytes_read: int = 0

    def __iadd__(self, o: "IoStats") -> "IoStats":
        self.pages_read += o.pages_read
        self.rows_read += o.rows_read
        self.neighbor_lists_read += o.neighbor_lists_read
        self.bytes_read += o.bytes_read
        return self

    def _add_c(self, c: IoStatsC) -> None:
        self.pages_read += c.pages_read
        self.rows_read += c.rows_read
        self.neighbor_lists_read += c.neighbor_lists_read
        self.bytes_read += c.bytes_read


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


# ---------------------------------------------------------------------------
# device context (one per process)
# ---------------------------------------------------------------------------
class Context:
    _default: Optional["Context"] = None

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.gx_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(int(os.environ.get("LOCAL_RANK", "0"))
                                   if os.environ.get("GX_USE_LOCAL_RANK") else 0)
        return cls._default

    def synchronize(self) -> None:
        check(lib.gx_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib.gx_ctx_stream(self.h)


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else Context.default()


# ---------------------------------------------------------------------------
# graph store (graph_store.hpp)
# ---------------------------------------------------------------------------
class GraphFile:
    """GraphFile (graph_store.hpp:106-197) with the whole CSC resident in HBM."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_graph_destroy(self.h)
            self.h = None

    @staticmethod
    def open(path: str, ctx: Optional[Context] = None) -> "GraphFile":
        """GraphFile::open (graph_store.hpp:108-133)"""
        c = _ctx(ctx)
        h = C.c_void_p()
        check(lib.gx_graph_open(c.h, os.fspath(path).encode(), C.byref(h)))
        return GraphFile(h, c)

    @staticmethod
    def from_csc(indptr, indices, ctx: Optional[Context] = None) -> "GraphFile":
        """From a CscGraph's arrays (graph_store.hpp:33-36)."""
        c = _ctx(ctx)
        ip, ind = _u64(indptr), _u64(indices)
        h = C.c_void_p()
        check(lib.gx_graph_from_csc(c.h, len(ip) - 1, _ptr(ip), _ptr(ind), C.byref(h)))
        return GraphFile(h, c)

    @staticmethod
    def generate_rmat(num_nodes: int, avg_degree: float, edge_seed: int, a: float = 0.57,
                      b: float = 0.19, c: float = 0.19, ctx: Optional[Context] = None) -> "GraphFile":
        """generate_edges + build_csc on the device (graphgen.hpp:55-70, graph_store.hpp:53-81)."""
        cx = _ctx(ctx)
        h = C.c_void_p()
        check(lib.gx_graph_generate_rmat(cx.h, num_nodes, float(avg_degree), a, b, c, edge_seed,
                                         C.byref(h)))
        return GraphFile(h, cx)

    def num_nodes(self) -> int:
        return lib.gx_graph_num_nodes(self.h)

    def num_edges(self) -> int:
        return lib.gx_graph_num_edges(self.h)

    def in_degree(self, v: int) -> int:
        out = C.c_uint64()
        check(lib.gx_graph_in_degree(self.h, v, C.byref(out)))
        return out.value

    def to_csc(self):
        ip = np.zeros(self.num_nodes() + 1, np.uint64)
        ind = np.zeros(max(self.num_edges(), 1), np.uint64)
        check(lib.gx_graph_copy_csc(self.h, ip.ctypes.data, ind.ctypes.data))
        return ip, ind[:self.num_edges()].copy()

    def write(self, path: str) -> None:
        """persist_graph (graph_store.hpp:83-98)"""
        check(lib.gx_graph_write(self.h, os.fspath(path).encode()))

    # -- row-partitioned CSC over the GPUs of one box (include/gx_b200.h)
    def partition_bounds(self, nranks: int) -> np.ndarray:
        """node bounds[nranks + 1] of the edge-balanced partition (no list is split)"""
        out = np.zeros(nranks + 1, np.uint64)
        check(lib.gx_graph_partition_bounds(self.h, nranks, out.ctypes.data))
        return out

    def partition(self, nranks: int, rank: int) -> "GraphFile":
        """keep only rank's in-neighbour lists (indptr stays replicated)"""
        check(lib.gx_graph_partition(self.h, nranks, rank))
        return self

    def ipc_handle(self) -> tuple:
        """-> (CUDA IPC handle bytes of this rank's lists, edge_lo, edge_hi)"""
        h = (C.c_uint8 * 64)()
        lo, hi = C.c_uint64(), C.c_uint64()
        check(lib.gx_graph_ipc_handle(self.h, h, C.byref(lo), C.byref(hi)))
        return bytes(h), lo.value, hi.value

    def attach_peers(self, handles: Sequence[tuple]) -> "GraphFile":
        """map every rank's partition (handles[q] = rank q's ipc_handle())"""
        buf = b"".join(h[0] for h in handles)
        lohi = np.array([x for h in handles for x in h[1:]], np.uint64)
        check(lib.gx_graph_attach_peers(self.h, buf, lohi.ctypes.data))
        self._peers = handles
        return self

    def attach_local(self, parts: Sequence["GraphFile"]) -> "GraphFile":
        """in-process form: parts[q] is rank q's graph (kept alive with this one)"""
        arr = (C.c_void_p * len(parts))(*[p.h.value if isinstance(p.h, C.c_void_p) else p.h for p in parts])
        check(lib.gx_graph_attach_local(self.h, arr, len(parts)))
        self._parts = list(parts)
        return self

    def partition_info(self) -> tuple:
        """-> (nranks (0 = whole CSC), rank, attached)"""
        n, r, a = C.c_int(), C.c_int(), C.c_int()
        check(lib.gx_graph_partition_info(self.h, C.byref(n), C.byref(r), C.byref(a)))
        return n.value, r.value, bool(a.value)


open_graph = GraphFile.open


# ---------------------------------------------------------------------------
# sampler (sampler.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class SampleOutput:
    """sampler.hpp:36-40: ids (seeds first, then discovery order) and per-layer
    (src_local, dst_local) u32 edge arrays of shape (E_l, 2)."""
    ids: np.ndarray
    num_seeds: int
    layers: List[np.ndarray]


@dataclasses.dataclass
class SeedPlan:
    batches: List[np.ndarray]


def plan_seed_batches(train_ids, batch_size: int, epoch_seed: int) -> SeedPlan:
    """sampler.hpp:48-65 (host-side sequential Fisher-Yates, in libgx_b200)."""
    t = _u64(train_ids)
    out = np.zeros(max(len(t), 1), np.uint64)
    check(lib.gx_plan_seed_batches(_ptr(t), len(t), batch_size, epoch_seed & 0xFFFFFFFFFFFFFFFF,
                                   out.ctypes.data))
    return SeedPlan([out[o:o + batch_size].copy() for o in range(0, len(t), batch_size)])


def derive_train_ids(num_nodes: int, seed: int, train_fraction: float) -> np.ndarray:
    """TrainingRunner::derive_train_ids (pipeline.hpp:384-399)."""
    out = np.zeros(max(num_nodes, 1), np.uint64)
    n = C.c_uint64()
    check(lib.gx_derive_train_ids(num_nodes, seed & 0xFFFFFFFFFFFFFFFF, float(train_fraction),
                                  out.ctypes.data, C.byref(n)))
    return out[:n.value].copy()


def epoch_seed(seed: int, epoch: int) -> int:
    """TrainingRunner::epoch_seed (pipeline.hpp:380-382)."""
    return lib.gx_epoch_seed(seed & 0xFFFFFFFFFFFFFFFF, epoch)


class Samples:
    """Device-resident result of sampling S batches (S x SampleOutput)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_samples_destroy(self.h)
            self.h = None

    def __len__(self) -> int:
        return lib.gx_samples_num_batches(self.h)

    @property
    def num_layers(self) -> int:
        return lib.gx_samples_num_layers(self.h)

    def total_edges(self) -> int:
        return lib.gx_samples_total_edges(self.h)

    def batch(self, b: int) -> SampleOutput:
        L = self.num_layers
        n_ids, n_seeds = C.c_uint64(), C.c_uint64()
        lc = np.zeros(max(L, 1), np.uint64)
        check(lib.gx_samples_batch_info(self.h, b, C.byref(n_ids), C.byref(n_seeds), lc.ctypes.data))
        ids = np.zeros(max(n_ids.value, 1), np.uint64)
        check(lib.gx_samples_copy_ids(self.h, b, ids.ctypes.data))
        layers = []
        for l in range(L):
            e = np.zeros((max(int(lc[l]), 1), 2), np.uint32)
            check(lib.gx_samples_copy_edges(self.h, b, l, e.ctypes.data))
            layers.append(e[:int(lc[l])].copy())
        return SampleOutput(ids[:n_ids.value].copy(), n_seeds.value, layers)

    def write_files(self, out_dir: str, sb_index: int) -> None:
        """write_ids_file / write_adj_file (sampler.hpp:132,147) for every batch."""
        os.makedirs(out_dir, exist_ok=True)
        check(lib.gx_samples_write_files(self.h, os.fspath(out_dir).encode(), sb_index))

    def precompute(self, num_nodes: int, num_entries: int) -> "Changesets":
        """precompute_changesets over this superbatch's device-resident trace
        (changeset.hpp:468-484 minus the file reads): the inspector path the
        fused pipeline runs (trusted sampler trace, gx_precompute_samples)."""
        h = C.c_void_p()
        check(lib.gx_precompute_samples(self.h, num_nodes, num_entries, C.byref(h)))
        return Changesets(h)


class NeighborCache:
    """Static neighbor cache (neighbor_cache.hpp). The CSC is HBM-resident, so
    the cache changes only the sampler's IoStats: a cached list charges nothing
    (sampler.hpp:91-97). build() = build_neighbor_cache (greedy by out/in
    degree within a byte budget), open()/write() = ncache.bin."""

    def __init__(self, handle, graph: GraphFile):
        self.h = handle
        self.graph = graph

    def __del__(self):
        if getattr(self, "h", None):
            g = getattr(self, "graph", None)
            if g is not None and getattr(g, "_ncache", None) is self:
                lib.gx_graph_set_neighbor_cache(g.h, None)
            lib.gx_ncache_destroy(self.h)
            self.h = None

    @staticmethod
    def build(graph: GraphFile, budget_bytes: int, stats: Optional[IoStats] = None) -> "NeighborCache":
        io = IoStatsC()
        h = C.c_void_p()
        check(lib.gx_ncache_build(graph.h, budget_bytes, C.byref(io), C.byref(h)))
        if stats is not None:
            stats._add_c(io)
        return NeighborCache(h, graph)

    @staticmethod
    def open(graph: GraphFile, path: str, stats: Optional[IoStats] = None) -> "NeighborCache":
        io = IoStatsC()
        h = C.c_void_p()
        check(lib.gx_ncache_open(graph.h, os.fspath(path).encode(), C.byref(io), C.byref(h)))
        if stats is not None:
            stats._add_c(io)
        return NeighborCache(h, graph)

    def write(self, path: str) -> None:
        check(lib.gx_ncache_write(self.h, os.fspath(path).encode()))

    def cached_node_count(self) -> int:
        return lib.gx_ncache_cached_nodes(self.h)

    def bytes_used(self) -> int:
        return lib.gx_ncache_bytes_used(self.h)

    def contains(self, v: int) -> bool:
        out = C.c_int()
        check(lib.gx_ncache_contains(self.h, v, C.byref(out)))
        return bool(out.value)


build_neighbor_cache = NeighborCache.build
load_neighbor_cache = NeighborCache.open


class _UseNcache:
    """Installs `cache` on the graph for one sampler call (the reference passes
    it per call, sampler.hpp:69,197)."""

    def __init__(self, graph: GraphFile, cache):
        if cache is not None and not isinstance(cache, NeighborCache):
            raise TypeError("cache must be a NeighborCache or None")
        if cache is not None and cache.graph.num_nodes() != graph.num_nodes():
            raise ValueError("neighbor cache and graph disagree on node count")
        self.graph, self.cache = graph, cache

    def __enter__(self):
        check(lib.gx_graph_set_neighbor_cache(self.graph.h, self.cache.h if self.cache is not None else None))

    def __exit__(self, *a):
        lib.gx_graph_set_neighbor_cache(self.graph.h, None)


def _fan(fanouts: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(list(fanouts), dtype=np.uint32).reshape(-1))


def sample_batch(graph: GraphFile, cache, seeds, fanouts: Sequence[int], batch_seed: int,
                 stats: Optional[IoStats] = None) -> SampleOutput:
    """sample_batch (sampler.hpp:69-117)."""
    s, f = _u64(seeds), _fan(fanouts)
    io = IoStatsC()
    h = C.c_void_p()
    with _UseNcache(graph, cache):
        check(lib.gx_sample_batch(graph.h, _ptr(s), len(s), _ptr(f), len(f),
                                  batch_seed & 0xFFFFFFFFFFFFFFFF, C.byref(h), C.byref(io)))
    if stats is not None:
        stats._add_c(io)
    return Samples(h).batch(0)


def _flatten(batches) -> tuple:
    lists = [_u64(b) for b in batches]
    off = np.zeros(len(lists) + 1, np.uint64)
    if lists:
        off[1:] = np.cumsum([len(x) for x in lists])
    flat = np.concatenate(lists) if lists and off[-1] else np.zeros(1, np.uint64)
    return flat, off


def sample_superbatch(graph: GraphFile, cache, batch_slice, fanouts: Sequence[int], global_seed: int,
                      first_global_batch: int, stats: Optional[IoStats] = None) -> Samples:
    """superbatch_sample's sampling part (sampler.hpp:197-243); result stays on the device."""
    flat, off = _flatten(batch_slice)
    f = _fan(fanouts)
    io = IoStatsC()
    h = C.c_void_p()
    with _UseNcache(graph, cache):
        check(lib.gx_sample_superbatch(graph.h, flat.ctypes.data, off.ctypes.data, len(off) - 1, _ptr(f),
                                       len(f), global_seed & 0xFFFFFFFFFFFFFFFF, first_global_batch,
                                       C.byref(h), C.byref(io)))
    if stats is not None:
        stats._add_c(io)
    return Samples(h)


@dataclasses.dataclass
class SuperbatchSampleResult:
    """sampler.hpp:188-192"""
    io: IoStats
    files_written: int
    batches: int


def superbatch_sample(graph: GraphFile, cache, batch_slice, fanouts: Sequence[int], global_seed: int,
                      first_global_batch: int, sb_index: int, out_dir: str,
                      workers: int = 1) -> SuperbatchSampleResult:
    """superbatch_sample (sampler.hpp:197-243): samples and writes ids/adj files.
    `workers` is accepted for signature parity; the device path has no host pool."""
    io = IoStats()
    s = sample_superbatch(graph, cache, batch_slice, fanouts, global_seed, first_global_batch, io)
    s.write_files(out_dir, sb_index)
    n = len(batch_slice)
    return SuperbatchSampleResult(io, 2 * n, n)


# ---------------------------------------------------------------------------
# runtime files (FORMATS.md; sampler.hpp:123-182, changeset.hpp:409-454)
# ---------------------------------------------------------------------------
def ids_file_path(d, sb, i):
    return os.path.join(d, f"ids_{sb}_{i}.bin")


def adj_file_path(d, sb, i):
    return os.path.join(d, f"adj_{sb}_{i}.bin")


def init_file_path(d, sb):
    return os.path.join(d, f"init_{sb}.bin")


def update_file_path(d, sb, i):
    return os.path.join(d, f"update_{sb}_{i}.bin")


def _read(path, magic: bytes) -> memoryview:
    with open(path, "rb") as fh:
        b = fh.read()
    if len(b) < 8 or b[:8] != magic:
        raise RuntimeError(f"bad magic in {path} (expected {magic.decode()})")
    return memoryview(b)


def _u64_at(b, pos, path):
    if len(b) < pos + 8:
        raise RuntimeError(f"truncated file: {path}")
    return int.from_bytes(b[pos:pos + 8], "little"), pos + 8


def _arr_at(b, pos, n, path):
    if len(b) < pos + 8 * n:
        raise RuntimeError(f"truncated file: {path}")
    return np.frombuffer(b[pos:pos + 8 * n], dtype="<u8").astype(np.uint64), pos + 8 * n


def read_ids_file(path) -> np.ndarray:
    b = _read(path, b"GXIDS001")
    n, p = _u64_at(b, 8, path)
    return _arr_at(b, p, n, path)[0]


def read_adj_file(path) -> List[np.ndarray]:
    b = _read(path, b"GXADJ001")
    if len(b) < 12:
        raise RuntimeError(f"truncated file: {path}")
    L = int.from_bytes(b[8:12], "little")
    p = 12
    out = []
    for _ in range(L):
        n, p = _u64_at(b, p, path)
        if len(b) < p + 8 * n:
            raise RuntimeError(f"truncated file: {path}")
        out.append(np.frombuffer(b[p:p + 8 * n], dtype="<u4").reshape(-1, 2).astype(np.uint32))
        p += 8 * n
    return out


def write_ids_file(path, ids) -> None:
    a = _u64(ids)
    with open(path, "wb") as fh:
        fh.write(b"GXIDS001" + len(a).to_bytes(8, "little") + a.astype("<u8").tobytes())


def write_adj_file(path, layers) -> None:
    with open(path, "wb") as fh:
        fh.write(b"GXADJ001" + len(layers).to_bytes(4, "little"))
        for e in layers:
            e = np.asarray(e, dtype="<u4").reshape(-1, 2)
            fh.write(len(e).to_bytes(8, "little") + e.tobytes())


def read_init_file(path) -> np.ndarray:
    b = _read(path, b"GXINIT01")
    n, p = _u64_at(b, 8, path)
    return _arr_at(b, p, n, path)[0]


@dataclasses.dataclass
class Changeset:
    """changeset.hpp:161-167: in_ids by position, out_ids by id."""
    in_ids: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint64))
    out_ids: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint64))
    in_positions: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.uint64))

    def __eq__(self, o) -> bool:
        return (np.array_equal(self.in_ids, o.in_ids) and np.array_equal(self.out_ids, o.out_ids)
                and np.array_equal(self.in_positions, o.in_positions))


def read_update_file(path) -> Changeset:
    b = _read(path, b"GXUPD001")
    p = 8
    n, p = _u64_at(b, p, path)
    a, p = _arr_at(b, p, n, path)
    n, p = _u64_at(b, p, path)
    o, p = _arr_at(b, p, n, path)
    n, p = _u64_at(b, p, path)
    q, p = _arr_at(b, p, n, path)
    if len(q) != len(a):
        raise RuntimeError(f"update file is inconsistent: {path}")
    return Changeset(a, o, q)


# ---------------------------------------------------------------------------
# inspector (changeset.hpp)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class AccessIndex:
    """changeset.hpp:61-71"""
    iters: np.ndarray
    ptr: np.ndarray

    def total_accesses(self) -> int:
        return len(self.iters) - 1

    def access_count(self, v: int) -> int:
        end = int(self.ptr[v + 1]) if v + 1 < len(self.ptr) else self.total_accesses()
        return end - int(self.ptr[v])


@dataclasses.dataclass
class SimulationResult:
    """changeset.hpp:169-178"""
    misses: np.ndarray
    total_accesses: int

    def total_misses(self) -> int:
        return int(np.sum(self.misses, dtype=np.uint64))


class Changesets:
    """Device-resident output of the inspector for one superbatch."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_changesets_destroy(self.h)
            self.h = None

    def __len__(self):
        return lib.gx_changesets_num_iters(self.h)

    def init_set(self) -> np.ndarray:
        n = lib.gx_changesets_init_size(self.h)
        out = np.zeros(max(n, 1), np.uint64)
        m = C.c_uint64()
        check(lib.gx_changesets_init(self.h, out.ctypes.data, C.byref(m)))
        return out[:m.value].copy()

    def misses(self) -> np.ndarray:
        out = np.zeros(max(len(self), 1), np.uint64)
        check(lib.gx_changesets_misses(self.h, out.ctypes.data))
        return out[:len(self)].copy()

    def changeset(self, i: int) -> Changeset:
        ni, no, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.gx_changesets_iter_info(self.h, i, C.byref(ni), C.byref(no), C.byref(m)))
        a = np.zeros(max(ni.value, 1), np.uint64)
        p = np.zeros(max(ni.value, 1), np.uint64)
        o = np.zeros(max(no.value, 1), np.uint64)
        check(lib.gx_changesets_copy_iter(self.h, i, a.ctypes.data, o.ctypes.data, p.ctypes.data))
        return Changeset(a[:ni.value].copy(), o[:no.value].copy(), p[:ni.value].copy())

    def write_files(self, out_dir: str, sb_index: int) -> None:
        os.makedirs(out_dir, exist_ok=True)
        check(lib.gx_changesets_write_files(self.h, os.fspath(out_dir).encode(), sb_index))


class MemoryTrace:
    """changeset.hpp:44-48: one deduplicated id list per iteration."""

    def __init__(self, trace):
        self.trace = [_u64(t) for t in trace]

    def iterations(self) -> int:
        return len(self.trace)

    def ids(self, i: int) -> np.ndarray:
        return self.trace[i]


class FileTrace:
    """changeset.hpp:51-55"""

    def __init__(self, files):
        self.files = list(files)

    def iterations(self) -> int:
        return len(self.files)

    def ids(self, i: int) -> np.ndarray:
        return read_ids_file(self.files[i])


def _trace_lists(trace):
    if isinstance(trace, (MemoryTrace, FileTrace)):
        return [trace.ids(i) for i in range(trace.iterations())]
    return [_u64(t) for t in trace]


def build_access_index(trace, num_nodes: int, ctx: Optional[Context] = None) -> AccessIndex:
    """build_access_index (changeset.hpp:124-129), computed on the device."""
    flat, off = _flatten(_trace_lists(trace))
    A = int(off[-1])
    iters = np.zeros(A + 1, np.uint64)
    ptr = np.zeros(max(num_nodes, 1), np.uint64)
    check(lib.gx_access_index(_ctx(ctx).h, flat.ctypes.data, off.ctypes.data, len(off) - 1, num_nodes,
                              iters.ctypes.data, ptr.ctypes.data))
    return AccessIndex(iters, ptr[:num_nodes].copy())


def precompute_trace(trace, num_nodes: int, num_entries: int, init=None,
                     ctx: Optional[Context] = None) -> Changesets:
    """compute_init_set + simulate_changesets on the device (changeset.hpp:137-295)."""
    flat, off = _flatten(_trace_lists(trace))
    h = C.c_void_p()
    if init is None:
        check(lib.gx_precompute_trace(_ctx(ctx).h, flat.ctypes.data, off.ctypes.data, len(off) - 1,
                                      num_nodes, num_entries, C.byref(h)))
    else:
        iv = _u64(init)
        check(lib.gx_simulate_trace(_ctx(ctx).h, flat.ctypes.data, off.ctypes.data, len(off) - 1,
                                    num_nodes, num_entries, _ptr(iv), len(iv), C.byref(h)))
    return Changesets(h)


# ---------------------------------------------------------------------------
# comparison policies of `gx simulate` (baselines.hpp)
# ---------------------------------------------------------------------------
POLICIES = ("none", "static_degree", "lru", "belady")


def parse_policy(s: str) -> str:
    """parse_policy (baselines.hpp:24-30)."""
    if s not in POLICIES:
        raise ValueError("unknown policy: " + s)
    return s


@dataclasses.dataclass
class PolicyResult:
    """PolicyResult (baselines.hpp:32-48)."""
    policy: str
    capacity: int
    misses: np.ndarray
    total_accesses: int

    def total_misses(self) -> int:
        return int(np.sum(self.misses, dtype=np.uint64))

    def miss_ratio(self) -> float:
        return 0.0 if self.total_accesses == 0 else self.total_misses() / self.total_accesses


def static_degree_set(graph: GraphFile, num_entries: int) -> np.ndarray:
    """static_degree_set (baselines.hpp:50-62) with out-degrees from the graph's CSC."""
    out = np.zeros(max(num_entries, 1), np.uint64)
    check(lib.gx_static_degree_set(graph.h, num_entries, out.ctypes.data))
    return out[:num_entries].copy()


def simulate_policy(trace, num_nodes: int, num_entries: int, policy: str,
                    graph: Optional[GraphFile] = None, ctx: Optional[Context] = None) -> PolicyResult:
    """simulate_policy (baselines.hpp:64-143). static_degree takes its
    out-degrees from `graph` (the reference takes them as a span); belady is
    the inspector; lru the device stack-distance count (gx_simulate_lru)."""
    policy = parse_policy(policy)
    lists = _trace_lists(trace)
    total = int(sum(len(x) for x in lists))
    if policy == "none":
        return PolicyResult(policy, num_entries, np.array([len(x) for x in lists], np.uint64), total)
    if policy == "static_degree":
        if graph is None or graph.num_nodes() != num_nodes:
            raise ValueError("static_degree requires out-degrees (pass the graph)")
        flat, off = _flatten(lists)
        m = np.zeros(max(len(lists), 1), np.uint64)
        check(lib.gx_simulate_static_degree(graph.h, flat.ctypes.data, off.ctypes.data, len(lists), num_entries,
                                            m.ctypes.data))
        return PolicyResult(policy, num_entries, m[:len(lists)].copy(), total)
    if policy == "belady":
        cs = precompute_trace(lists, num_nodes, num_entries, ctx=ctx)
        return PolicyResult(policy, num_entries, cs.misses().astype(np.uint64), total)
    # lru: LRU stack distances on the device (gx_simulate_lru, baselines.cu)
    flat, off = _flatten(lists)
    m = np.zeros(max(len(lists), 1), np.uint64)
    check(lib.gx_simulate_lru(_ctx(ctx).h, flat.ctypes.data, off.ctypes.data, len(lists), num_nodes, num_entries,
                              m.ctypes.data))
    return PolicyResult(policy, num_entries, m[:len(lists)].copy(), total)


def compute_init_set(trace, num_entries: int, num_nodes: int,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """compute_init_set (changeset.hpp:137-153)."""
    if num_entries == 0:
        for t in _trace_lists(trace):  # the reference returns early without checks
            pass
        return np.zeros(0, np.uint64)
    return precompute_trace(trace, num_nodes, num_entries, ctx=ctx).init_set()


def simulate_changesets(index: Optional[AccessIndex], trace, num_entries: int, init,
                        sink: Optional[Callable] = None, num_nodes: Optional[int] = None,
                        ctx: Optional[Context] = None) -> SimulationResult:
    """simulate_changesets (changeset.hpp:228-295). `index` is accepted for
    signature parity (the device recomputes next-use itself); sink(i, cs, state)
    receives the sorted state after each update, reconstructed on the host."""
    lists = _trace_lists(trace)
    if num_nodes is None:
        if index is None:
            raise ValueError("num_nodes is required without an AccessIndex")
        num_nodes = len(index.ptr)
    cs = precompute_trace(lists, num_nodes, num_entries, init=_u64(init), ctx=ctx)
    misses = cs.misses()
    if sink is not None:
        state = set(int(v) for v in _u64(init))
        for i in range(len(lists)):
            c = cs.changeset(i)
            state.difference_update(int(v) for v in c.out_ids)
            state.update(int(v) for v in c.in_ids)
            sink(i, c, np.array(sorted(state), dtype=np.uint64))
    return SimulationResult(misses, int(sum(len(t) for t in lists)))


@dataclasses.dataclass
class PrecomputeResult:
    """changeset.hpp:460-464"""
    files_written: int
    sim: SimulationResult
    init_size: int


def precompute_changesets(trace: FileTrace, num_nodes: int, num_entries: int, out_dir: str,
                          sb_index: int, ctx: Optional[Context] = None) -> PrecomputeResult:
    """precompute_changesets (changeset.hpp:468-484): init + update files."""
    lists = _trace_lists(trace)
    cs = precompute_trace(lists, num_nodes, num_entries, ctx=ctx)
    cs.write_files(out_dir, sb_index)
    sim = SimulationResult(cs.misses(), int(sum(len(t) for t in lists)))
    return PrecomputeResult(len(lists) + 1, sim, len(cs.init_set()))


# ---------------------------------------------------------------------------
# executor (feature_cache.hpp) and the feature table (graph_store.hpp:217-333)
# ---------------------------------------------------------------------------
BACKING = {"device": 0, "host": 1, "file": 2}


def partition_bounds(num_nodes: int, nranks: int, rank: int) -> tuple:
    """Rows [lo, hi) rank `rank` of `nranks` owns: [N*r/P, N*(r+1)/P)."""
    lo, hi = C.c_uint64(), C.c_uint64()
    check(lib.gx_partition_bounds(num_nodes, nranks, rank, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


_HOST_XCHG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                         C.POINTER(C.c_uint64))


class Comm:
    """Communicator of a row-partitioned feature table: NCCL (one process per
    GPU) or the in-process hub (one host thread per rank, for tests)."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_comm_destroy(self.h)
            self.h = None

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib.gx_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(ctx: Context, uid: bytes, nranks: int, rank: int) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib.gx_comm_init_nccl(ctx.h, buf, nranks, rank, C.byref(h)))
        return Comm(h, ctx)

    @staticmethod
    def local(ctxs: Sequence[Context]) -> List["Comm"]:
        n = len(ctxs)
        arr = (C.c_void_p * n)(*[c.h.value if isinstance(c.h, C.c_void_p) else c.h for c in ctxs])
        outs = (C.c_void_p * n)()
        check(lib.gx_comm_init_local(arr, n, outs))
        return [Comm(C.c_void_p(outs[r]), ctxs[r]) for r in range(n)]

    @staticmethod
    def host(ctx: Context, nranks: int, rank: int, group=None) -> "Comm":
        """Host-staged transport (gx_comm_init_host): the same grouping,
        owner-gather and scatter kernels, with the bytes exchanged by
        torch.distributed all_to_all_single over the process group (gloo) --
        for ranks NCCL cannot connect, e.g. several processes on one GPU."""
        import torch
        import torch.distributed as dist

        def xchg(user, send, scnt, recv, rcnt):
            try:
                sc = [int(scnt[p]) for p in range(nranks)]
                rc = [int(rcnt[p]) for p in range(nranks)]
                t_in = torch.empty(sum(sc), dtype=torch.uint8)
                if sum(sc):
                    C.memmove(t_in.data_ptr(), send, sum(sc))
                t_out = torch.empty(sum(rc), dtype=torch.uint8)
                dist.all_to_all_single(t_out, t_in, output_split_sizes=rc, input_split_sizes=sc, group=group)
                if sum(rc):
                    C.memmove(recv, t_out.data_ptr(), sum(rc))
                return 0
            except Exception:   # reported as GX_RUNTIME_ERROR by the library
                return 1

        cb = _HOST_XCHG(xchg)
        h = C.c_void_p()
        check(lib.gx_comm_init_host(ctx.h, nranks, rank, cb, None, C.byref(h)))
        c = Comm(h, ctx)
        c._cb = cb      # the callback must outlive the communicator
        return c

    @property
    def rank(self) -> int:
        return lib.gx_comm_rank(self.h)

    @property
    def size(self) -> int:
        return lib.gx_comm_size(self.h)


@dataclasses.dataclass
class ExchangeStats:
    """gx_exchange_stats: all-to-all traffic of a partitioned table."""
    calls: int
    rows_requested: int
    rows_remote: int
    rows_served: int
    bytes_sent: int
    ms: float


@dataclasses.dataclass
class StorageStats:
    """gx_storage_stats: physical reads of a file-backed table since open."""
    rows: int
    preads: int
    bytes: int
    h2d_bytes: int
    read_ms: float
    threads: int
    direct: bool


class FeatureFile:
    """FeatureFile (graph_store.hpp:280-333): the table lives in HBM ("device"),
    in pinned host memory ("host", misses read over PCIe by the kernel) or stays
    in features.bin ("file": the SSD tier -- missed rows are read with pread,
    O_DIRECT where the filesystem allows it, into pinned staging and copied to
    HBM on a side stream). A file-backed table opened with ctx=None serves
    read_rows from the host alone."""

    def __init__(self, handle, ctx: Optional[Context], dtype=np.float32):
        self.h = handle
        self.ctx = ctx
        self.dtype = dtype

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_features_destroy(self.h)
            self.h = None

    @staticmethod
    def open(path: str, backing: str = "device", ctx: Optional[Context] = None) -> "FeatureFile":
        c = ctx if (ctx is not None or backing == "file") else _ctx(ctx)
        h = C.c_void_p()
        check(lib.gx_features_open(c.h if c is not None else None, os.fspath(path).encode(),
                                   BACKING[backing], C.byref(h)))
        f = FeatureFile(h, c)
        if f.row_bytes() == 2 * f.dim():
            f.dtype = np.float16
        return f

    @staticmethod
    def from_array(rows: np.ndarray, backing: str = "device",
                   ctx: Optional[Context] = None) -> "FeatureFile":
        c = _ctx(ctx)
        rows = np.ascontiguousarray(rows)
        if rows.dtype not in (np.float32, np.float16):
            raise ValueError("feature rows must be float32 or float16")
        n, dim = rows.shape
        h = C.c_void_p()
        check(lib.gx_features_from_host(c.h, n, dim, rows.dtype.itemsize, _ptr(rows.reshape(-1)),
                                        BACKING[backing], C.byref(h)))
        return FeatureFile(h, c, rows.dtype.type)

    @staticmethod
    def generate(num_nodes: int, dim: int, value_seed: int, ctx: Optional[Context] = None,
                 dtype=np.float32) -> "FeatureFile":
        """feature_value table (graphgen.hpp:74-77) generated in HBM; dtype
        float16 = the scalar_width 2 extension (fp16 of the same values)."""
        c = _ctx(ctx)
        h = C.c_void_p()
        if np.dtype(dtype) == np.float16:
            check(lib.gx_features_generate_fp16(c.h, num_nodes, dim, value_seed, C.byref(h)))
            return FeatureFile(h, c, np.float16)
        check(lib.gx_features_generate(c.h, num_nodes, dim, value_seed, C.byref(h)))
        return FeatureFile(h, c)

    # -- row-partitioned tables (include/gx_b200.h) ----------
    @staticmethod
    def partitioned_from_array(local_rows: np.ndarray, num_nodes: int, comm: "Comm",
                               ctx: Optional[Context] = None) -> "FeatureFile":
        """This rank's rows [lo, hi) of an N-row table partitioned over comm."""
        c = ctx if ctx is not None else comm.ctx
        rows = np.ascontiguousarray(local_rows)
        lo, hi = partition_bounds(num_nodes, comm.size, comm.rank)
        if rows.shape[0] != hi - lo:
            raise ValueError(f"rank {comm.rank} owns rows [{lo}, {hi}), got {rows.shape[0]}")
        h = C.c_void_p()
        check(lib.gx_features_partitioned_from_host(c.h, comm.h, num_nodes, rows.shape[1], rows.dtype.itemsize,
                                                    _ptr(rows.reshape(-1)) if rows.size else None,
                                                    C.byref(h)))
        f = FeatureFile(h, c, rows.dtype.type)
        f.comm = comm
        return f

    @staticmethod
    def partitioned_open(path: str, comm: "Comm", ctx: Optional[Context] = None) -> "FeatureFile":
        """This rank's rows of features.bin (only those bytes are read)."""
        c = ctx if ctx is not None else comm.ctx
        h = C.c_void_p()
        check(lib.gx_features_partitioned_open(c.h, comm.h, os.fspath(path).encode(), C.byref(h)))
        f = FeatureFile(h, c)
        if f.row_bytes() == 2 * f.dim():
            f.dtype = np.float16
        f.comm = comm
        return f

    @staticmethod
    def partitioned_generate(num_nodes: int, dim: int, value_seed: int, comm: "Comm",
                             ctx: Optional[Context] = None, dtype=np.float32) -> "FeatureFile":
        c = ctx if ctx is not None else comm.ctx
        sw = np.dtype(dtype).itemsize
        h = C.c_void_p()
        check(lib.gx_features_partitioned_generate(c.h, comm.h, num_nodes, dim, sw, value_seed, C.byref(h)))
        f = FeatureFile(h, c, np.dtype(dtype).type)
        f.comm = comm
        return f

    def exchange_stats(self) -> "ExchangeStats":
        st = ExchangeStatsC()
        check(lib.gx_features_exchange_stats(self.h, C.byref(st)))
        return ExchangeStats(st.calls, st.rows_requested, st.rows_remote, st.rows_served, st.bytes_sent, st.ms)

    def num_nodes(self) -> int:
        return lib.gx_features_num_nodes(self.h)

    def dim(self) -> int:
        return lib.gx_features_dim(self.h)

    def row_bytes(self) -> int:
        return lib.gx_features_row_bytes(self.h)

    def write(self, path: str) -> None:
        """FeatureWriter (graph_store.hpp:237-250): features.bin of this table."""
        check(lib.gx_features_write(self.h, os.fspath(path).encode()))

    def storage_stats(self) -> StorageStats:
        st = StorageStatsC()
        check(lib.gx_features_storage_stats(self.h, C.byref(st)))
        return StorageStats(st.rows, st.preads, st.bytes, st.h2d_bytes, st.read_ms, st.threads,
                            bool(st.direct))

    def read_rows(self, ids, stats: Optional[IoStats] = None) -> np.ndarray:
        """FeatureFile::read_rows (graph_store.hpp:319-324)."""
        ids = _u64(ids)
        out = np.zeros((len(ids), self.dim()), self.dtype)
        io = IoStatsC()
        check(lib.gx_features_read_rows(self.h, _ptr(ids), len(ids), _ptr(out), C.byref(io)))
        if stats is not None:
            stats._add_c(io)
        return out


open_features = FeatureFile.open


class Batch:
    """Gathered batch buffer (RowMatrix, graph_store.hpp:222-234), device resident."""

    def __init__(self, ctx: Context, dim: int, dtype):
        h = C.c_void_p()
        check(lib.gx_batch_create(ctx.h, C.byref(h)))
        self.h = h
        self.dim = dim
        self.dtype = dtype

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_batch_destroy(self.h)
            self.h = None

    @property
    def rows(self) -> int:
        return lib.gx_batch_rows(self.h)

    def numpy(self) -> np.ndarray:
        out = np.zeros((self.rows, self.dim), self.dtype)
        check(lib.gx_batch_copy_to_host(self.h, _ptr(out)))
        return out

    @property
    def device_ptr(self) -> int:
        return lib.gx_batch_device_ptr(self.h)


@dataclasses.dataclass
class GatherCounts:
    """feature_cache.hpp:50-53"""
    hits: int = 0
    misses: int = 0


class FeatureCache:
    """FeatureCache (feature_cache.hpp:15-138) with rows and the address table in HBM."""

    def __init__(self, store: FeatureFile, init_ids, num_entries: int, stats: Optional[IoStats] = None):
        ids = _u64(init_ids)
        io = IoStatsC()
        h = C.c_void_p()
        check(lib.gx_cache_create(store.h, _ptr(ids), len(ids), num_entries, C.byref(io), C.byref(h)))
        self.h = h
        self.store = store
        if stats is not None:
            stats._add_c(io)

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_cache_destroy(self.h)
            self.h = None

    def num_entries(self) -> int:
        return lib.gx_cache_num_entries(self.h)

    def dim(self) -> int:
        return self.store.dim()

    def contains(self, v: int) -> bool:
        out = C.c_int()
        check(lib.gx_cache_contains(self.h, v, C.byref(out)))
        return bool(out.value)

    def cached_row(self, v: int) -> np.ndarray:
        out = np.zeros(self.store.dim(), self.store.dtype)
        check(lib.gx_cache_cached_row(self.h, v, out.ctypes.data))
        return out

    def gather(self, store: FeatureFile, ids, stats: Optional[IoStats] = None,
               out: Optional[Batch] = None) -> tuple:
        """FeatureCache::gather (feature_cache.hpp:58-76) -> (Batch, GatherCounts)."""
        if store is not self.store and store.h != self.store.h:
            raise ValueError("gather must use the cache's own feature store")
        ids = _u64(ids)
        b = out if out is not None else Batch(store.ctx, store.dim(), store.dtype)
        hits, misses = C.c_uint64(), C.c_uint64()
        io = IoStatsC()
        check(lib.gx_cache_gather(self.h, _ptr(ids), len(ids), b.h, C.byref(hits), C.byref(misses),
                                  C.byref(io)))
        if stats is not None:
            stats._add_c(io)
        return b, GatherCounts(hits.value, misses.value)

    def apply_changeset(self, batch: Batch, ids, cs: Changeset) -> None:
        """FeatureCache::apply_changeset (feature_cache.hpp:89-130)."""
        a, p, o = _u64(cs.in_ids), _u64(cs.in_positions), _u64(cs.out_ids)
        if len(a) != len(p):
            raise ValueError("changeset arrays disagree in length")
        ids = _u64(ids)
        check(lib.gx_cache_apply(self.h, batch.h, _ptr(ids), len(ids), _ptr(a), _ptr(p), len(a),
                                 _ptr(o), len(o)))

    def resident_set(self) -> np.ndarray:
        out = np.zeros(max(self.num_entries(), 1), np.uint64)
        n = C.c_uint64()
        check(lib.gx_cache_resident_set(self.h, out.ctypes.data, len(out), C.byref(n)))
        return out[:n.value].copy()


# ---------------------------------------------------------------------------
# fused device pipeline (pipeline.hpp:338-377 stages 1-4)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class PipelineStats:
    sampled_edges: int
    gathered_rows: int
    total_misses: int
    predicted_misses: int
    init_size: int
    total_in: int
    total_out: int
    sample_io: IoStats
    gather_io: IoStats
    ms_sample: float
    ms_inspect: float
    ms_switch: float
    ms_gather: float
    ms_gather_kernels: float
    ms_apply_kernels: float
    kernel_launches: int
    gather_launches: int
    misses: np.ndarray
    ms_storage: float = 0.0      # file-backed tables: host read phase of the superbatch
    storage_rows: int = 0
    storage_bytes: int = 0
    fill_rows: int = 0           # rows the switch wrote (init set)
    gather_kernel_rows: int = 0  # rows the gather launches moved
    fused_fill: bool = False     # all-fit: the switch also wrote each init node's first batch row
    fan_out: bool = False        # all-fit, fan-out form: each init row written to all its batch rows
    init_fan: bool = False       # changesets: each init row written to its slot + every access it serves


def _io(c: IoStatsC) -> IoStats:
    return IoStats(c.pages_read, c.rows_read, c.neighbor_lists_read, c.bytes_read)


class Pipeline:
    """sample -> precompute -> cache init -> S x (gather, apply) on one GPU."""

    def __init__(self, graph: GraphFile, features: FeatureFile, fanouts: Sequence[int],
                 num_entries: int, digest: bool = False, overlap: bool = False):
        """overlap: with two superbatches in flight (submit/wait), let superbatch
        k+1's sampler and inspector run concurrently with k's executor instead
        of after it (gx_pipeline_set_overlap)."""
        f = _fan(fanouts)
        h = C.c_void_p()
        check(lib.gx_pipeline_create(graph.h, features.h, _ptr(f), len(f), num_entries, C.byref(h)))
        self.h = h
        self.graph, self.features = graph, features
        self._K = num_entries
        if digest:
            check(lib.gx_pipeline_set_digest(h, 1))
        if overlap:
            check(lib.gx_pipeline_set_overlap(h, 1))
        self._S = 0
        self._last = -1
        self._sizes = {}

    def __del__(self):
        if getattr(self, "h", None):
            lib.gx_pipeline_destroy(self.h)
            self.h = None

    def run_superbatch(self, batches, global_seed: int, first_global_batch: int) -> PipelineStats:
        """Synchronous: one superbatch end to end (gx_pipeline_superbatch)."""
        return self.wait(self.submit(batches, global_seed, first_global_batch))

    def submit(self, batches, global_seed: int, first_global_batch: int) -> int:
        """Sampler + inspector now, executor queued on the pipeline stream;
        returns a ticket. At most two superbatches may be in flight."""
        flat, off = _flatten(batches)
        t = C.c_uint64()
        check(lib.gx_pipeline_submit(self.h, flat.ctypes.data, off.ctypes.data, len(off) - 1,
                                     global_seed & 0xFFFFFFFFFFFFFFFF, first_global_batch, C.byref(t)))
        self._sizes[t.value] = len(off) - 1
        return t.value

    def wait(self, ticket: int) -> PipelineStats:
        S = self._sizes.pop(ticket)
        misses = np.zeros(max(S, 1), np.uint64)
        st = PipelineStatsC()
        check(lib.gx_pipeline_wait(self.h, ticket, misses.ctypes.data, C.byref(st)))
        self._S = S
        self._last = ticket
        return PipelineStats(st.sampled_edges, st.gathered_rows, st.total_misses, st.predicted_misses,
                             st.init_size, st.total_in, st.total_out, _io(st.sample_io),
                             _io(st.gather_io), st.ms_sample, st.ms_inspect, st.ms_switch,
                             st.ms_gather, st.ms_gather_kernels, st.ms_apply_kernels, st.kernel_launches,
                             st.gather_launches, misses[:S].copy(), st.ms_storage, st.storage_rows,
                             st.storage_bytes, st.fill_rows, st.gather_kernel_rows, st.fused_fill in (1, 2),
                             st.fused_fill == 2, st.fused_fill == 3)

    def batch(self, i: int, ticket: Optional[int] = None) -> np.ndarray:
        """Iteration i's gathered rows of a waited-for superbatch (default: the
        last one waited for) -- a host copy of the device-resident batch
        (gx_pipeline_batch)."""
        ticket = self._last if ticket is None else ticket
        n = C.c_uint64()
        check(lib.gx_pipeline_batch(self.h, ticket, i, None, C.byref(n), None))
        f = self.features
        out = np.empty((n.value, f.dim()), dtype=f.dtype)
        if n.value:
            check(lib.gx_pipeline_batch(self.h, ticket, i, None, None, out.ctypes.data))
        return out

    @property
    def exec_stream(self) -> int:
        return lib.gx_pipeline_exec_stream(self.h)

    def copy_superbatch(self, host_ptr: int, cap_bytes: int, ticket: Optional[int] = None) -> int:
        """All iterations' rows of a waited-for superbatch into host memory at
        host_ptr (pinned for PCIe rate) in one D2H -> bytes copied
        (gx_pipeline_copy_superbatch)."""
        ticket = self._last if ticket is None else ticket
        n = C.c_uint64()
        check(lib.gx_pipeline_copy_superbatch(self.h, ticket, host_ptr, cap_bytes, C.byref(n)))
        return n.value

    def cache_rows(self) -> np.ndarray:
        """Test hook: the feature cache's K slot rows after the last waited-for
        superbatch (gx_pipeline_cache_rows); never-filled slots are unspecified."""
        f = self.features
        K = self._K
        out = np.empty((K, f.dim()), dtype=f.dtype)
        if K:
            check(lib.gx_pipeline_cache_rows(self.h, out.ctypes.data))
        return out

    def digests(self) -> np.ndarray:
        out = np.zeros(max(self._S, 1), np.uint64)
        check(lib.gx_pipeline_digests(self.h, out.ctypes.data))
        return out[:self._S].copy()


def batch_digest(rows: np.ndarray) -> int:
    """Host mirror of the pipeline digest: sum_x (w[x] + 1) * mix64(x) mod 2^64
    over the u32 words of the batch (include/gx_b200.h)."""
    w = np.ascontiguousarray(rows).view(np.uint32).reshape(-1).astype(np.uint64)
    x = np.arange(len(w), dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return int(np.sum((w + np.uint64(1)) * z, dtype=np.uint64))
