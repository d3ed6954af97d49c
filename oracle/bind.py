"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

Both libraries take plain arrays; these wrappers take/return numpy arrays and
raise the Python counterpart of the reference's C++ exception type:
invalid_argument -> ValueError, out_of_range -> IndexError,
logic_error -> OracleLogicError, runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C_
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
oracle_lib_path = os.path.join(HERE, "_build", "libgx_oracle.so")
ref_lib_path = os.path.join(HERE, "_ref", "libgx_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
vp = C_.c_void_p
u64 = C_.c_uint64
u32 = C_.c_uint32


class OracleError(Exception):
    pass


class OracleLogicError(OracleError):
    pass


def _raise(rc, msg=""):
    if rc == 0:
        return
    if rc == 1:
        raise ValueError(msg or "invalid_argument")
    if rc == 2:
        raise IndexError(msg or "out_of_range")
    if rc == 3:
        raise OracleLogicError(msg or "logic_error")
    if rc == 5:
        raise OverflowError(msg or "overflow_error")
    raise RuntimeError(msg or "runtime_error")


def build(ref=True):
    """Compile the checkers (oracle/Makefile). ref=True also builds oracle/_ref
    from /root/reference when that tree exists."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/include/gx"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _a64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(-1))


def _trace(trace):
    lists = [_a64(t) for t in trace]
    off = np.zeros(len(lists) + 1, np.uint64)
    if lists:
        off[1:] = np.cumsum([len(t) for t in lists])
    flat = np.concatenate(lists) if lists and off[-1] > 0 else np.zeros(1, np.uint64)
    return flat, off


class _Oracle:
    """The C restatement (oracle/gx_oracle.c)."""

    def __init__(self, path):
        self.path = path
        self._lib = None

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(self.path):
                build(ref=False)
            L = C_.CDLL(self.path)
            L.gxo_mix64.restype = u64
            L.gxo_mix64.argtypes = [u64]
            L.gxo_derive_seed.restype = u64
            L.gxo_derive_seed.argtypes = [u64, u64]
            L.gxo_pages_touched.restype = u64
            L.gxo_pages_touched.argtypes = [u64, u64]
            L.gxo_page_count_for_row.restype = u64
            L.gxo_page_count_for_row.argtypes = [u64, u64]
            L.gxo_generate_edges.argtypes = [u64, C_.c_double, C_.c_double, C_.c_double,
                                             C_.c_double, u64, u64p, u64p, u64, C_.POINTER(u64)]
            L.gxo_build_csc.argtypes = [u64, u64p, u64p, u64, u64p, u64p, C_.POINTER(u64)]
            L.gxo_feature_value.restype = C_.c_float
            L.gxo_feature_value.argtypes = [u64, u64, u32]
            L.gxo_plan_seed_batches.argtypes = [u64p, u64, u64, u64, u64p]
            L.gxo_train_ids.restype = u64
            L.gxo_train_ids.argtypes = [u64, u64, C_.c_double, u64p]
            L.gxo_epoch_seed.restype = u64
            L.gxo_epoch_seed.argtypes = [u64, u64]
            L.gxo_sample_batch.argtypes = [u64p, u64p, u64, u64p, u64, u32p, u32, u64, u64p, u64,
                                           C_.POINTER(u64), u32p, u64, u64p, u64p]
            L.gxo_access_index.argtypes = [u64p, u64p, u64, u64, u64p, u64p]
            L.gxo_compute_init_set.argtypes = [u64p, u64p, u64, u64, u64, u64p, C_.POINTER(u64)]
            L.gxo_simulate.argtypes = [u64p, u64p, u64, u64, u64, u64p, u64, u64p, u64p, u64p,
                                       u64p, u64p, u64p, vp, vp, u64]
            L.gxo_cache_create.argtypes = [vp, u64, u32, u64p, u64, u64, u64p, C_.POINTER(vp)]
            L.gxo_cache_destroy.argtypes = [vp]
            L.gxo_cache_slot.restype = C_.c_int64
            L.gxo_cache_slot.argtypes = [vp, u64]
            L.gxo_cache_gather.argtypes = [vp, u64p, u64, vp, C_.POINTER(u64), C_.POINTER(u64),
                                           u64p]
            L.gxo_cache_apply.argtypes = [vp, vp, u64, u64p, u64, u64p, u64p, u64, u64p, u64]
            L.gxo_cache_resident.restype = u64
            L.gxo_cache_resident.argtypes = [vp, u64p]
            L.gxo_compute_stub.restype = u64
            L.gxo_compute_stub.argtypes = [vp, u64, u64, vp, vp, u32]
            self._lib = L
        return self._lib

    # -- primitives
    def mix64(self, z):
        return self.lib.gxo_mix64(z)

    def derive_seed(self, b, i):
        return self.lib.gxo_derive_seed(b, i)

    def epoch_seed(self, seed, epoch):
        return self.lib.gxo_epoch_seed(seed, epoch)

    def pages_touched(self, lo, hi):
        return self.lib.gxo_pages_touched(lo, hi)

    def page_count_for_row(self, w, r):
        return self.lib.gxo_page_count_for_row(w, r)

    def feature_value(self, seed, node, col):
        return self.lib.gxo_feature_value(seed, node, col)

    # -- datasets
    def generate_edges(self, n, avg_deg, seed, a=0.57, b=0.19, c=0.19):
        target = int(avg_deg * float(n))
        src = np.zeros(max(target, 1), np.uint64)
        dst = np.zeros(max(target, 1), np.uint64)
        cnt = u64()
        _raise(self.lib.gxo_generate_edges(n, avg_deg, a, b, c, seed, src, dst, len(src),
                                           C_.byref(cnt)))
        return src[:cnt.value], dst[:cnt.value]

    def build_csc(self, n, src, dst):
        src, dst = _a64(src), _a64(dst)
        m = len(src)
        indptr = np.zeros(n + 1, np.uint64)
        ind = np.zeros(max(m, 1), np.uint64)
        e = u64()
        _raise(self.lib.gxo_build_csc(n, src if m else np.zeros(1, np.uint64),
                                      dst if m else np.zeros(1, np.uint64), m, indptr, ind,
                                      C_.byref(e)))
        return indptr, ind[:e.value].copy()

    def rmat_graph(self, n, avg_deg, seed):
        s, d = self.generate_edges(n, avg_deg, seed)
        return self.build_csc(n, s, d)

    def features(self, n, dim, value_seed):
        """features.bin payload rows (graphgen.hpp:74-77, 94-100), vectorised."""
        node = np.arange(n, dtype=np.uint64)[:, None]
        col = np.arange(dim, dtype=np.uint64)[None, :]
        with np.errstate(over="ignore"):
            h = _np_mix64(np.uint64(value_seed) ^ _np_mix64(node * np.uint64(0x10001) + col))
        return ((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)

    def train_ids(self, n, seed, frac):
        out = np.zeros(max(n, 1), np.uint64)
        k = self.lib.gxo_train_ids(n, seed, frac, out)
        return out[:k].copy()

    def plan_seed_batches(self, train, batch_size, epoch_seed):
        train = _a64(train)
        out = np.zeros(max(len(train), 1), np.uint64)
        _raise(self.lib.gxo_plan_seed_batches(train if len(train) else out, len(train), batch_size,
                                              epoch_seed, out))
        return [out[o:o + batch_size].copy() for o in range(0, len(train), batch_size)]

    # -- sampler
    def sample_batch(self, indptr, indices, seeds, fanouts, batch_seed):
        """-> (ids u64[], layers [u32 (E_l,2)], io[4])"""
        indptr, indices, seeds = _a64(indptr), _a64(indices), _a64(seeds)
        n = len(indptr) - 1
        fan = np.ascontiguousarray(fanouts, dtype=np.uint32)
        ids_cap = len(seeds)
        e_cap = 0
        f = len(seeds)
        for fl in fan:
            e_cap += f * int(fl)
            f += f * int(fl)
        ids_cap = min(f, max(n, len(seeds)))
        ids = np.zeros(max(ids_cap, 1), np.uint64)
        edges = np.zeros(max(2 * e_cap, 2), np.uint32)
        lc = np.zeros(max(len(fan), 1), np.uint64)
        io = np.zeros(4, np.uint64)
        nid = u64()
        _raise(self.lib.gxo_sample_batch(indptr, indices if len(indices) else np.zeros(1, np.uint64),
                                         n, seeds if len(seeds) else np.zeros(1, np.uint64),
                                         len(seeds), fan if len(fan) else np.zeros(1, np.uint32),
                                         len(fan), batch_seed, ids, len(ids), C_.byref(nid), edges,
                                         e_cap, lc, io))
        layers, k = [], 0
        for l in range(len(fan)):
            c = int(lc[l])
            layers.append(edges[2 * k:2 * (k + c)].reshape(-1, 2).copy())
            k += c
        return ids[:nid.value].copy(), layers, io

    # -- inspector
    def access_index(self, trace, N):
        flat, off = _trace(trace)
        A = int(off[-1])
        iters = np.zeros(A + 1, np.uint64)
        ptr = np.zeros(max(N, 1), np.uint64)
        _raise(self.lib.gxo_access_index(flat, off, len(off) - 1, N, iters, ptr))
        return iters, ptr[:N].copy()

    def compute_init_set(self, trace, K, N):
        flat, off = _trace(trace)
        out = np.zeros(max(min(K, int(off[-1])), 1), np.uint64)
        n = u64()
        _raise(self.lib.gxo_compute_init_set(flat, off, len(off) - 1, K, N, out, C_.byref(n)))
        return out[:n.value].copy()

    def simulate(self, trace, N, K, init, states=False):
        """-> dict(misses, in_ids, in_pos, in_off, out_ids, out_off[, state, state_off])"""
        flat, off = _trace(trace)
        S = len(off) - 1
        A = int(off[-1])
        init = _a64(init)
        misses = np.zeros(max(S, 1), np.uint64)
        in_ids = np.zeros(A + 1, np.uint64)
        in_pos = np.zeros(A + 1, np.uint64)
        in_off = np.zeros(S + 1, np.uint64)
        out_ids = np.zeros(A + len(init) + 1, np.uint64)
        out_off = np.zeros(S + 1, np.uint64)
        st = st_off = None
        cap = 0
        if states:
            cap = S * max(K, 1) if S else 1
            cap = min(cap, S * (A + len(init)) + 1)
            st = np.zeros(max(cap, 1), np.uint64)
            st_off = np.zeros(S + 1, np.uint64)
        _raise(self.lib.gxo_simulate(flat, off, S, N, K, init if len(init) else np.zeros(1, np.uint64),
                                     len(init), misses, in_ids, in_pos, in_off, out_ids, out_off,
                                     st.ctypes.data if states else None,
                                     st_off.ctypes.data if states else None, cap))
        r = dict(misses=misses[:S].copy(), in_ids=in_ids[:int(in_off[-1])].copy(),
                 in_pos=in_pos[:int(in_off[-1])].copy(), in_off=in_off,
                 out_ids=out_ids[:int(out_off[-1])].copy(), out_off=out_off)
        if states:
            r["state"] = st[:int(st_off[-1])].copy()
            r["state_off"] = st_off
        return r

    def compute_stub(self, rows, layers):
        """compute_stub (pipeline.hpp:35-57) of a batch (n, dim) and its layers [(E_l, 2) u32]"""
        rows = np.ascontiguousarray(rows)
        pairs = np.ascontiguousarray(np.concatenate([np.asarray(l, np.uint32).reshape(-1) for l in layers])
                                     if layers else np.zeros(0, np.uint32))
        cnt = np.array([len(l) for l in layers] or [0], np.uint64)
        return self.lib.gxo_compute_stub(rows.ctypes.data, rows.shape[0], rows.shape[1] * rows.itemsize,
                                         pairs.ctypes.data if pairs.size else None, cnt.ctypes.data, len(layers))

    # -- executor
    def cache(self, store_rows, init, K):
        return _OCache(self, store_rows, init, K)


class _OCache:
    """FeatureCache restatement over an in-memory (n, dim) row table."""

    def __init__(self, o, store, init, K):
        self.o = o
        self.store = np.ascontiguousarray(store)
        self.n, self.dim = self.store.shape
        self.w = self.store.dtype.itemsize * self.dim
        init = _a64(init)
        self.io = np.zeros(4, np.uint64)
        h = vp()
        _raise(o.lib.gxo_cache_create(self.store.ctypes.data, self.n, self.w,
                                      init if len(init) else np.zeros(1, np.uint64), len(init), K,
                                      self.io, C_.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.gxo_cache_destroy(self.h)
            self.h = None

    def gather(self, ids):
        ids = _a64(ids)
        out = np.zeros((len(ids), self.dim), self.store.dtype)
        h, m = u64(), u64()
        io = np.zeros(4, np.uint64)
        _raise(self.o.lib.gxo_cache_gather(self.h, ids if len(ids) else np.zeros(1, np.uint64),
                                           len(ids), out.ctypes.data, C_.byref(h), C_.byref(m), io))
        return out, h.value, m.value, io

    def apply(self, batch, ids, in_ids, in_pos, out_ids):
        ids, in_ids, in_pos, out_ids = _a64(ids), _a64(in_ids), _a64(in_pos), _a64(out_ids)
        batch = np.ascontiguousarray(batch)
        z = np.zeros(1, np.uint64)
        _raise(self.o.lib.gxo_cache_apply(self.h, batch.ctypes.data, batch.shape[0],
                                          ids if len(ids) else z, len(ids),
                                          in_ids if len(in_ids) else z,
                                          in_pos if len(in_pos) else z, len(in_ids),
                                          out_ids if len(out_ids) else z, len(out_ids)))

    def slot(self, v):
        return self.o.lib.gxo_cache_slot(self.h, v)

    def resident(self):
        out = np.zeros(max(self.n, 1), np.uint64)
        k = self.o.lib.gxo_cache_resident(self.h, out)
        return out[:k].copy()


def _np_mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


class _Ref:
    """The unmodified reference, via oracle/_ref/libgx_ref.so."""

    def __init__(self, path):
        self.path = path
        self._lib = None

    def available(self):
        return os.path.exists(self.path)

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(self.path):
                raise RuntimeError("oracle/_ref/libgx_ref.so not built (needs /root/reference)")
            L = C_.CDLL(self.path)
            L.gxr_last_error.restype = C_.c_char_p
            L.gxr_mix64.restype = u64
            L.gxr_mix64.argtypes = [u64]
            L.gxr_derive_seed.restype = u64
            L.gxr_derive_seed.argtypes = [u64, u64]
            L.gxr_generate_dataset.argtypes = [C_.c_char_p, u64, C_.c_double, u32, u64, u64,
                                               C_.POINTER(u64)]
            L.gxr_generate_edges.argtypes = [u64, C_.c_double, u64, u64p, u64p, u64,
                                             C_.POINTER(u64)]
            L.gxr_write_graph.argtypes = [C_.c_char_p, u64, u64p, u64p, u64]
            L.gxr_write_graph_csc.argtypes = [C_.c_char_p, u64, u64p, u64p, u64]
            L.gxr_feature_value.restype = C_.c_float
            L.gxr_feature_value.argtypes = [u64, u64, u32]
            L.gxr_write_features.argtypes = [C_.c_char_p, u64, u32, f32p]
            L.gxr_graph_open.argtypes = [C_.c_char_p, C_.POINTER(vp)]
            L.gxr_graph_close.argtypes = [vp]
            L.gxr_graph_num_nodes.restype = u64
            L.gxr_graph_num_nodes.argtypes = [vp]
            L.gxr_graph_num_edges.restype = u64
            L.gxr_graph_num_edges.argtypes = [vp]
            L.gxr_graph_read_all.argtypes = [vp, u64p, u64p]
            L.gxr_sample_batch.argtypes = [vp, u64p, u64, u32p, u32, u64, u64p, u64,
                                           C_.POINTER(u64), u32p, u64, u64p, u64p]
            L.gxr_sample_batch_nc.argtypes = [vp, C_.c_char_p] + L.gxr_sample_batch.argtypes[1:]
            L.gxr_ncache_build.argtypes = [vp, u64, C_.c_char_p, u64p, C_.POINTER(u64)]
            L.gxr_simulate_policy.argtypes = [vp, u64p, u64p, u64, u64, C_.c_int, u64p, C_.POINTER(u64)]
            L.gxr_superbatch_sample.argtypes = [vp, u64p, u64p, u64, u32p, u32, u64, u64, u64,
                                                C_.c_char_p, C_.c_uint, u64p,
                                                C_.POINTER(C_.c_double)]
            L.gxr_plan_seed_batches.argtypes = [u64p, u64, u64, u64, u64p]
            L.gxr_train_ids.argtypes = [C_.c_char_p, C_.c_char_p, u64, C_.c_double, u64p, u64,
                                        C_.POINTER(u64)]
            L.gxr_access_index.argtypes = [u64p, u64p, u64, u64, u64p, u64p]
            L.gxr_compute_init_set.argtypes = [u64p, u64p, u64, u64, u64, u64p, C_.POINTER(u64)]
            L.gxr_simulate.argtypes = [u64p, u64p, u64, u64, u64, u64p, u64, C_.c_int, u64p,
                                       u64p, u64p, u64p, u64p, u64p, vp, vp, u64,
                                       C_.POINTER(C_.c_double)]
            L.gxr_dp_optimal_misses.argtypes = [u64p, u64p, u64, u64, C_.POINTER(u64)]
            L.gxr_precompute_changesets.argtypes = [C_.c_char_p, u64, u64, u64, u64, vp, vp,
                                                    C_.POINTER(C_.c_double)]
            L.gxr_run_training.argtypes = [C_.c_char_p, C_.c_char_p, C_.c_char_p, C_.c_char_p, vp, u32, u64, u64,
                                           u64, u64, C_.c_int, C_.c_int, C_.c_uint, u64, C_.c_double, vp, u64,
                                           C_.POINTER(u64)]
            L.gxr_compute_stub.restype = u64
            L.gxr_compute_stub.argtypes = [vp, u64, u32, vp, vp, u32]
            L.gxr_features_open.argtypes = [C_.c_char_p, C_.POINTER(vp)]
            L.gxr_features_close.argtypes = [vp]
            L.gxr_cache_create.argtypes = [vp, u64p, u64, u64, u64p, C_.POINTER(vp)]
            L.gxr_cache_destroy.argtypes = [vp]
            L.gxr_cache_gather.argtypes = [vp, vp, u64p, u64, vp, C_.POINTER(u64),
                                           C_.POINTER(u64), u64p]
            L.gxr_cache_apply.argtypes = [vp, vp, u64, u32, u64p, u64, u64p, u64p, u64, u64p, u64]
            L.gxr_cache_resident.argtypes = [vp, u64p, u64, C_.POINTER(u64)]
            L.gxr_cache_row.argtypes = [vp, u64, vp]
            L.gxr_run_superbatch.argtypes = [C_.c_char_p, C_.c_char_p, C_.c_char_p, u64p, u64p, u64,
                                             u32p, u32, u64, u64, u64, C_.c_uint,
                                             np.ctypeslib.ndpointer(np.float64), C_.POINTER(u64),
                                             C_.POINTER(u64), C_.POINTER(u64)]
            self._lib = L
        return self._lib

    def _chk(self, rc):
        if rc:
            _raise(rc, self.lib.gxr_last_error().decode())

    def generate_edges(self, n, avg_deg, seed):
        target = int(avg_deg * float(n))
        s = np.zeros(max(target, 1), np.uint64)
        d = np.zeros(max(target, 1), np.uint64)
        c = u64()
        self._chk(self.lib.gxr_generate_edges(n, avg_deg, seed, s, d, len(s), C_.byref(c)))
        return s[:c.value], d[:c.value]

    def write_graph(self, path, n, src, dst):
        self._chk(self.lib.gxr_write_graph(path.encode(), n, _a64(src), _a64(dst), len(src)))

    def write_graph_csc(self, path, indptr, indices):
        ind = _a64(indices)
        self._chk(self.lib.gxr_write_graph_csc(path.encode(), len(indptr) - 1, _a64(indptr),
                                               ind if len(ind) else np.zeros(1, np.uint64), len(ind)))

    def write_features(self, path, rows):
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        self._chk(self.lib.gxr_write_features(path.encode(), rows.shape[0], rows.shape[1],
                                              rows.reshape(-1)))

    def train_ids(self, graph_path, feature_path, seed, train_fraction):
        """TrainingRunner::train_ids (pipeline.hpp:384-399) on the given files."""
        n = u64()
        self._chk(self.lib.gxr_train_ids(os.fspath(graph_path).encode(), os.fspath(feature_path).encode(),
                                         seed, train_fraction, np.zeros(1, np.uint64), 0, C_.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint64)
        self._chk(self.lib.gxr_train_ids(os.fspath(graph_path).encode(), os.fspath(feature_path).encode(),
                                         seed, train_fraction, out, len(out), C_.byref(n)))
        return out[:n.value].copy()

    def plan_seed_batches(self, train, batch_size, epoch_seed):
        """plan_seed_batches (sampler.hpp:46-62) -> list of batches"""
        train = _a64(train)
        out = np.zeros(max(len(train), 1), np.uint64)
        self._chk(self.lib.gxr_plan_seed_batches(train if len(train) else out, len(train), batch_size,
                                                 epoch_seed, out))
        return [out[o:o + batch_size].copy() for o in range(0, len(train), batch_size)]

    def generate_dataset(self, d, n, avg_deg, dim, edge_seed, value_seed):
        e = u64()
        self._chk(self.lib.gxr_generate_dataset(d.encode(), n, avg_deg, dim, edge_seed, value_seed,
                                                C_.byref(e)))
        return e.value

    def open_graph(self, path):
        return _RefGraph(self, path)

    def access_index(self, trace, N):
        flat, off = _trace(trace)
        iters = np.zeros(int(off[-1]) + 1, np.uint64)
        ptr = np.zeros(max(N, 1), np.uint64)
        self._chk(self.lib.gxr_access_index(flat, off, len(off) - 1, N, iters, ptr))
        return iters, ptr[:N].copy()

    def compute_init_set(self, trace, K, N):
        flat, off = _trace(trace)
        out = np.zeros(max(min(K, int(off[-1])), 1), np.uint64)
        n = u64()
        self._chk(self.lib.gxr_compute_init_set(flat, off, len(off) - 1, K, N, out, C_.byref(n)))
        return out[:n.value].copy()

    def simulate(self, trace, N, K, init, naive=False, states=False):
        flat, off = _trace(trace)
        S = len(off) - 1
        A = int(off[-1])
        init = _a64(init)
        misses = np.zeros(max(S, 1), np.uint64)
        in_ids = np.zeros(A + 1, np.uint64)
        in_pos = np.zeros(A + 1, np.uint64)
        in_off = np.zeros(S + 1, np.uint64)
        out_ids = np.zeros(A + len(init) + 1, np.uint64)
        out_off = np.zeros(S + 1, np.uint64)
        cap = min(S * max(K, 1), S * (A + len(init)) + 1) if states else 0
        st = np.zeros(max(cap, 1), np.uint64)
        st_off = np.zeros(S + 1, np.uint64)
        secs = C_.c_double()
        self._chk(self.lib.gxr_simulate(flat, off, S, N, K, init if len(init) else np.zeros(1, np.uint64),
                                        len(init), 1 if naive else 0, misses, in_ids, in_pos,
                                        in_off, out_ids, out_off,
                                        st.ctypes.data if states else None,
                                        st_off.ctypes.data if states else None, cap,
                                        C_.byref(secs)))
        r = dict(misses=misses[:S].copy(), in_ids=in_ids[:int(in_off[-1])].copy(),
                 in_pos=in_pos[:int(in_off[-1])].copy(), in_off=in_off,
                 out_ids=out_ids[:int(out_off[-1])].copy(), out_off=out_off, seconds=secs.value)
        if states:
            r["state"] = st[:int(st_off[-1])].copy()
            r["state_off"] = st_off
        return r

    def precompute_changesets(self, d, sb, S, N, K):
        """precompute_changesets (changeset.hpp:468-484) over ids_{sb}_{i}.bin
        already in d; writes init_{sb}.bin + update_{sb}_{i}.bin there.
        -> (misses per iteration, init size)"""
        m = np.zeros(max(S, 1), np.uint64)
        n = u64()
        secs = C_.c_double()
        self._chk(self.lib.gxr_precompute_changesets(os.fspath(d).encode(), sb, S, N, K, m.ctypes.data,
                                                     C_.addressof(n),
                                                     C_.byref(secs)))
        return m[:S].copy(), n.value

    def run_training(self, graph_path, feature_path, ncache_path, rt_dir, fanouts, batch_size, superbatch_size,
                     epochs, cache_entries, use_ncache, overlap, workers, seed, train_fraction):
        """run_training (pipeline.hpp:451) -> every iteration's compute_stub checksum"""
        fan = np.ascontiguousarray(fanouts, dtype=np.uint32)
        out = np.zeros(1 << 16, np.uint64)
        n = u64()
        self._chk(self.lib.gxr_run_training(os.fspath(graph_path).encode(), os.fspath(feature_path).encode(),
                                            os.fspath(ncache_path).encode() if ncache_path else None,
                                            os.fspath(rt_dir).encode(), fan.ctypes.data, len(fan), batch_size,
                                            superbatch_size, epochs, cache_entries, int(use_ncache), int(overlap),
                                            workers, seed, train_fraction, out.ctypes.data, len(out), C_.byref(n)))
        return out[:n.value].copy()

    def compute_stub(self, rows, layers):
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        pairs = np.ascontiguousarray(np.concatenate([np.asarray(l, np.uint32).reshape(-1) for l in layers])
                                     if layers else np.zeros(0, np.uint32))
        cnt = np.array([len(l) for l in layers] or [0], np.uint64)
        return self.lib.gxr_compute_stub(rows.ctypes.data, rows.shape[0], rows.shape[1],
                                         pairs.ctypes.data if pairs.size else None, cnt.ctypes.data, len(layers))

    def dp_optimal_misses(self, trace, K):
        flat, off = _trace(trace)
        o = u64()
        self._chk(self.lib.gxr_dp_optimal_misses(flat, off, len(off) - 1, K, C_.byref(o)))
        return o.value

    def open_features(self, path):
        return _RefFeat(self, path)


class _RefGraph:
    def __init__(self, r, path):
        self.r = r
        h = vp()
        r._chk(r.lib.gxr_graph_open(path.encode(), C_.byref(h)))
        self.h = h
        self.num_nodes = r.lib.gxr_graph_num_nodes(h)
        self.num_edges = r.lib.gxr_graph_num_edges(h)

    def close(self):
        if self.h:
            self.r.lib.gxr_graph_close(self.h)
            self.h = None

    __del__ = close

    def read_all(self):
        ip = np.zeros(self.num_nodes + 1, np.uint64)
        ind = np.zeros(max(self.num_edges, 1), np.uint64)
        self.r._chk(self.r.lib.gxr_graph_read_all(self.h, ip, ind))
        return ip, ind[:self.num_edges].copy()

    def simulate_policy(self, trace, K, policy):
        """simulate_policy (baselines.hpp:64-143) -> (misses per iteration, total accesses)."""
        flat, off = _trace(trace)
        pol = {"none": 0, "static_degree": 1, "lru": 2, "belady": 3}[policy]
        m = np.zeros(max(len(trace), 1), np.uint64)
        tot = u64()
        self.r._chk(self.r.lib.gxr_simulate_policy(self.h, flat if len(flat) else np.zeros(1, np.uint64), off,
                                                   len(trace), K, pol, m, C_.byref(tot)))
        return m[:len(trace)].copy(), tot.value

    def ncache_build(self, budget_bytes, path):
        """build_neighbor_cache + persist_neighbor_cache -> (IoStats, cached nodes)."""
        io = np.zeros(4, np.uint64)
        k = u64()
        self.r._chk(self.r.lib.gxr_ncache_build(self.h, budget_bytes, path.encode(), io, C_.byref(k)))
        return io, k.value

    def sample_batch(self, seeds, fanouts, batch_seed, ncache_path=None):
        seeds = _a64(seeds)
        fan = np.ascontiguousarray(fanouts, dtype=np.uint32)
        f = len(seeds)
        e_cap = 0
        for fl in fan:
            e_cap += f * int(fl)
            f += f * int(fl)
        ids = np.zeros(max(min(f, max(self.num_nodes, len(seeds))), 1), np.uint64)
        edges = np.zeros(max(2 * e_cap, 2), np.uint32)
        lc = np.zeros(max(len(fan), 1), np.uint64)
        io = np.zeros(4, np.uint64)
        nid = u64()
        args = (seeds if len(seeds) else np.zeros(1, np.uint64), len(seeds),
                fan if len(fan) else np.zeros(1, np.uint32), len(fan), batch_seed, ids, len(ids),
                C_.byref(nid), edges, e_cap, lc, io)
        if ncache_path is None:
            self.r._chk(self.r.lib.gxr_sample_batch(self.h, *args))
        else:
            self.r._chk(self.r.lib.gxr_sample_batch_nc(self.h, ncache_path.encode(), *args))
        layers, k = [], 0
        for l in range(len(fan)):
            c = int(lc[l])
            layers.append(edges[2 * k:2 * (k + c)].reshape(-1, 2).copy())
            k += c
        return ids[:nid.value].copy(), layers, io

    def superbatch_sample(self, batches, fanouts, global_seed, first_global_batch, sb, out_dir,
                          workers=1):
        flat, off = _trace(batches)
        fan = np.ascontiguousarray(fanouts, dtype=np.uint32)
        io = np.zeros(4, np.uint64)
        secs = C_.c_double()
        self.r._chk(self.r.lib.gxr_superbatch_sample(self.h, flat, off, len(batches), fan, len(fan),
                                                     global_seed, first_global_batch, sb,
                                                     out_dir.encode(), workers, io, C_.byref(secs)))
        return io, secs.value


class _RefFeat:
    def __init__(self, r, path):
        self.r = r
        h = vp()
        r._chk(r.lib.gxr_features_open(path.encode(), C_.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.r.lib.gxr_features_close(self.h)
            self.h = None

    __del__ = close

    def cache(self, init, K):
        return _RefCache(self, init, K)


class _RefCache:
    def __init__(self, f, init, K):
        self.f = f
        r = f.r
        self.r = r
        init = _a64(init)
        self.io = np.zeros(4, np.uint64)
        h = vp()
        r._chk(r.lib.gxr_cache_create(f.h, init if len(init) else np.zeros(1, np.uint64), len(init),
                                      K, self.io, C_.byref(h)))
        self.h = h
        self.dim = r.lib.gxr_features_dim(f.h) if hasattr(r.lib, "gxr_features_dim") else None

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.gxr_cache_destroy(self.h)
            self.h = None

    def gather(self, ids, dim):
        ids = _a64(ids)
        out = np.zeros((len(ids), dim), np.float32)
        h, m = u64(), u64()
        io = np.zeros(4, np.uint64)
        self.r._chk(self.r.lib.gxr_cache_gather(self.h, self.f.h, ids if len(ids) else np.zeros(1, np.uint64),
                                                len(ids), out.ctypes.data, C_.byref(h),
                                                C_.byref(m), io))
        return out, h.value, m.value, io

    def apply(self, batch, ids, in_ids, in_pos, out_ids):
        batch = np.ascontiguousarray(batch, dtype=np.float32)
        ids, in_ids, in_pos, out_ids = _a64(ids), _a64(in_ids), _a64(in_pos), _a64(out_ids)
        z = np.zeros(1, np.uint64)
        self.r._chk(self.r.lib.gxr_cache_apply(self.h, batch.ctypes.data, batch.shape[0],
                                               batch.shape[1], ids if len(ids) else z, len(ids),
                                               in_ids if len(in_ids) else z,
                                               in_pos if len(in_pos) else z, len(in_ids),
                                               out_ids if len(out_ids) else z, len(out_ids)))

    def resident(self, n):
        out = np.zeros(max(n, 1), np.uint64)
        k = u64()
        self.r._chk(self.r.lib.gxr_cache_resident(self.h, out, len(out), C_.byref(k)))
        return out[:k.value].copy()

    def row(self, v, dim):
        out = np.zeros(dim, np.float32)
        self.r._chk(self.r.lib.gxr_cache_row(self.h, int(v), out.ctypes.data))
        return out


gen_lib_path = os.path.join(HERE, "_build", "libgx_gen.so")


class _Gen:
    """oracle/gen_dataset.cpp: threaded writer of generate_dataset's files
    (graph.bin + features.bin, byte-identical to graphgen.hpp:82-108)."""

    def __init__(self, path):
        self.path = path
        self._lib = None

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(self.path):
                build(ref=False)
            L = C_.CDLL(self.path)
            L.gxg_graph_file.argtypes = [C_.c_char_p, u64, C_.c_double, C_.c_double, C_.c_double,
                                         C_.c_double, u64, C_.c_int, C_.POINTER(u64)]
            L.gxg_features_file.argtypes = [C_.c_char_p, u64, u32, u64, C_.c_int]
            self._lib = L
        return self._lib

    def graph_file(self, path, n, avg_deg, edge_seed, threads=None, a=0.57, b=0.19, c=0.19):
        """-> number of edges after dedup"""
        e = u64()
        _raise(self.lib.gxg_graph_file(os.fspath(path).encode(), n, avg_deg, a, b, c, edge_seed,
                                       threads or os.cpu_count() or 1, C_.byref(e)))
        return e.value

    def features_file(self, path, n, dim, value_seed, threads=None):
        _raise(self.lib.gxg_features_file(os.fspath(path).encode(), n, dim, value_seed,
                                          threads or os.cpu_count() or 1))


C = _Oracle(oracle_lib_path)
REF = _Ref(ref_lib_path)
GEN = _Gen(gen_lib_path)


def ref_available():
    return REF.available()
