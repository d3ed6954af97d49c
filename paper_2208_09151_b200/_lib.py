"""ctypes binding of libgx_b200.so (include/gx_b200.h).

The shared library is built in-tree (paper_2208_09151_b200/libgx_b200.so) by
`python -m paper_2208_09151_b200._build` or __graft_entry__.build(). There is no
fallback: if the library is missing, importing the package raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GX_LIB_PATH") or os.path.join(HERE, "libgx_b200.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int
P64 = C.POINTER(C.c_uint64)
P32 = C.POINTER(C.c_uint32)
PVP = C.POINTER(C.c_void_p)
dbl = C.c_double
cstr = C.c_char_p


class IoStatsC(C.Structure):
    _fields_ = [("pages_read", u64), ("rows_read", u64), ("neighbor_lists_read", u64),
                ("bytes_read", u64)]


class PipelineStatsC(C.Structure):
    _fields_ = [("sampled_edges", u64), ("gathered_rows", u64), ("total_misses", u64),
                ("predicted_misses", u64), ("init_size", u64), ("total_in", u64),
                ("total_out", u64), ("sample_io", IoStatsC), ("gather_io", IoStatsC),
                ("ms_sample", dbl), ("ms_inspect", dbl), ("ms_switch", dbl), ("ms_gather", dbl),
                ("ms_gather_kernels", dbl), ("ms_apply_kernels", dbl),
                ("kernel_launches", u64), ("gather_launches", u64),
                ("ms_storage", dbl), ("storage_rows", u64), ("storage_bytes", u64),
                ("fill_rows", u64), ("gather_kernel_rows", u64), ("fused_fill", u32), ("reserved0", u32)]


class ExchangeStatsC(C.Structure):
    _fields_ = [("calls", u64), ("rows_requested", u64), ("rows_remote", u64), ("rows_served", u64),
                ("bytes_sent", u64), ("ms", dbl)]


class StorageStatsC(C.Structure):
    _fields_ = [("rows", u64), ("preads", u64), ("bytes", u64), ("h2d_bytes", u64), ("read_ms", dbl),
                ("threads", u32), ("direct", i32)]


PIO = C.POINTER(IoStatsC)

# name: (restype, [argtypes])  -- every symbol declared in include/gx_b200.h
SIGNATURES = {
    "gx_last_error": (cstr, []),
    "gx_version": (cstr, []),
    "gx_ctx_create": (i32, [i32, PVP]),
    "gx_ctx_destroy": (None, [vp]),
    "gx_ctx_synchronize": (i32, [vp]),
    "gx_ctx_stream": (vp, [vp]),
    "gx_mix64": (u64, [u64]),
    "gx_derive_seed": (u64, [u64, u64]),
    "gx_pages_touched": (u64, [u64, u64]),
    "gx_page_count_for_row": (i32, [u64, u64, P64]),
    "gx_derive_train_ids": (i32, [u64, u64, dbl, vp, P64]),
    "gx_plan_seed_batches": (i32, [vp, u64, u64, u64, vp]),
    "gx_epoch_seed": (u64, [u64, u64]),
    "gx_graph_open": (i32, [vp, cstr, PVP]),
    "gx_graph_from_csc": (i32, [vp, u64, vp, vp, PVP]),
    "gx_graph_generate_rmat": (i32, [vp, u64, dbl, dbl, dbl, dbl, u64, PVP]),
    "gx_graph_destroy": (None, [vp]),
    "gx_graph_num_nodes": (u64, [vp]),
    "gx_graph_num_edges": (u64, [vp]),
    "gx_graph_in_degree": (i32, [vp, u64, P64]),
    "gx_graph_copy_csc": (i32, [vp, vp, vp]),
    "gx_graph_write": (i32, [vp, cstr]),
    "gx_graph_partition_bounds": (i32, [vp, i32, vp]),
    "gx_graph_partition": (i32, [vp, i32, i32]),
    "gx_graph_ipc_handle": (i32, [vp, vp, P64, P64]),
    "gx_graph_attach_peers": (i32, [vp, vp, vp]),
    "gx_graph_attach_local": (i32, [vp, vp, i32]),
    "gx_graph_partition_info": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
    "gx_sample_superbatch": (i32, [vp, vp, vp, u64, vp, u32, u64, u64, PVP, PIO]),
    "gx_sample_batch": (i32, [vp, vp, u64, vp, u32, u64, PVP, PIO]),
    "gx_samples_destroy": (None, [vp]),
    "gx_samples_num_batches": (u64, [vp]),
    "gx_samples_num_layers": (u32, [vp]),
    "gx_samples_batch_info": (i32, [vp, u64, P64, P64, vp]),
    "gx_samples_copy_ids": (i32, [vp, u64, vp]),
    "gx_samples_copy_edges": (i32, [vp, u64, u32, vp]),
    "gx_samples_total_edges": (u64, [vp]),
    "gx_samples_write_files": (i32, [vp, cstr, u64]),
    "gx_precompute_trace": (i32, [vp, vp, vp, u64, u64, u64, PVP]),
    "gx_simulate_trace": (i32, [vp, vp, vp, u64, u64, u64, vp, u64, PVP]),
    "gx_precompute_samples": (i32, [vp, u64, u64, PVP]),
    "gx_access_index": (i32, [vp, vp, vp, u64, u64, vp, vp]),
    "gx_changesets_destroy": (None, [vp]),
    "gx_changesets_num_iters": (u64, [vp]),
    "gx_changesets_init": (i32, [vp, vp, P64]),
    "gx_changesets_init_size": (u64, [vp]),
    "gx_changesets_iter_info": (i32, [vp, u64, P64, P64, P64]),
    "gx_changesets_copy_iter": (i32, [vp, u64, vp, vp, vp]),
    "gx_changesets_misses": (i32, [vp, vp]),
    "gx_changesets_write_files": (i32, [vp, cstr, u64]),
    "gx_features_open": (i32, [vp, cstr, i32, PVP]),
    "gx_features_write": (i32, [vp, cstr]),
    "gx_ncache_build": (i32, [vp, u64, PIO, PVP]),
    "gx_ncache_open": (i32, [vp, cstr, PIO, PVP]),
    "gx_ncache_write": (i32, [vp, cstr]),
    "gx_ncache_destroy": (None, [vp]),
    "gx_ncache_cached_nodes": (u64, [vp]),
    "gx_ncache_bytes_used": (u64, [vp]),
    "gx_ncache_contains": (i32, [vp, u64, C.POINTER(C.c_int)]),
    "gx_graph_set_neighbor_cache": (i32, [vp, vp]),
    "gx_static_degree_set": (i32, [vp, u64, vp]),
    "gx_pipeline_set_overlap": (i32, [vp, i32]),
    "gx_simulate_static_degree": (i32, [vp, vp, vp, u64, u64, vp]),
    "gx_simulate_lru": (i32, [vp, vp, vp, u64, u64, u64, vp]),
    "gx_features_generate_fp16": (i32, [vp, u64, u32, u64, PVP]),
    "gx_comm_unique_id": (i32, [vp]),
    "gx_comm_init_nccl": (i32, [vp, vp, i32, i32, PVP]),
    "gx_comm_init_local": (i32, [vp, i32, vp]),
    "gx_comm_init_host": (i32, [vp, i32, i32, vp, vp, PVP]),
    "gx_comm_destroy": (None, [vp]),
    "gx_comm_rank": (i32, [vp]),
    "gx_comm_size": (i32, [vp]),
    "gx_partition_bounds": (i32, [u64, i32, i32, P64, P64]),
    "gx_features_partitioned_from_host": (i32, [vp, vp, u64, u32, u32, vp, PVP]),
    "gx_features_partitioned_open": (i32, [vp, vp, cstr, PVP]),
    "gx_features_partitioned_generate": (i32, [vp, vp, u64, u32, u32, u64, PVP]),
    "gx_features_exchange_stats": (i32, [vp, vp]),
    "gx_features_storage_stats": (i32, [vp, vp]),
    "gx_features_from_host": (i32, [vp, u64, u32, u32, vp, i32, PVP]),
    "gx_features_generate": (i32, [vp, u64, u32, u64, PVP]),
    "gx_features_destroy": (None, [vp]),
    "gx_features_num_nodes": (u64, [vp]),
    "gx_features_dim": (u32, [vp]),
    "gx_features_row_bytes": (u64, [vp]),
    "gx_features_read_rows": (i32, [vp, vp, u64, vp, PIO]),
    "gx_batch_create": (i32, [vp, PVP]),
    "gx_batch_destroy": (None, [vp]),
    "gx_batch_rows": (u64, [vp]),
    "gx_batch_copy_to_host": (i32, [vp, vp]),
    "gx_batch_device_ptr": (vp, [vp]),
    "gx_batch_upload": (i32, [vp, vp, u64, u64]),
    "gx_cache_create": (i32, [vp, vp, u64, u64, PIO, PVP]),
    "gx_cache_destroy": (None, [vp]),
    "gx_cache_num_entries": (u64, [vp]),
    "gx_cache_gather": (i32, [vp, vp, u64, vp, P64, P64, PIO]),
    "gx_cache_apply": (i32, [vp, vp, vp, u64, vp, vp, u64, vp, u64]),
    "gx_cache_contains": (i32, [vp, u64, C.POINTER(C.c_int)]),
    "gx_cache_cached_row": (i32, [vp, u64, vp]),
    "gx_cache_resident_set": (i32, [vp, vp, u64, P64]),
    "gx_pipeline_create": (i32, [vp, vp, vp, u32, u64, PVP]),
    "gx_pipeline_destroy": (None, [vp]),
    "gx_pipeline_superbatch": (i32, [vp, vp, vp, u64, u64, u64, vp, C.POINTER(PipelineStatsC)]),
    "gx_pipeline_submit": (i32, [vp, vp, vp, u64, u64, u64, P64]),
    "gx_pipeline_wait": (i32, [vp, u64, vp, C.POINTER(PipelineStatsC)]),
    "gx_pipeline_exec_stream": (vp, [vp]),
    "gx_pipeline_batch": (i32, [vp, u64, u64, C.POINTER(vp), P64, vp]),
    "gx_pipeline_set_digest": (i32, [vp, i32]),
    "gx_pipeline_digests": (i32, [vp, vp]),
    "gx_pipeline_cache_rows": (i32, [vp, vp]),
    "gx_pipeline_copy_superbatch": (i32, [vp, u64, vp, u64, P64]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


# gx_status -> the Python image of the reference's C++ exception type
class LogicError(Exception):
    """std::logic_error"""


class CudaError(RuntimeError):
    """device failure (no reference counterpart)"""


_STATUS = {1: ValueError, 2: IndexError, 3: LogicError, 4: RuntimeError, 5: OverflowError,
           6: CudaError}


def check(rc: int) -> None:
    if rc:
        msg = (lib.gx_last_error() or b"").decode(errors="replace")
        raise _STATUS.get(rc, RuntimeError)(msg)
