"""B200-native Ginex data-preparation hot path (arXiv 2208.09151).

sampler -> Belady inspector -> feature-cache executor, as sm_100a CUDA kernels
behind the C-ABI in include/gx_b200.h. The Python API mirrors the reference's
host API (see api.py); importing fails if libgx_b200.so has not been built.
"""
from ._lib import LIB_PATH, CudaError, LogicError  # noqa: F401  (raises ImportError if unbuilt)
from .api import *  # noqa: F401,F403
from .api import (AccessIndex, Batch, Changeset, Changesets, Context, FeatureCache,  # noqa: F401
                  FeatureFile, FileTrace, GatherCounts, GraphFile, IoStats, MemoryTrace, Pipeline,
                  PipelineStats, PrecomputeResult, SampleOutput, Samples, SeedPlan,
                  SimulationResult, SplitMix64, batch_digest, build_access_index, compute_init_set,
                  derive_train_ids, epoch_seed,
                  derive_seed, mix64, page_count_for_row, pages_touched, plan_seed_batches,
                  precompute_changesets, precompute_trace, read_adj_file, read_ids_file,
                  read_init_file, read_update_file, sample_batch, sample_superbatch,
                  simulate_changesets, superbatch_sample)

__version__ = "0.1.0"
