/* gx_b200.h -- C-ABI of the B200-native Ginex data-preparation hot path.
 *
 * The reference ("gx", header-only C++20 at /root/reference/proj/include/gx) is
 * bound by C++ callers; this header is the drop-in boundary a maintainer binds
 * instead (see INTEGRATION.md for the C++ adapter and the ctypes binding used by
 * the Python mirror in paper_2208_09151_b200/api.py). Every entry point names the
 * reference interface it replaces as file:line relative to /root/reference/proj.
 *
 * Conventions
 *  - Plain pointers + sizes only; host pointers unless a name ends in _dev.
 *  - Node ids are u64 at the boundary (as in the reference, common.hpp:22) and
 *    u32 on the device; graphs with >= 2^32-1 nodes are rejected (GX_OVERFLOW).
 *  - Every call returns gx_status. On failure gx_last_error() holds the message
 *    (thread-local). The status maps 1:1 onto the C++ exception type the
 *    reference throws at the same point (std::invalid_argument, out_of_range,
 *    logic_error, runtime_error, overflow_error); the C++ adapter rethrows it.
 *  - Validation happens before any state mutation, as in the reference
 *    (feature_cache.hpp:96-112).
 *  - Handles are opaque; results live in device memory until copied out.
 */
#ifndef GX_B200_H
#define GX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gx_status {
    GX_OK = 0,
    GX_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    GX_OUT_OF_RANGE = 2,     /* std::out_of_range */
    GX_LOGIC_ERROR = 3,      /* std::logic_error */
    GX_RUNTIME_ERROR = 4,    /* std::runtime_error (I/O, format) */
    GX_OVERFLOW = 5,         /* std::overflow_error */
    GX_CUDA_ERROR = 6        /* device failure (no reference counterpart) */
} gx_status;

/* IoStats (common.hpp:32-45): same field order and meaning. */
typedef struct gx_iostats {
    uint64_t pages_read;
    uint64_t rows_read;
    uint64_t neighbor_lists_read;
    uint64_t bytes_read;
} gx_iostats;

const char* gx_last_error(void);
const char* gx_version(void);

/* ---- context: one per process per GPU ---------------------------------- */
typedef struct gx_ctx gx_ctx;
gx_status gx_ctx_create(int device, gx_ctx** out);
void gx_ctx_destroy(gx_ctx* ctx);
gx_status gx_ctx_synchronize(gx_ctx* ctx);
/* the cudaStream_t all work of this context is ordered on */
void* gx_ctx_stream(gx_ctx* ctx);

/* ---- primitives (common.hpp:48-61, 90-101) ------------------------------ */
uint64_t gx_mix64(uint64_t z);
uint64_t gx_derive_seed(uint64_t base, uint64_t index);
uint64_t gx_pages_touched(uint64_t lo, uint64_t hi);
gx_status gx_page_count_for_row(uint64_t row_bytes, uint64_t row_index, uint64_t* pages);

/* ---- seed plans (host-side, as in the reference) -------------------------
 * derive_train_ids (pipeline.hpp:384-399): partial Fisher-Yates over [0,n)
 * under derive_seed(mix64(seed) ^ 0x545241494E, 0), first floor(n*frac)
 * (clamped to [1,n]) ids, sorted. `out` needs n entries of scratch. */
gx_status gx_derive_train_ids(uint64_t n, uint64_t seed, double train_fraction, uint64_t* out,
                              uint64_t* n_out);
/* plan_seed_batches (sampler.hpp:48-65): the shuffled order (batches are
 * consecutive runs of batch_size); epoch_seed per pipeline.hpp:380-382. */
gx_status gx_plan_seed_batches(const uint64_t* train, uint64_t n, uint64_t batch_size,
                               uint64_t epoch_seed, uint64_t* shuffled);
uint64_t gx_epoch_seed(uint64_t seed, uint64_t epoch);

/* ---- graph: GraphFile (graph_store.hpp:106-197), CscGraph (:33-49) ------
 * The whole CSC (indptr u64[N+1], indices u32[E]) is HBM-resident. */
typedef struct gx_graph gx_graph;
/* GraphFile::open (graph_store.hpp:108-133): same header checks and errors. */
gx_status gx_graph_open(gx_ctx* ctx, const char* path, gx_graph** out);
/* from a host CSC (CscGraph layout, graph_store.hpp:33-36) */
gx_status gx_graph_from_csc(gx_ctx* ctx, uint64_t num_nodes, const uint64_t* indptr,
                            const uint64_t* indices, gx_graph** out);
/* generate_edges + build_csc on the device (graphgen.hpp:55-70,
 * graph_store.hpp:53-81): byte-identical CSC to the reference generator. */
gx_status gx_graph_generate_rmat(gx_ctx* ctx, uint64_t num_nodes, double avg_degree, double a,
                                 double b, double c, uint64_t edge_seed, gx_graph** out);
void gx_graph_destroy(gx_graph* g);
uint64_t gx_graph_num_nodes(const gx_graph* g);
uint64_t gx_graph_num_edges(const gx_graph* g);
/* GraphFile::in_degree (graph_store.hpp:138-141) */
gx_status gx_graph_in_degree(const gx_graph* g, uint64_t v, uint64_t* deg);
/* copy the CSC back to the host (load_graph, graph_store.hpp:202-215) */
gx_status gx_graph_copy_csc(const gx_graph* g, uint64_t* indptr, uint64_t* indices);
/* persist_graph (graph_store.hpp:83-98): writes graph.bin byte-identically */
gx_status gx_graph_write(const gx_graph* g, const char* path);

/* ---- row-partitioned CSC over the GPUs of one box -----------
 * The reference reads every in-neighbour list of sample_batch's layer loop
 * from one graph.bin (sampler.hpp:89-115 -> GraphFile::read_in_neighbors,
 * graph_store.hpp:145-154). Here rank r of P keeps the lists of nodes
 * [bounds[r], bounds[r+1]) -- bounds balanced by edge count, no list split --
 * and the replicated indptr. The per-layer request/response exchange is fused
 * into the sampler kernel: a draw's child id is loaded from the owner's HBM
 * through a CUDA IPC peer mapping (NVLink/NVSwitch), so sampled output is
 * bit-identical to the whole-CSC path (the draws depend only on degrees, which
 * indptr gives every rank). Collective use: every rank partitions, exports its
 * handle, and attaches all handles in rank order.
 * After gx_graph_partition, copy_csc / write / neighbor-cache build / static
 * degree policy fail with GX_LOGIC_ERROR; sampling fails until attached. */
#define GX_IPC_HANDLE_BYTES 64
#define GX_MAX_PARTS 16
/* node bounds[nranks + 1] of the edge-balanced partition */
gx_status gx_graph_partition_bounds(const gx_graph* g, int nranks, uint64_t* node_bounds);
/* keep only rank `rank`'s lists (frees the others' share of indices) */
gx_status gx_graph_partition(gx_graph* g, int nranks, int rank);
/* this rank's edge range and the IPC handle of its indices allocation */
gx_status gx_graph_ipc_handle(const gx_graph* g, void* handle, uint64_t* edge_lo, uint64_t* edge_hi);
/* map every peer's partition: handles[q * GX_IPC_HANDLE_BYTES] and edge_lo_hi[2q..2q+1]
 * from rank q (this rank's own entry is ignored); the edge ranges must match */
gx_status gx_graph_attach_peers(gx_graph* g, const void* handles, const uint64_t* edge_lo_hi);
/* in-process form (P ranks on one device in one process, tests): parts[q] is rank q's graph */
gx_status gx_graph_attach_local(gx_graph* g, gx_graph* const* parts, int nranks);
/* partition count (0 = whole CSC) and this graph's rank */
gx_status gx_graph_partition_info(const gx_graph* g, int* nranks, int* rank, int* attached);

/* ---- static neighbor cache (neighbor_cache.hpp) --------------------------
 * The CSC is HBM-resident, so the cache changes only the sampler's IoStats (a
 * cached list charges nothing, sampler.hpp:91-97), exactly as in the
 * reference; the address table and cache array are kept for ncache.bin. */
typedef struct gx_ncache gx_ncache;
/* build_neighbor_cache (neighbor_cache.hpp:88-116): greedy by out/in degree
 * (descending, ties by id) within budget_bytes (address table + regions) */
gx_status gx_ncache_build(gx_graph* g, uint64_t budget_bytes, gx_iostats* io, gx_ncache** out);
/* load_neighbor_cache / persist_neighbor_cache (neighbor_cache.hpp:118-148) */
gx_status gx_ncache_open(gx_graph* g, const char* path, gx_iostats* io, gx_ncache** out);
gx_status gx_ncache_write(const gx_ncache* c, const char* path);
void gx_ncache_destroy(gx_ncache* c);
uint64_t gx_ncache_cached_nodes(const gx_ncache* c);
uint64_t gx_ncache_bytes_used(const gx_ncache* c);   /* NeighborCache::bytes_used */
gx_status gx_ncache_contains(const gx_ncache* c, uint64_t v, int* out);
/* the sampler calls on this graph (and its pipelines) consult `c` (NULL: none);
 * `c` must outlive its use */
gx_status gx_graph_set_neighbor_cache(gx_graph* g, const gx_ncache* c);

/* ---- comparison policies of `gx simulate` (baselines.hpp) ----------------
 * static_degree_set (baselines.hpp:50-62): the K nodes of highest out-degree
 * (out-degrees from this graph's CSC), ties by lower id, in that order. */
gx_status gx_static_degree_set(gx_graph* g, uint64_t num_entries, uint64_t* out);
/* simulate_policy(..., static_degree) (baselines.hpp:81-96): per-iteration
 * misses of a fixed resident set over a trace of distinct-id lists. The belady
 * policy is gx_precompute_trace's misses; none = every access; LRU: gx_simulate_lru. */
gx_status gx_simulate_static_degree(gx_graph* g, const uint64_t* ids_flat, const uint64_t* offsets,
                                    uint64_t n_iters, uint64_t num_entries, uint64_t* misses);
/* LRU policy (baselines.hpp:104-128): per-iteration misses of an LRU cache of
 * K entries over the trace, from per-access stack distances on the device
 * (prev-access sort + a merge-sort inversion count; baselines.cu). */
gx_status gx_simulate_lru(gx_ctx* ctx, const uint64_t* ids_flat, const uint64_t* offsets, uint64_t S,
                          uint64_t num_nodes, uint64_t K, uint64_t* misses);

/* ---- sampler (sampler.hpp) ---------------------------------------------- */
typedef struct gx_samples gx_samples; /* S batches: ids + per-layer edges, on device */
/* superbatch_sample (sampler.hpp:197-243) minus the file writes (see
 * gx_samples_write_files): batch i is seeded derive_seed(global_seed,
 * first_global_batch + i). seeds_flat/batch_offsets give S seed lists. */
gx_status gx_sample_superbatch(gx_graph* g, const uint64_t* seeds_flat,
                               const uint64_t* batch_offsets, uint64_t n_batches,
                               const uint32_t* fanouts, uint32_t n_layers, uint64_t global_seed,
                               uint64_t first_global_batch, gx_samples** out, gx_iostats* io);
/* sample_batch (sampler.hpp:69-117) with an explicit batch seed. */
gx_status gx_sample_batch(gx_graph* g, const uint64_t* seeds, uint64_t n_seeds,
                          const uint32_t* fanouts, uint32_t n_layers, uint64_t batch_seed,
                          gx_samples** out, gx_iostats* io);
void gx_samples_destroy(gx_samples* s);
uint64_t gx_samples_num_batches(const gx_samples* s);
uint32_t gx_samples_num_layers(const gx_samples* s);
/* SampleOutput sizes (sampler.hpp:36-40): ids count, seed count, edges per layer */
gx_status gx_samples_batch_info(const gx_samples* s, uint64_t b, uint64_t* n_ids,
                                uint64_t* n_seeds, uint64_t* layer_counts);
gx_status gx_samples_copy_ids(const gx_samples* s, uint64_t b, uint64_t* ids);
/* (src_local, dst_local) u32 pairs of one layer (LocalEdge, sampler.hpp:34) */
gx_status gx_samples_copy_edges(const gx_samples* s, uint64_t b, uint32_t layer, uint32_t* pairs);
/* total sampled edges over all batches/layers */
uint64_t gx_samples_total_edges(const gx_samples* s);
/* write ids_{sb}_{i}.bin / adj_{sb}_{i}.bin (sampler.hpp:123-182, FORMATS.md) */
gx_status gx_samples_write_files(const gx_samples* s, const char* dir, uint64_t sb_index);

/* ---- inspector (changeset.hpp) ------------------------------------------ */
typedef struct gx_changesets gx_changesets;
/* precompute_changesets (changeset.hpp:468-484) minus the files: init set =
 * compute_init_set (:137-153), changesets = simulate_changesets (:228-295).
 * Trace = S distinct-id lists given flat with offsets[S+1]. */
gx_status gx_precompute_trace(gx_ctx* ctx, const uint64_t* ids_flat, const uint64_t* offsets,
                              uint64_t n_iters, uint64_t num_nodes, uint64_t num_entries,
                              gx_changesets** out);
/* same, with an explicit init set (simulate_changesets' `init`, :230) */
gx_status gx_simulate_trace(gx_ctx* ctx, const uint64_t* ids_flat, const uint64_t* offsets,
                            uint64_t n_iters, uint64_t num_nodes, uint64_t num_entries,
                            const uint64_t* init, uint64_t n_init, gx_changesets** out);
/* precompute over a device-resident sampler result (the inspector stage of
 * the pipeline: no host round trip of the ids trace) */
gx_status gx_precompute_samples(const gx_samples* s, uint64_t num_nodes, uint64_t num_entries,
                                gx_changesets** out);
/* build_access_index (changeset.hpp:124-129): iters[A+1] and ptr[N], byte
 * layout of AccessIndex including MSB region flags and the dummy tail. */
gx_status gx_access_index(gx_ctx* ctx, const uint64_t* ids_flat, const uint64_t* offsets,
                          uint64_t n_iters, uint64_t num_nodes, uint64_t* iters, uint64_t* ptr);
void gx_changesets_destroy(gx_changesets* cs);
uint64_t gx_changesets_num_iters(const gx_changesets* cs);
/* init set in admission (slot) order */
gx_status gx_changesets_init(const gx_changesets* cs, uint64_t* out, uint64_t* n);
uint64_t gx_changesets_init_size(const gx_changesets* cs);
/* Changeset sizes + SimulationResult::misses[i] (changeset.hpp:161-178) */
gx_status gx_changesets_iter_info(const gx_changesets* cs, uint64_t i, uint64_t* n_in,
                                  uint64_t* n_out, uint64_t* misses);
/* in_ids (by position), out_ids (by id), in_positions */
gx_status gx_changesets_copy_iter(const gx_changesets* cs, uint64_t i, uint64_t* in_ids,
                                  uint64_t* out_ids, uint64_t* in_positions);
/* all per-iteration misses (SimulationResult::misses) */
gx_status gx_changesets_misses(const gx_changesets* cs, uint64_t* misses);
/* write init_{sb}.bin + update_{sb}_{i}.bin (changeset.hpp:409-454) */
gx_status gx_changesets_write_files(const gx_changesets* cs, const char* dir, uint64_t sb_index);

/* ---- executor: feature table + FeatureCache (feature_cache.hpp) ---------- */
typedef struct gx_features gx_features;
typedef enum gx_backing {
    GX_BACKING_DEVICE = 0, /* whole table in HBM (fits one B200 up to ~150 GB) */
    GX_BACKING_HOST = 1,   /* pinned host memory, misses read over PCIe by the gather kernel */
    GX_BACKING_PARTITIONED = 3, /* row-partitioned across ranks (gx_features_partitioned_*): rows
                              of other ranks are fetched by a variable all-to-all (NCCL) */
    GX_BACKING_FILE = 2    /* the 'SSD' tier: features.bin stays on storage; the rows a
                              superbatch misses (cache init + changeset misses) are read with
                              pread (O_DIRECT when the filesystem allows it, whole 4 KB pages)
                              by a host thread pool into pinned staging and copied to HBM on a
                              side stream (FeatureFile::read_row, graph_store.hpp:308-315) */
} gx_backing;
/* FeatureFile::open (graph_store.hpp:282-302) + load of the payload (DEVICE,
 * HOST) or an open descriptor only (FILE). With GX_BACKING_FILE, ctx may be
 * NULL: the handle then serves gx_features_read_rows from the host only. */
gx_status gx_features_open(gx_ctx* ctx, const char* path, int backing, gx_features** out);
/* FeatureWriter (graph_store.hpp:237-250): writes features.bin (36-byte header,
 * payload at 4096) from a DEVICE or HOST backed table. */
gx_status gx_features_write(const gx_features* f, const char* path);
/* Storage-tier counters of a GX_BACKING_FILE table since open (physical reads;
 * the reference's page accounting stays in gx_iostats). direct = 1 when reads
 * bypass the page cache (O_DIRECT). */
typedef struct gx_storage_stats {
    uint64_t rows;        /* rows delivered */
    uint64_t preads;      /* pread calls (one per coalesced page run) */
    uint64_t bytes;       /* bytes read from storage (whole pages) */
    uint64_t h2d_bytes;   /* bytes copied pinned -> HBM */
    double read_ms;       /* wall time of the host read phase (all workers) */
    uint32_t threads;     /* reader threads */
    int32_t direct;       /* 1 = O_DIRECT, 0 = buffered fallback */
} gx_storage_stats;
gx_status gx_features_storage_stats(const gx_features* f, gx_storage_stats* out);
/* from host rows (RowMatrix layout, graph_store.hpp:222-234); row_bytes =
 * dim * scalar_width (scalar_width 4 = the reference format; 2 = fp16 ext.) */
gx_status gx_features_from_host(gx_ctx* ctx, uint64_t num_nodes, uint32_t dim,
                                uint32_t scalar_width, const void* rows, int backing,
                                gx_features** out);
/* generate the table on the device: feature_value (graphgen.hpp:74-77) */
gx_status gx_features_generate(gx_ctx* ctx, uint64_t num_nodes, uint32_t dim,
                               uint64_t value_seed, gx_features** out);
/* fp16 extension (scalar_width 2, cfg4 MAG240M-shape): element = the fp16
 * round-to-nearest-even of feature_value */
gx_status gx_features_generate_fp16(gx_ctx* ctx, uint64_t num_nodes, uint32_t dim, uint64_t value_seed,
                                    gx_features** out);
void gx_features_destroy(gx_features* f);
uint64_t gx_features_num_nodes(const gx_features* f);
uint32_t gx_features_dim(const gx_features* f);
uint64_t gx_features_row_bytes(const gx_features* f);
/* FeatureFile::read_rows (graph_store.hpp:319-324) into host memory */
gx_status gx_features_read_rows(gx_features* f, const uint64_t* ids, uint64_t n, void* out,
                                gx_iostats* io);

/* ---- multi-GPU: row-partitioned feature table -----------
 * The reference is single-process (its only parallelism is a thread pool,
 * sampler.hpp:205-235); this is the B200 extension north_star asks for. One
 * process per GPU (or, for tests, one host thread per rank). Rank r of P owns
 * feature rows [N*r/P, N*(r+1)/P) in its HBM. Every row a rank's cache needs
 * from the backing store (cache init, changeset misses) is fetched by ONE
 * variable all-to-all per request set: per-owner request lists (u32 local ids)
 * out, rows back, as grouped NCCL send/recv over NVLink/NVSwitch; the owner
 * serves them with the row-gather kernel. Collective: every rank must make
 * the same sequence of calls that touch a partitioned table (pipeline
 * superbatches, cache create/gather), with empty request sets where it has none. */
typedef struct gx_comm gx_comm;
#define GX_COMM_ID_BYTES 128
/* a fresh NCCL unique id (rank 0 creates it, the caller broadcasts the bytes) */
gx_status gx_comm_unique_id(void* id_out);
/* NCCL communicator over this context's GPU (libnccl.so.2 resolved at run time) */
gx_status gx_comm_init_nccl(gx_ctx* ctx, const void* id, int nranks, int rank, gx_comm** out);
/* in-process transport: nranks contexts (one per host thread; they may share a
 * GPU), peer copies through the CUDA runtime; outs[r] belongs to ctxs[r] */
gx_status gx_comm_init_local(gx_ctx* const* ctxs, int nranks, gx_comm** outs);
/* host-staged transport: device bytes are staged through pinned host buffers and
 * exchanged by the caller's callback (MPI / gloo / sockets) -- for ranks NCCL
 * cannot connect (e.g. several processes sharing one GPU). The callback sends
 * send[sum(scnt[<p]) ..] (scnt[p] bytes) to rank p and receives rcnt[p] bytes
 * from rank p into recv (packed in rank order); returns 0 on success. It is
 * called collectively, in the same order on every rank. */
typedef int (*gx_host_alltoallv_fn)(void* user, const void* send, const uint64_t* scnt, void* recv,
                                    const uint64_t* rcnt);
gx_status gx_comm_init_host(gx_ctx* ctx, int nranks, int rank, gx_host_alltoallv_fn fn, void* user,
                            gx_comm** out);
void gx_comm_destroy(gx_comm* c);
int gx_comm_rank(const gx_comm* c);
int gx_comm_size(const gx_comm* c);
/* rows [lo, hi) owned by `rank` */
gx_status gx_partition_bounds(uint64_t num_nodes, int nranks, int rank, uint64_t* lo, uint64_t* hi);
/* this rank's partition from its own rows (host, (hi-lo) x row_bytes), from
 * features.bin (reads only this rank's rows) or generated (feature_value) */
gx_status gx_features_partitioned_from_host(gx_ctx* ctx, gx_comm* comm, uint64_t num_nodes, uint32_t dim,
                                            uint32_t scalar_width, const void* local_rows, gx_features** out);
gx_status gx_features_partitioned_open(gx_ctx* ctx, gx_comm* comm, const char* path, gx_features** out);
gx_status gx_features_partitioned_generate(gx_ctx* ctx, gx_comm* comm, uint64_t num_nodes, uint32_t dim,
                                           uint32_t scalar_width, uint64_t value_seed, gx_features** out);
typedef struct gx_exchange_stats {
    uint64_t calls;           /* all-to-all request sets served */
    uint64_t rows_requested;  /* rows this rank asked for (own partition included) */
    uint64_t rows_remote;     /* of those, rows owned by other ranks */
    uint64_t rows_served;     /* rows this rank sent to requesters (itself included) */
    uint64_t bytes_sent;      /* ids + rows this rank put on the wire to other ranks */
    double ms;                /* host wall time inside the exchanges */
} gx_exchange_stats;
gx_status gx_features_exchange_stats(const gx_features* f, gx_exchange_stats* out);

/* Gathered batch buffer (RowMatrix, graph_store.hpp:222-234), device resident. */
typedef struct gx_batch gx_batch;
gx_status gx_batch_create(gx_ctx* ctx, gx_batch** out);
void gx_batch_destroy(gx_batch* b);
uint64_t gx_batch_rows(const gx_batch* b);
gx_status gx_batch_copy_to_host(const gx_batch* b, void* out);
void* gx_batch_device_ptr(const gx_batch* b);
/* load host rows into a batch (e.g. a RowMatrix handed to apply_changeset) */
gx_status gx_batch_upload(gx_batch* b, const void* rows, uint64_t n_rows, uint64_t row_bytes);

typedef struct gx_cache gx_cache;
/* FeatureCache ctor (feature_cache.hpp:19-37): init ids -> slots 0..k-1. */
gx_status gx_cache_create(gx_features* f, const uint64_t* init, uint64_t n_init,
                          uint64_t num_entries, gx_iostats* io, gx_cache** out);
void gx_cache_destroy(gx_cache* c);
uint64_t gx_cache_num_entries(const gx_cache* c);
/* FeatureCache::gather (feature_cache.hpp:58-76) into a device batch */
gx_status gx_cache_gather(gx_cache* c, const uint64_t* ids, uint64_t n, gx_batch* out,
                          uint64_t* hits, uint64_t* misses, gx_iostats* io);
/* FeatureCache::apply_changeset (feature_cache.hpp:89-130) */
gx_status gx_cache_apply(gx_cache* c, const gx_batch* batch, const uint64_t* ids, uint64_t n_ids,
                         const uint64_t* in_ids, const uint64_t* in_positions, uint64_t n_in,
                         const uint64_t* out_ids, uint64_t n_out);
/* test hooks: contains / cached_row / resident_set (feature_cache.hpp:28-34,119-125) */
gx_status gx_cache_contains(const gx_cache* c, uint64_t v, int* out);
gx_status gx_cache_cached_row(const gx_cache* c, uint64_t v, void* out);
gx_status gx_cache_resident_set(const gx_cache* c, uint64_t* out, uint64_t cap, uint64_t* n);

/* ---- fused device pipeline (TrainingRunner::run_superbatch stages 1-4,
 * pipeline.hpp:338-377, minus the runtime files and the compute stub) ------
 * sample -> precompute -> cache init ("switch") -> S x (gather, apply), all on
 * the device; the ids trace, changesets and gathered batches never leave HBM.
 * The pipeline owns its buffers and reuses them across superbatches. */
typedef struct gx_pipeline gx_pipeline;
typedef struct gx_pipeline_stats {
    uint64_t sampled_edges;
    uint64_t gathered_rows;   /* = accesses A = sum |ids_i| */
    uint64_t total_misses;    /* observed by the gather; equals the inspector's prediction */
    uint64_t predicted_misses;
    uint64_t init_size;
    uint64_t total_in, total_out;
    gx_iostats sample_io;
    gx_iostats gather_io;
    double ms_sample, ms_inspect, ms_switch, ms_gather; /* device-timed stage durations */
    double ms_gather_kernels;  /* sum of the S gather-kernel durations (CUDA events) */
    double ms_apply_kernels;   /* sum of the S apply-kernel durations */
    uint64_t kernel_launches;  /* this library's kernel launches for the superbatch
                                  (sampler, inspector, cache init, gathers, non-empty applies) */
    uint64_t gather_launches;  /* gather launches: one per run of iterations with empty changesets */
    /* GX_BACKING_FILE only (zero otherwise): the superbatch's storage reads */
    double ms_storage;         /* wall time of the host read phase (pread + staging) */
    uint64_t storage_rows;     /* rows read: cache init + changeset misses */
    uint64_t storage_bytes;    /* bytes read from storage (whole pages) */
    /* executor kernel work, for roofline accounting */
    uint64_t fill_rows;        /* rows the switch wrote into cache slots (= init_size) */
    uint64_t gather_kernel_rows; /* rows the gather launches moved (all accesses; fused_fill 1:
                                    the accesses that are not an init node's first use; fused_fill 2:
                                    0, or all accesses fanned out from the cache on staged tiers;
                                    fused_fill 3: the accesses the init rows do not serve) */
    uint32_t fused_fill;       /* all-fit superbatch: 1 = the switch also wrote each init node's
                                  first-use batch row; 2 = fan-out: each init row was read once and
                                  written to its slot and to every batch row of its node;
                                  changeset superbatch: 3 = each init row was read once and written
                                  to its slot and to every access it serves (slot still holding it) */
    uint32_t reserved0;
} gx_pipeline_stats;
gx_status gx_pipeline_create(gx_graph* g, gx_features* f, const uint32_t* fanouts,
                             uint32_t n_layers, uint64_t num_entries, gx_pipeline** out);
void gx_pipeline_destroy(gx_pipeline* p);
gx_status gx_pipeline_superbatch(gx_pipeline* p, const uint64_t* seeds_flat,
                                 const uint64_t* batch_offsets, uint64_t n_batches,
                                 uint64_t global_seed, uint64_t first_global_batch,
                                 uint64_t* misses_per_iter, gx_pipeline_stats* stats);
/* Asynchronous, double-buffered form. submit() runs the sampler and the
 * inspector of a superbatch on the context stream and queues its executor
 * (cache init + S x gather/apply) on the pipeline's own stream, returning
 * without waiting for it, so the executor of superbatch k overlaps the
 * sampler/inspector of k+1 (the reference overlaps sample(k+1) with
 * precompute(k), pipeline.hpp:299-315). At most two superbatches may be in
 * flight; wait(ticket) returns that superbatch's results. gx_pipeline_superbatch
 * is submit + wait. */
gx_status gx_pipeline_submit(gx_pipeline* p, const uint64_t* seeds_flat,
                             const uint64_t* batch_offsets, uint64_t n_batches,
                             uint64_t global_seed, uint64_t first_global_batch, uint64_t* ticket);
gx_status gx_pipeline_wait(gx_pipeline* p, uint64_t ticket, uint64_t* misses_per_iter,
                           gx_pipeline_stats* stats);
/* With two superbatches in flight, 0 (default): the GPU runs superbatch k+1's
 * sampler after k's executor (stages back to back; only the host preparation
 * of k+1 overlaps k); 1: k+1's sampler/inspector run concurrently with k's
 * executor. */
gx_status gx_pipeline_set_overlap(gx_pipeline* p, int concurrent);
/* the cudaStream_t the executor of this pipeline runs on */
void* gx_pipeline_exec_stream(gx_pipeline* p);
/* Device pointer to iteration i's gathered rows (|ids_i| x row_bytes, the
 * RowMatrix of feature_cache.hpp:58 kept in HBM) of a waited-for superbatch.
 * Valid until the slot is resubmitted (ticket + 2). The executor keeps the whole
 * superbatch's batches resident (rows of iteration i at row offset
 * sum_{j<i}|ids_j|) when they fit the free HBM (or GX_BATCH_BUDGET_MB per slot);
 * otherwise it reuses one iteration-sized buffer and only the last iteration is
 * readable (GX_LOGIC_ERROR for the others). host_out (nullable) additionally
 * receives a copy of the rows. */
gx_status gx_pipeline_batch(gx_pipeline* p, uint64_t ticket, uint64_t i, const void** rows,
                            uint64_t* n_rows, void* host_out);
/* Every iteration's rows of a waited-for, HBM-resident superbatch copied to
 * host memory in one D2H (the S RowMatrix objects of the reference's executor
 * back to back; pinned host_out streams at PCIe rate). *bytes = rows x
 * row_bytes; host_out == NULL only reports the size. */
gx_status gx_pipeline_copy_superbatch(gx_pipeline* p, uint64_t ticket, void* host_out, uint64_t cap_bytes,
                                      uint64_t* bytes);

/* Optional per-iteration digest of each gathered batch (for end-to-end parity
 * checks; off by default, costs one extra read of every batch):
 *   digest_i = sum_k sum_j (w_kj + 1) * mix64(k * W + j)  (mod 2^64)
 * over the u32 words w_kj (W per row) of row k of iteration i's batch. */
gx_status gx_pipeline_set_digest(gx_pipeline* p, int enable);
gx_status gx_pipeline_digests(const gx_pipeline* p, uint64_t* digests_per_iter);
/* test hook: the feature cache's K slot rows (K x row_bytes) after the last
 * waited-for superbatch -- FeatureCache's rows after its last apply_changeset
 * (feature_cache.hpp:114-129); slots never filled are unspecified */
gx_status gx_pipeline_cache_rows(gx_pipeline* p, void* host_out);

#ifdef __cplusplus
}
#endif
#endif /* GX_B200_H */
