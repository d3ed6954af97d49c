// gx_internal.cuh -- definitions behind the opaque C-ABI handles.
#pragma once

#include <atomic>
#include <memory>

#include "gx_common.cuh"

namespace gx {
// The 'SSD' tier (storage.cu): a features.bin payload read with pread in whole
// 4 KB pages (O_DIRECT when the filesystem allows it) by a host thread pool.
struct RowReader {
    std::string path;
    int fd = -1;
    bool direct = false;
    uint64_t poff = 0, rb = 0, n = 0, fsize = 0;
    unsigned threads = 1;
    uint64_t run_cap = 0;    // bytes per pread (coalesced page run)
    uint64_t gap_pages = 0;  // merge runs separated by at most this many unneeded pages
    std::atomic<uint64_t> rows{0}, preads{0}, bytes{0}, h2d{0}, read_ns{0};
    RowReader(const char* path, uint64_t payload_off, uint64_t row_bytes, uint64_t n_rows);
    ~RowReader();
    // dst + q * rb <- row sorted[q] for q in [0, n); sorted ascending (runs coalesce)
    void read_sorted(const uint32_t* sorted, uint64_t n, uint8_t* dst);
    // any order (host-only API path): sorts a copy
    void read_rows(const uint64_t* ids, uint64_t n, uint8_t* dst);
  private:
    void read_range(const uint32_t* sorted, uint64_t lo, uint64_t hi, uint8_t* dst, uint8_t* bounce);
    void pread_full(uint8_t* dst, uint64_t len, uint64_t off, uint64_t need);
};
// Exchange scratch of a partitioned features handle (comm.cu).
struct PartScratch {
    DevBuf<uint32_t> keys, keys_alt, vals, vals_alt, send_ids, recv_ids;
    DevBuf<unsigned long long> counts;
    DevBuf<uint8_t> cub_tmp, send_rows, recv_rows;
    DevBuf<unsigned long long> dummy;
};
// Device-side staging scratch of one features handle (storage.cu).
struct StageScratch {
    DevBuf<uint32_t> keys, keys_alt, vals, vals_alt;
    DevBuf<uint8_t> cub_tmp;
    DevBuf<uint8_t> land[2];
    PinBuf<uint8_t> pin[2];
    PinBuf<uint32_t> h_sorted;
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr}, ev_ready = nullptr;
    ~StageScratch();
};
}  // namespace gx

namespace gx {
// Sampler scratch (sampler.cu); grow-only, reused across calls.
struct SampleScratch {
    DevBuf<uint32_t> F, T, seeds32;
    DevBuf<uint64_t> dbase, bseed, seed_off;
    DevBuf<uint32_t> pscan, pdeg, idslot;
    DevBuf<uint64_t> plo;
    DevBuf<uint32_t> tsum, tsum2;
    DevBuf<uint32_t> dslot, drank;
    DevBuf<unsigned long long> tab[2];
    uint64_t tab_slots = 0;  // per table, = S * tab_cap
    DevBuf<unsigned long long> io;
    DevBuf<uint32_t> tctr;  // dynamic tile counters (4 per layer), zeroed by the kernel
};
// Inspector scratch (inspector.cu).
struct InspectScratch {
    DevBuf<uint32_t> last;       // N, node-indexed "next access" cursor (kNever when clean)
    DevBuf<int32_t> node_slot;   // N, -1 when clean
    DevBuf<uint32_t> firstx;     // N, epoch-encoded first access (trusted traces)
    uint64_t fx_base = 0;        // last epoch handed out
    uint64_t N = 0;
    DevBuf<uint32_t> trace, next_use, acc_slot;
    DevBuf<uint64_t> trace_off;
    DevBuf<uint32_t> tile_cnt, slot_node, slot_key, hist_new, rh, pkey, out_node, out_slot, c_id,
        c_ref, in_node, in_pos, chunk_cnt, bm_words, bm_top, bm_cnt, init_ext, toff, st;
    DevBuf<int32_t> hist_inc;
    DevBuf<uint8_t> pmiss;
    // deferred-ordering recurrence (inspector.cu: recurrence_deferred, k_finish_changesets)
    DevBuf<uint32_t> slot_tag, slot_nk, pnk, out_raw, out_tagraw, tag_sorted, ev_slot, fin_unres, blk_max;
    DevBuf<int32_t> never_hist;
    DevBuf<uint8_t> sort_tmp;
    DevBuf<uint32_t> o_pack;  // 2 IStates (32 words), then misses / in_off / out_off (S+1 each)
    DevBuf<unsigned long long> bits;  // N * ceil(S/64) iteration bitmask, clean between calls
    uint64_t bits_words = 0;
    DevBuf<uint8_t> isfirst;
    DevBuf<int32_t> init_pos;         // N, -1 when clean (explicit-init API path)
    uint64_t init_pos_n = 0;
    std::vector<uint32_t> h_m, h_io, h_oo;
    gx::PinBuf<uint8_t> h_pin;  // pinned landing area of the post-inspector readback (one sync)
};
}  // namespace gx

struct gx_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    gx::DevBuf<gx::GridBarrier> barrier;  // one barrier per context (stream-serialised users)
    gx::SampleScratch ss;
    gx::InspectScratch is;
    gx::DevBuf<uint32_t> resolve_slots;  // executor API path scratch
    gx::DevBuf<uint32_t> stage_ids;      // API path: miss ids staged from storage
    gx::DevBuf<uint8_t> stage_rows;      // API path: their rows
    gx::DevBuf<uint32_t> miss_flags, miss_ranks;  // stage_misses scan scratch (storage.cu)
    gx::DevBuf<uint8_t> miss_tmp;
    cudaStream_t launch_stream = nullptr;  // executor launches go here when set (pipeline stream)
};

// stream the executor launchers use
inline cudaStream_t lstream(const gx_ctx* c) { return c->launch_stream ? c->launch_stream : c->stream; }

namespace gx {
constexpr int kMaxParts = 16;  // ranks of one box that can share a row-partitioned CSC
// Row-partitioned CSC: rank r holds the in-neighbour lists of
// nodes [node_bounds[r], node_bounds[r+1]) = edges [ebound[r], ebound[r+1])
// (bounds balanced by edge count, lists never split); indptr stays replicated.
// ptr[q] addresses rank q's edges (ptr[q][e - ebound[q]]): this rank's own
// buffer, or a peer's HBM mapped over NVLink through CUDA IPC.
struct GraphParts {
    int P = 0, rank = 0;
    bool attached = false;
    uint64_t node_bounds[kMaxParts + 1] = {};
    uint64_t ebound[kMaxParts + 1] = {};
    const uint32_t* ptr[kMaxParts] = {};
    std::vector<void*> ipc_opened;  // peer mappings to close
    ~GraphParts();
};
}  // namespace gx

struct gx_graph {
    gx_ctx* ctx = nullptr;
    uint64_t n = 0, e = 0;
    gx::DevBuf<uint64_t> indptr;   // N+1
    gx::DevBuf<uint32_t> indices;  // E (u32 device ids); partitioned: only this rank's edges
    const uint32_t* ncache_bits = nullptr;  // neighbor cache in use (bit v: list cached, charges no I/O)
    gx::GraphParts part;           // P == 0: not partitioned
};
namespace gx {
// operations that need every list on this device refuse a partitioned graph
inline void require_whole_csc(const gx_graph* g, const char* what) {
    if (g->part.P) fail(GX_LOGIC_ERROR, std::string(what) + " needs the whole CSC; the graph is row-partitioned");
}
}  // namespace gx

// Sampler output for S batches (SampleOutput x S, sampler.hpp:36-40).
// Per-batch regions have fixed capacities so every batch can be written in
// parallel without a device allocator.
struct gx_samples {
    gx_ctx* ctx = nullptr;
    uint64_t S = 0;
    uint32_t L = 0;
    std::vector<uint32_t> fanouts;
    uint64_t cap_ids = 0;                 // ids per batch
    std::vector<uint64_t> cap_e;          // per layer edge capacity per batch
    std::vector<uint64_t> e_off;          // per layer offset inside a batch's edge region
    uint64_t cap_e_batch = 0;             // sum of cap_e
    gx::DevBuf<uint32_t> ids;             // S * cap_ids
    gx::DevBuf<uint32_t> n_ids;           // S
    gx::DevBuf<uint2> edges;              // S * cap_e_batch  (src_local, dst_local)
    gx::DevBuf<uint32_t> layer_count;     // S * L
    bool dup_seed = false;                // a batch had a duplicate seed (set by samples_sync_host)
    std::vector<uint32_t> h_n_ids;        // host mirrors, valid after the call
    std::vector<uint32_t> h_layer_count;
    std::vector<uint64_t> h_n_seeds;
    gx::PinBuf<uint32_t> h_pin;  // pinned landing area of samples_sync_host (one sync)
    gx_iostats io{};
};

struct gx_changesets {
    gx_ctx* ctx = nullptr;
    uint64_t S = 0, N = 0, K = 0;
    uint64_t n_init = 0;
    gx::DevBuf<uint32_t> init;      // n_init (slot order)
    gx::DevBuf<uint32_t> in_ids;    // total in
    gx::DevBuf<uint32_t> in_pos;
    gx::DevBuf<uint32_t> in_slot;   // FeatureCache slot each insertion lands in
    gx::DevBuf<uint32_t> out_ids;   // total out (sorted per iteration)
    gx::DevBuf<uint32_t> first_acc; // all-fit: access index of each init slot's first use
    gx::DevBuf<uint32_t> rest_x, rest_slot;  // all-fit: the other accesses and their slots
    // all-fit, fan-out form: init slot r serves first_acc[r] and the accesses
    // fan_list[r ? fan_off[r - 1] : 0 .. fan_off[r])
    gx::DevBuf<uint32_t> fan_cnt, fan_off, fan_list;
    gx::DevBuf<uint8_t> cub_tmp;
    uint64_t n_rest = 0;
    bool first_marked = false;      // first_acc / rest_* (or fan_*) valid (pipeline only)
    bool fan = false;               // fan_off / fan_list valid
    std::vector<uint64_t> h_in_off, h_out_off, h_misses;  // S+1, S+1, S
};

struct gx_features {
    gx_ctx* ctx = nullptr;
    uint64_t n = 0;
    uint32_t dim = 0;
    uint32_t scalar_width = 4;
    uint64_t row_bytes = 0;
    int backing = GX_BACKING_DEVICE;
    gx::DevBuf<uint8_t> dev;       // device backing store
    gx::PinBuf<uint8_t> host;      // pinned host backing store (mapped)
    const uint8_t* rows_dev_view = nullptr;  // pointer usable by kernels
    std::unique_ptr<gx::RowReader> file;     // GX_BACKING_FILE
    std::unique_ptr<gx::StageScratch> stage;
    // GX_BACKING_PARTITIONED: this rank's rows [part_lo, part_hi) in `dev`
    gx_comm* comm = nullptr;
    uint64_t part_lo = 0, part_hi = 0;
    std::unique_ptr<gx::PartScratch> part;
    gx_exchange_stats xstats{};
};

struct gx_batch {
    gx_ctx* ctx = nullptr;
    uint64_t rows = 0;
    uint64_t row_bytes = 0;
    gx::DevBuf<uint8_t> data;
};

namespace gx {

// Device scratch for one superbatch of sampling; reused across calls.
struct SampleScratch;

// Internal entry points shared between translation units.
// firstx != nullptr (pipeline): also fill the inspector's first-use array with
// keys (b << 21 | local) under epoch fx_epoch; returns whether it did
bool sample_run(gx_graph* g, const uint64_t* seeds_flat, const uint64_t* batch_off, uint64_t S,
                const uint32_t* fanouts, uint32_t L, const uint64_t* batch_seeds,
                gx_samples* out, uint32_t* firstx = nullptr, uint32_t fx_epoch = 0);
// reserve an epoch of `keyrange` keys in the first-use array (allocated and
// zeroed for N nodes on first use, reset when the epochs wrap)
uint32_t inspect_reserve_epoch(gx_ctx* ctx, uint64_t N, uint64_t keyrange);
void samples_sync_host(gx_samples* s);

// Inspector (inspector.cu). The flat u32 trace lives in ctx->is.trace.
void inspect_fill_from_device(gx_ctx* ctx, const uint32_t* d_ids, uint64_t stride,
                              const std::vector<uint64_t>& off);
void inspect_fill_from_host(gx_ctx* ctx, const uint64_t* flat, const std::vector<uint64_t>& off,
                            uint64_t N);
// trusted: the trace comes from the sampler (ids < N, distinct per iteration)
// presampled_epoch != 0: the sampler already filled firstx with (b << 21 | local) keys
void inspect_run(gx_ctx* ctx, const std::vector<uint64_t>& off, uint64_t N, uint64_t K,
                 const uint64_t* h_init, int64_t n_init_explicit, gx_changesets* out, bool trusted,
                 int mark_first = 0, uint32_t presampled_epoch = 0);
void access_index_run(gx_ctx* ctx, const std::vector<uint64_t>& off, uint64_t N, uint64_t* h_iters,
                      uint64_t* h_ptr);

// Executor launchers (executor.cu).
void launch_gather(gx_ctx* ctx, const uint32_t* ids, uint64_t n, const int32_t* table,
                   const uint8_t* cache_rows, gx_features* f, uint8_t* out,
                   unsigned long long* counters);
// gather with the serving slot of every row already resolved (kNever = miss)
// staged: `store` is a staging buffer addressed by flagged slots (kStageFlag).
// seg_off != nullptr: segment mode -- rows of nseg consecutive iterations
// (absolute offsets seg_off[0..nseg]); misses/pages are charged per iteration
// into counters[8 * it + 1 / + 2] (executor.cu, SegInfo).
void launch_gather_resolved(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, uint64_t n,
                            const uint8_t* cache_rows, const uint8_t* store, uint64_t row_bytes, uint8_t* out,
                            unsigned long long* counters, const uint32_t* seg_off = nullptr, uint32_t nseg = 0,
                            bool staged = false, bool skip_first = false);
void launch_apply_slots(gx_ctx* ctx, const uint32_t* in_ids, const uint32_t* in_pos,
                        const uint32_t* in_slot, uint32_t n_in, const uint32_t* out_ids,
                        uint32_t n_out, int32_t* table, const uint8_t* batch, uint8_t* cache_rows,
                        uint64_t row_bytes);
// counters: 5 words as for the gather (init rows are charged as misses)
void launch_cache_init(gx_ctx* ctx, const uint32_t* init, uint32_t n, int32_t* table,
                       gx_features* f, uint8_t* cache_rows, unsigned long long* counters);
void launch_reset_table(gx_ctx* ctx, const uint32_t* nodes, uint64_t n, int32_t* table);
void launch_digest(gx_ctx* ctx, const uint8_t* batch, uint64_t rows, uint64_t row_bytes,
                   unsigned long long* out);
// whole resident superbatch in one bulk-copy launch (k_gather_sb): accesses
// whose slot still holds its init node read the cache, the rest the table;
// false if the row size does not suit the bulk-copy kernel
bool launch_gather_superbatch(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, uint64_t n,
                              const uint32_t* init, uint32_t n_init, const uint8_t* cache_rows, const uint8_t* store,
                              uint64_t rb, uint8_t* out);
// changeset regime, device-backed, whole superbatch resident: the switch fans
// each init row out to its slot and to every access it serves (init-served:
// acc_slot[x] = s < n_init with init[s] == trace[x]; rank[x] = its index in
// slot s's list, kNever otherwise); launch_gather_rest copies every access
// with rank kNever from the table. Scratch buffers are the caller's.
void launch_init_fan(gx_ctx* ctx, const uint32_t* trace, const uint32_t* acc_slot, uint64_t A, const uint32_t* init,
                     uint32_t n_init, const uint8_t* store, uint64_t rb, uint8_t* cache_rows, uint8_t* batch,
                     DevBuf<uint32_t>& cnt, DevBuf<uint32_t>& off, DevBuf<uint32_t>& list, DevBuf<uint32_t>& rank,
                     DevBuf<uint8_t>& tmp);
void launch_gather_rest(gx_ctx* ctx, const uint32_t* trace, const uint32_t* rank, uint64_t A, const uint8_t* store,
                        uint64_t rb, uint8_t* batch, unsigned long long* nrows);  // += rows copied
// every changeset of a superbatch applied at once (the cache is not read in
// between): each slot gets its last insert's batch row; `last` = K zeroed u32
// marks (left zeroed), in_off / bat_off = insert / batch-row offsets per iteration
void launch_apply_all(gx_ctx* ctx, const uint32_t* in_pos, const uint32_t* in_slot, const uint32_t* in_off,
                      uint32_t S, uint32_t n, const uint32_t* bat_off, uint32_t* last, const uint8_t* batch,
                      uint8_t* cache_rows, uint64_t rb);
// counters[8 i + 1 / + 2] += misses / pages of iteration i of a resolved access
// list (slot kNever = miss), d_off = the S + 1 iteration offsets on the device
void launch_count_iter_misses(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, const uint32_t* d_off,
                              uint32_t S, uint64_t maxw, uint64_t rb, unsigned long long* counters);

// Storage tier (storage.cu). A slot value with kStageFlag set (and != kNever)
// is a miss whose row was staged: the gather reads row (slot & ~kStageFlag)
// of the store pointer it is given and charges the miss to ids[k] as usual.
constexpr uint32_t kStageFlag = 0x80000000u;
// All-fit pipeline superbatches: the fused fill (launch_fill_first) serves the
// first use of every init slot; the other accesses come as a dense list
// (rest_x: batch row, rest_slot: cache slot) served by the gather's DSTIDX form
// (skip_first = true: ids = rest_x, slots = rest_slot).
void launch_fill_first(gx_ctx* ctx, const uint32_t* init, const uint32_t* first_acc, uint32_t n,
                       const uint8_t* store, uint64_t rb, uint8_t* cache_rows, uint8_t* batch);
// Fan-out form (mark_first = 2): each init row is read once and written to its
// cache slot (cache_rows != nullptr), to the batch row of its first use
// first[r] and to batch rows list[j] for j in [r ? off[r - 1] : 0, off[r]).
// idx == nullptr: source row r is row r of `src`; first == nullptr: no
// first-use rows (the staged tiers fan out from the filled cache to the other
// accesses only, reading just the slots that have any).
void launch_fan_rows(gx_ctx* ctx, const uint32_t* idx, uint32_t n, const uint8_t* src, uint64_t rb,
                     uint8_t* cache_rows, const uint32_t* first, const uint32_t* off, const uint32_t* list,
                     uint8_t* batch);
bool gather_can_skip_first(uint64_t rb);
// d_out row j <- feature row d_ids[j] from storage, for j in [0, n). Sorts the
// requests by id on `s`, reads page runs on the host into pinned chunks,
// copies them to HBM on the features' copy stream and scatters them to their
// rows on `s`; returns when everything is enqueued (work on `s` after the call
// sees the rows). Returns the host read wall time in ms.
// out2/idx2 (optional): row j also goes to out2 row idx2[j]
double stage_fetch(gx_features* f, const uint32_t* d_ids, uint64_t n, uint8_t* d_out, cudaStream_t s,
                   uint8_t* out2 = nullptr, const uint32_t* idx2 = nullptr);
// Misses of a resolved access list: miss_ids[r] = ids[k] for the r-th k with
// slots[k] == kNever (access order), slots[k] := kStageFlag | r. Returns the
// count (synchronises `s`).
uint64_t stage_misses(gx_ctx* ctx, const uint32_t* ids, uint32_t* slots, uint64_t n, DevBuf<uint32_t>& miss_ids,
                      cudaStream_t s);
// Row-partitioned table (comm.cu): the same contract as stage_fetch, served by
// the owners through one variable all-to-all. Collective (call on every rank,
// also with n == 0).
double part_fetch(gx_features* f, const uint32_t* d_ids, uint64_t n, uint8_t* d_out, cudaStream_t s,
                  uint8_t* out2 = nullptr, const uint32_t* idx2 = nullptr);
// storage tiers that deliver rows through staging (FILE, PARTITIONED)
inline bool staged_backing(const gx_features* f) {
    return f->backing == GX_BACKING_FILE || f->backing == GX_BACKING_PARTITIONED;
}
// d_out row j <- feature row d_ids[j] through the table's staged tier
inline double fetch_rows(gx_features* f, const uint32_t* d_ids, uint64_t n, uint8_t* d_out, cudaStream_t s,
                         uint8_t* out2 = nullptr, const uint32_t* idx2 = nullptr) {
    return f->backing == GX_BACKING_PARTITIONED ? part_fetch(f, d_ids, n, d_out, s, out2, idx2)
                                                : stage_fetch(f, d_ids, n, d_out, s, out2, idx2);
}
// feature_value rows [node0, node0 + n) (graph.cu), scalar_width 4 or 2
void launch_features(uint8_t* out, uint64_t n, uint32_t dim, uint32_t sw, uint64_t vseed, uint64_t node0,
                     int num_sms, cudaStream_t s);
// k_scatter_rows launcher (storage.cu): out row dst_idx[q] <- src row q
void launch_scatter_rows(const uint8_t* src, const uint32_t* dst_idx, uint64_t cnt, uint8_t* out, uint64_t rb,
                         int num_sms, cudaStream_t s, uint8_t* out2 = nullptr, const uint32_t* idx2 = nullptr);

}  // namespace gx
