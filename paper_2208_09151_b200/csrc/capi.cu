// capi.cu -- context, errors, primitives, changeset/sample accessors, runtime
// file codecs (FORMATS.md "Runtime files") and the fused device pipeline.
#include <algorithm>
#include <cstdio>
#include <fcntl.h>
#include <unistd.h>
#include <unordered_set>

#include "files.cuh"
#include "gx_internal.cuh"

namespace gx {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

static const char kIdsMagic[8] = {'G', 'X', 'I', 'D', 'S', '0', '0', '1'};
static const char kAdjMagic[8] = {'G', 'X', 'A', 'D', 'J', '0', '0', '1'};
static const char kInitMagic[8] = {'G', 'X', 'I', 'N', 'I', 'T', '0', '1'};
static const char kUpdMagic[8] = {'G', 'X', 'U', 'P', 'D', '0', '0', '1'};

static std::string rt_path(const char* dir, const char* stem, uint64_t sb, int64_t i) {
    std::string p = std::string(dir) + "/" + stem + "_" + std::to_string(sb);
    if (i >= 0) p += "_" + std::to_string(i);
    return p + ".bin";
}

static void d2h_u32_as_u64(const uint32_t* d, uint64_t n, uint64_t* h) {
    if (!n) return;
    std::vector<uint32_t> t(n);
    GX_CUDA(cudaMemcpy(t.data(), d, n * 4, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < n; ++i) h[i] = t[i];
}

}  // namespace gx

// ---------------------------------------------------------------------------
// fused pipeline handle: two superbatch slots in flight. The sampler and the
// inspector run on the context stream; the executor of a slot runs on the
// pipeline's own stream, so executor(k) overlaps sampler/inspector(k+1).
// ---------------------------------------------------------------------------
struct PipeSlot {
    bool pending = false;
    uint64_t S = 0;
    gx_changesets cs;
    gx::DevBuf<uint32_t> trace, acc_slot;  // swapped with ctx->is while the inspector runs
    gx::DevBuf<unsigned long long> counters, digests;
    gx::PinBuf<unsigned long long> h_cnt, h_dig;
    std::vector<uint64_t> o;  // trace offsets
    // gathered rows: every iteration's batch at row o[i] (whole superbatch
    // resident: `full`), or one iteration-sized buffer reused per iteration
    gx::DevBuf<uint8_t> batch;
    bool full = false;
    gx::DevBuf<uint32_t> d_off;  // o[] on the device (segment-mode miss charging)
    gx::PinBuf<uint32_t> h_off;
    // one-launch executor: insert offsets per iteration, per-slot last-insert marks (K, kept zeroed)
    gx::DevBuf<uint32_t> d_in_off, last_ins;
    gx::PinBuf<uint32_t> h_in_off32;
    uint64_t last_ins_n = 0;
    uint64_t nseg = 0;     // gather launches (segments of iterations)
    uint64_t ticket = ~0ull;
    uint64_t sampled_edges = 0;
    uint64_t launches = 0;  // this library's kernels launched for the superbatch
    gx_iostats sample_io{};
    // GX_BACKING_FILE: miss ids (access order) and their staged rows
    gx::DevBuf<uint32_t> miss_ids;
    gx::DevBuf<uint8_t> stage;
    double ms_storage = 0;
    uint64_t storage_rows = 0, storage_bytes = 0;
    bool fused = false;
    bool ifan = false;  // changeset regime: init rows fanned out in the switch (launch_init_fan)
    uint64_t last_row = 0;  // not resident: row of the last iteration in the batch window
    gx::DevBuf<uint32_t> ifan_cnt, ifan_off, ifan_list, ifan_rank;
    gx::DevBuf<uint8_t> ifan_tmp;
    uint64_t gather_rows = 0;
    cudaEvent_t ev[6] = {};  // A: start, sampled, inspected; B: exec start, switched, done
    std::vector<cudaEvent_t> kev;
};

struct gx_pipeline {
    gx_graph* g = nullptr;
    gx_features* f = nullptr;
    gx_ctx* ctx = nullptr;
    std::vector<uint32_t> fanouts;
    uint64_t K = 0;
    gx_samples samples;
    gx::DevBuf<uint8_t> cache_rows;
    cudaStream_t exec = nullptr;
    PipeSlot slot[2];
    uint64_t submitted = 0;
    bool digest = false;
    // 0 (default): a superbatch's sampler waits for the previous superbatch's
    // executor -- the GPU runs the stages back to back while the host prepares
    // the next submission; 1: they run concurrently (measured slower at papers
    // shape: the HBM-bound gather stretches the latency-bound sampler/inspector)
    int overlap = 0;
    std::vector<uint64_t> h_digests;
};

using namespace gx;

extern "C" {

const char* gx_last_error(void) { return g_last_error.c_str(); }
const char* gx_version(void) { return "gx_b200 0.1 (sm_100a)"; }

uint64_t gx_mix64(uint64_t z) { return mix64(z); }
uint64_t gx_derive_seed(uint64_t b, uint64_t i) { return derive_seed(b, i); }
uint64_t gx_pages_touched(uint64_t lo, uint64_t hi) { return pages_touched(lo, hi); }
gx_status gx_page_count_for_row(uint64_t w, uint64_t r, uint64_t* pages) {
    return guard([&] {
        if (w == 0) fail(GX_INVALID_ARGUMENT, "page_count_for_row: row_bytes must be > 0");
        *pages = pages_touched(r * w, r * w + w);
    });
}

gx_status gx_derive_train_ids(uint64_t n, uint64_t seed, double frac, uint64_t* out, uint64_t* n_out) {
    return guard([&] {
        if (frac <= 0.0 || frac > 1.0) fail(GX_INVALID_ARGUMENT, "train_fraction must be in (0, 1]");
        uint64_t want = (uint64_t)((double)n * frac);
        want = std::min(std::max<uint64_t>(want, 1), n);
        for (uint64_t v = 0; v < n; ++v) out[v] = v;
        uint64_t st = derive_seed(mix64(seed) ^ 0x545241494EULL, 0);
        for (uint64_t i = 0; i < want; ++i) {
            st += kGamma;
            uint64_t z = st;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            z ^= z >> 31;
            const uint64_t j = i + (uint64_t)(((unsigned __int128)z * (n - i)) >> 64);
            std::swap(out[i], out[j]);
        }
        std::sort(out, out + want);
        *n_out = want;
    });
}

gx_status gx_plan_seed_batches(const uint64_t* train, uint64_t n, uint64_t batch_size, uint64_t epoch_seed,
                               uint64_t* sh) {
    return guard([&] {
        if (n == 0) fail(GX_INVALID_ARGUMENT, "training set is empty");
        if (batch_size < 1) fail(GX_INVALID_ARGUMENT, "batch_size must be >= 1");
        std::copy(train, train + n, sh);
        uint64_t st = epoch_seed;
        for (uint64_t i = n - 1; i > 0; --i) {
            st += kGamma;
            uint64_t z = st;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            z ^= z >> 31;
            const uint64_t j = (uint64_t)(((unsigned __int128)z * (i + 1)) >> 64);
            std::swap(sh[i], sh[j]);
        }
    });
}

uint64_t gx_epoch_seed(uint64_t seed, uint64_t epoch) { return derive_seed(mix64(seed) ^ 0x45504F4348ULL, epoch); }

gx_status gx_ctx_create(int device, gx_ctx** out) {
    return guard([&] {
        int n = 0;
        GX_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(GX_INVALID_ARGUMENT, "no such CUDA device");
        GX_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        GX_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            fail(GX_CUDA_ERROR, std::string("gx_b200 is built for sm_100a; found ") + prop.name);
        auto c = new gx_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        try {
            GX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->barrier.alloc(1);
            GX_CUDA(cudaMemset(c->barrier.p, 0, sizeof(GridBarrier)));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void gx_ctx_destroy(gx_ctx* c) {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    cudaStream_t s = c->stream;
    delete c;
    if (s) cudaStreamDestroy(s);
}
gx_status gx_ctx_synchronize(gx_ctx* c) {
    return guard([&] { GX_CUDA(cudaStreamSynchronize(c->stream)); });
}
void* gx_ctx_stream(gx_ctx* c) { return c ? (void*)c->stream : nullptr; }

// ---- inspector API ---------------------------------------------------------

static std::vector<uint64_t> offsets_vec(const uint64_t* off, uint64_t S) {
    std::vector<uint64_t> o(off, off + S + 1);
    for (uint64_t i = 0; i < S; ++i)
        if (o[i + 1] < o[i]) fail(GX_INVALID_ARGUMENT, "trace offsets must be non-decreasing");
    if (o[0] != 0) {
        const uint64_t b = o[0];
        for (auto& x : o) x -= b;
    }
    return o;
}

gx_status gx_precompute_trace(gx_ctx* ctx, const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N,
                              uint64_t K, gx_changesets** out) {
    return guard([&] {
        auto o = offsets_vec(off, S);
        inspect_fill_from_host(ctx, flat + off[0], o, N);
        auto cs = new gx_changesets();
        try {
            inspect_run(ctx, o, N, K, nullptr, -1, cs, false);
        } catch (...) {
            delete cs;
            throw;
        }
        *out = cs;
    });
}

gx_status gx_simulate_trace(gx_ctx* ctx, const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N,
                            uint64_t K, const uint64_t* init, uint64_t n_init, gx_changesets** out) {
    return guard([&] {
        auto o = offsets_vec(off, S);
        inspect_fill_from_host(ctx, flat + off[0], o, N);
        // build_access_index's checks happen first (duplicates), via the device run
        // below; init checks in simulate_changesets order (changeset.hpp:238-246)
        {
            std::unordered_set<uint64_t> in_trace;
            std::unordered_set<uint64_t> want(init, init + n_init);
            for (uint64_t x = 0; x < o[S]; ++x)
                if (want.count(flat[off[0] + x])) in_trace.insert(flat[off[0] + x]);
            std::unordered_set<uint64_t> seen;
            for (uint64_t k = 0; k < n_init; ++k) {
                if (init[k] >= N) fail(GX_OUT_OF_RANGE, "init id out of range");
                if (!in_trace.count(init[k]))
                    fail(GX_LOGIC_ERROR, "init id never appears in the trace (index/trace mismatch)");
                if (!seen.insert(init[k]).second) fail(GX_LOGIC_ERROR, "duplicate id in init set");
            }
            if (n_init > K) fail(GX_INVALID_ARGUMENT, "init set exceeds capacity");
        }
        auto cs = new gx_changesets();
        try {
            inspect_run(ctx, o, N, K, init, (int64_t)n_init, cs, false);
        } catch (...) {
            delete cs;
            throw;
        }
        *out = cs;
    });
}

gx_status gx_precompute_samples(const gx_samples* s, uint64_t N, uint64_t K, gx_changesets** out) {
    return guard([&] {
        std::vector<uint64_t> o(s->S + 1, 0);
        for (uint64_t i = 0; i < s->S; ++i) o[i + 1] = o[i] + s->h_n_ids[i];
        inspect_fill_from_device(s->ctx, s->ids.p, s->cap_ids, o);
        auto cs = new gx_changesets();
        try {
            inspect_run(s->ctx, o, N, K, nullptr, -1, cs, true);
        } catch (...) {
            delete cs;
            throw;
        }
        *out = cs;
    });
}

gx_status gx_access_index(gx_ctx* ctx, const uint64_t* flat, const uint64_t* off, uint64_t S, uint64_t N,
                          uint64_t* iters, uint64_t* ptr) {
    return guard([&] {
        auto o = offsets_vec(off, S);
        inspect_fill_from_host(ctx, flat + off[0], o, N);
        access_index_run(ctx, o, N, iters, ptr);
    });
}

void gx_changesets_destroy(gx_changesets* cs) { delete cs; }
uint64_t gx_changesets_num_iters(const gx_changesets* cs) { return cs ? cs->S : 0; }
uint64_t gx_changesets_init_size(const gx_changesets* cs) { return cs ? cs->n_init : 0; }

gx_status gx_changesets_init(const gx_changesets* cs, uint64_t* out, uint64_t* n) {
    return guard([&] {
        if (n) *n = cs->n_init;
        if (out) d2h_u32_as_u64(cs->init.p, cs->n_init, out);
    });
}

gx_status gx_changesets_iter_info(const gx_changesets* cs, uint64_t i, uint64_t* n_in, uint64_t* n_out,
                                  uint64_t* misses) {
    return guard([&] {
        if (i >= cs->S) fail(GX_OUT_OF_RANGE, "iteration index out of range");
        if (n_in) *n_in = cs->h_in_off[i + 1] - cs->h_in_off[i];
        if (n_out) *n_out = cs->h_out_off[i + 1] - cs->h_out_off[i];
        if (misses) *misses = cs->h_misses[i];
    });
}

gx_status gx_changesets_copy_iter(const gx_changesets* cs, uint64_t i, uint64_t* in_ids, uint64_t* out_ids,
                                  uint64_t* in_pos) {
    return guard([&] {
        if (i >= cs->S) fail(GX_OUT_OF_RANGE, "iteration index out of range");
        const uint64_t a = cs->h_in_off[i], ni = cs->h_in_off[i + 1] - a;
        const uint64_t b = cs->h_out_off[i], no = cs->h_out_off[i + 1] - b;
        if (in_ids) d2h_u32_as_u64(cs->in_ids.p + a, ni, in_ids);
        if (in_pos) d2h_u32_as_u64(cs->in_pos.p + a, ni, in_pos);
        if (out_ids) d2h_u32_as_u64(cs->out_ids.p + b, no, out_ids);
    });
}

gx_status gx_changesets_misses(const gx_changesets* cs, uint64_t* misses) {
    return guard([&] {
        for (uint64_t i = 0; i < cs->S; ++i) misses[i] = cs->h_misses[i];
    });
}

// init_{sb}.bin + update_{sb}_{i}.bin (changeset.hpp:409-454): the byte images
// of all S + 1 files are packed on the device and written asynchronously
// (files.cu: side-stream D2H into pinned chunks, host writer threads)
gx_status gx_changesets_write_files(const gx_changesets* cs, const char* dir, uint64_t sb) {
    return guard([&] {
        FileImage im;
        im.add_file(rt_path(dir, "init", sb, -1));
        im.header(kInitMagic, 8);
        im.value<uint64_t>(cs->n_init);
        im.widen(cs->init.p, cs->n_init);
        for (uint64_t i = 0; i < cs->S; ++i) {
            const uint64_t a = cs->h_in_off[i], ni = cs->h_in_off[i + 1] - a;
            const uint64_t b = cs->h_out_off[i], no = cs->h_out_off[i + 1] - b;
            im.add_file(rt_path(dir, "update", sb, (int64_t)i));
            im.header(kUpdMagic, 8);
            im.value<uint64_t>(ni);
            im.widen(cs->in_ids.p + a, ni);
            im.value<uint64_t>(no);
            im.widen(cs->out_ids.p + b, no);
            im.value<uint64_t>(ni);
            im.widen(cs->in_pos.p + a, ni);
        }
        write_file_image(cs->ctx, im);
    });
}

// ids_{sb}_{i}.bin + adj_{sb}_{i}.bin (sampler.hpp:123-182), written like the
// changeset files (files.cu)
gx_status gx_samples_write_files(const gx_samples* s, const char* dir, uint64_t sb) {
    return guard([&] {
        FileImage im;
        for (uint64_t b = 0; b < s->S; ++b) {
            const uint64_t n = s->h_n_ids[b];
            im.add_file(rt_path(dir, "ids", sb, (int64_t)b));
            im.header(kIdsMagic, 8);
            im.value<uint64_t>(n);
            im.widen(s->ids.p + b * s->cap_ids, n);
            im.add_file(rt_path(dir, "adj", sb, (int64_t)b));
            im.header(kAdjMagic, 8);
            im.value<uint32_t>(s->L);
            for (uint32_t l = 0; l < s->L; ++l) {
                const uint64_t c = s->h_layer_count[b * s->L + l];
                im.value<uint64_t>(c);
                im.copy8(s->edges.p + b * s->cap_e_batch + s->e_off[l], c);
            }
        }
        write_file_image(s->ctx, im);
    });
}

// ---- fused pipeline ---------------------------------------------------------

gx_status gx_pipeline_create(gx_graph* g, gx_features* f, const uint32_t* fanouts, uint32_t L, uint64_t K,
                             gx_pipeline** out) {
    return guard([&] {
        if (!g || !f) fail(GX_INVALID_ARGUMENT, "null handle");
        if (f->n != g->n) fail(GX_INVALID_ARGUMENT, "graph and feature files disagree on node count");
        if (!f->ctx) fail(GX_INVALID_ARGUMENT, "feature table was opened without a context");
        if (K >= 0x7FFFFFFFull) fail(GX_INVALID_ARGUMENT, "cache capacity exceeds 2^31 - 1 slots");
        auto p = new gx_pipeline();
        try {
            p->g = g;
            p->f = f;
            p->ctx = g->ctx;
            p->fanouts.assign(fanouts, fanouts + L);
            p->K = K;
            p->cache_rows.alloc(std::max<uint64_t>(K * f->row_bytes, 16));
            GX_CUDA(cudaStreamCreateWithFlags(&p->exec, cudaStreamNonBlocking));
            for (auto& sl : p->slot)
                for (auto& e : sl.ev) GX_CUDA(cudaEventCreate(&e));
        } catch (...) {
            gx_pipeline_destroy(p);
            throw;
        }
        *out = p;
    });
}

void gx_pipeline_destroy(gx_pipeline* p) {
    if (!p) return;
    if (p->exec) cudaStreamSynchronize(p->exec);
    if (p->ctx) cudaStreamSynchronize(p->ctx->stream);
    for (auto& sl : p->slot) {
        for (auto& e : sl.ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : sl.kev) cudaEventDestroy(e);
    }
    if (p->exec) cudaStreamDestroy(p->exec);
    delete p;
}

gx_status gx_pipeline_set_overlap(gx_pipeline* p, int concurrent) {
    return guard([&] {
        if (!p) fail(GX_INVALID_ARGUMENT, "null pipeline");
        p->overlap = concurrent != 0;
    });
}

gx_status gx_pipeline_set_digest(gx_pipeline* p, int enable) {
    return guard([&] { p->digest = enable != 0; });
}

gx_status gx_pipeline_digests(const gx_pipeline* p, uint64_t* d) {
    return guard([&] {
        for (size_t i = 0; i < p->h_digests.size(); ++i) d[i] = p->h_digests[i];
    });
}

gx_status gx_pipeline_cache_rows(gx_pipeline* p, void* host_out) {
    return guard([&] {
        if (!p) fail(GX_INVALID_ARGUMENT, "null pipeline");
        for (const auto& sl : p->slot)
            if (sl.pending) fail(GX_LOGIC_ERROR, "cache rows are readable when no superbatch is in flight");
        const uint64_t n = p->K * p->f->row_bytes;
        if (n) GX_CUDA(cudaMemcpy(host_out, p->cache_rows.p, n, cudaMemcpyDeviceToHost));
    });
}

void* gx_pipeline_exec_stream(gx_pipeline* p) { return p ? (void*)p->exec : nullptr; }

gx_status gx_pipeline_submit(gx_pipeline* p, const uint64_t* seeds_flat, const uint64_t* batch_off, uint64_t S,
                             uint64_t global_seed, uint64_t first_global_batch, uint64_t* ticket) {
    return guard([&] {
        gx_ctx* ctx = p->ctx;
        cudaStream_t A = ctx->stream, B = p->exec;
        const uint64_t N = p->g->n;
        if (S == 0) fail(GX_INVALID_ARGUMENT, "empty superbatch");
        for (uint64_t b = 0; b < S; ++b) {
            const uint64_t n = batch_off[b + 1] - batch_off[b];
            if (n == 0) fail(GX_RUNTIME_ERROR, "superbatch sample failed: sample_batch: seeds are empty");
            for (uint64_t k = batch_off[b]; k < batch_off[b + 1]; ++k)
                if (seeds_flat[k] >= N) fail(GX_RUNTIME_ERROR, "superbatch sample failed: seed node out of range");
        }
        const uint64_t t = p->submitted;
        PipeSlot& sl = p->slot[t & 1];
        if (sl.pending) fail(GX_LOGIC_ERROR, "two superbatches already in flight: wait for the older one first");
        const uint64_t launches0 = gx::g_kernel_launches.load(std::memory_order_relaxed);
        std::vector<uint64_t> bs(S);
        for (uint64_t i = 0; i < S; ++i) bs[i] = derive_seed(global_seed, first_global_batch + i);
        const uint32_t L = (uint32_t)p->fanouts.size();
        // this slot's buffers were last read by its previous executor (already waited)
        const PipeSlot& prev = p->slot[(t + 1) & 1];
        if (!p->overlap && prev.pending) GX_CUDA(cudaStreamWaitEvent(A, prev.ev[5], 0));
        GX_CUDA(cudaEventRecord(sl.ev[0], A));
        // (1) sample
        // the sampler also records every id's first use for the inspector
        static const bool fx_pre = gx::env_int("GX_SAMPLER_FIRSTUSE", 0) != 0;  // measured a wash: sampler +0.23 ms, inspector -0.25 ms
        const uint32_t fx_epoch = fx_pre && S <= 2048 ? inspect_reserve_epoch(ctx, N, S << 21) : 0;
        const bool presampled = sample_run(p->g, seeds_flat, batch_off, S, p->fanouts.data(), L, bs.data(),
                                           &p->samples, fx_epoch ? ctx->is.firstx.p : nullptr, fx_epoch);
        GX_CUDA(cudaEventRecord(sl.ev[1], A));
        samples_sync_host(&p->samples);  // host needs |ids_i| (stream A only)
        // duplicate seeds are found by the sampler's layer-0 table build; the
        // reference's sample_batch throws and superbatch_sample rethrows it as
        // runtime_error (sampler.hpp:83, 236). Nothing downstream ran yet.
        if (p->samples.dup_seed) fail(GX_RUNTIME_ERROR, "superbatch sample failed: duplicate seed in batch");
        sl.sampled_edges = gx_samples_total_edges(&p->samples);
        sl.sample_io = p->samples.io;
        sl.S = S;
        // (2) inspect into this slot's trace / acc_slot / changesets
        sl.o.assign(S + 1, 0);
        for (uint64_t i = 0; i < S; ++i) sl.o[i + 1] = sl.o[i] + p->samples.h_n_ids[i];
        std::swap(ctx->is.trace, sl.trace);
        std::swap(ctx->is.acc_slot, sl.acc_slot);
        // all-fit superbatches fuse the cache fill with the first uses when the
        // whole superbatch is resident in HBM and the backing table is too
        const uint64_t rb = p->f->row_bytes;
        // the whole superbatch's rows stay in HBM when they fit: GX_BATCH_BUDGET_MB
        // caps a slot explicitly; by default whatever the device has free (the
        // slot's current buffer included) minus a margin for the inspector's
        // trace-sized scratch (S = 500 at papers shape: 46 GB per slot)
        const uint64_t need = sl.o[S] * rb;
        static const int budget_mb = gx::env_int("GX_BATCH_BUDGET_MB", -1);
        bool resident;
        if (budget_mb >= 0) {
            resident = need <= ((uint64_t)budget_mb << 20);
        } else if (need <= sl.batch.n) {
            resident = true;
        } else {
            size_t fr = 0, total = 0;
            GX_CUDA(cudaMemGetInfo(&fr, &total));
            // (the deferred recurrence keeps ~12 A-sized u32 arrays: trace,
            // next use, acc_slot, raw/sorted out lists, in lists, ...; the init
            // fan-out two more: per-access ranks and the slot lists)
            const uint64_t margin = (4ull << 30) + 56ull * sl.o[S];
            // (what the grow-only buffer would actually allocate, headroom included)
            resident = (uint64_t)sl.batch.reserved_after(need) + margin <= (uint64_t)fr + sl.batch.n;
        }
        // fan-out form (default): each init row read once, written to its slot
        // and every batch row of its node; GX_FANOUT=0: fill + first use, then
        // a gather of the other accesses from the cache
        static const bool fan = gx::env_int("GX_FANOUT", 1) != 0;
        const bool src_ok = staged_backing(p->f) || p->f->rows_dev_view;
        const int mark = !resident || !src_ok ? 0 : fan && rb % 16 == 0 ? 2 : gather_can_skip_first(rb) ? 1 : 0;
        try {
            inspect_fill_from_device(ctx, p->samples.ids.p, p->samples.cap_ids, sl.o);
            inspect_run(ctx, sl.o, N, p->K, nullptr, -1, &sl.cs, true, mark, presampled ? fx_epoch : 0);
        } catch (...) {
            std::swap(ctx->is.trace, sl.trace);
            std::swap(ctx->is.acc_slot, sl.acc_slot);
            throw;
        }
        std::swap(ctx->is.trace, sl.trace);
        std::swap(ctx->is.acc_slot, sl.acc_slot);
        // storage tier: the accesses the cache will miss read staged rows
        const bool file = staged_backing(p->f);
        // (an all-fit superbatch has no misses, and with the fused executor its
        // acc_slot only holds the first uses -- nothing to stage)
        const uint64_t n_miss =
            file && !sl.cs.first_marked ? stage_misses(ctx, sl.trace.p, sl.acc_slot.p, sl.o[S], sl.miss_ids, A) : 0;
        GX_CUDA(cudaEventRecord(sl.ev[2], A));
        // (3)+(4) executor on stream B, after the inspector and the previous executor
        GX_CUDA(cudaStreamWaitEvent(B, sl.ev[2], 0));
        GX_CUDA(cudaEventRecord(sl.ev[3], B));
        uint64_t maxw = 0;
        for (uint64_t i = 0; i < S; ++i) maxw = std::max(maxw, sl.o[i + 1] - sl.o[i]);
        // whole superbatch resident when it fits the per-slot budget (GX_BATCH_BUDGET_MB)
        sl.full = resident;
        const bool fused = sl.cs.first_marked;  // implies all-fit (no changesets) and resident
        sl.fused = fused;
        sl.gather_rows = fused ? (sl.cs.fan ? (file ? sl.cs.n_rest : 0) : sl.cs.n_rest) : sl.o[S];
        // not resident: a window of up to GX_BATCH_WINDOW iterations' rows, so a
        // run of iterations without changesets is still one gather launch
        // (S = 500 all-fit at 35-50 % cache: 500 launches of ~30 us -> 32)
        static const uint64_t win_iters = (uint64_t)std::max(1, gx::env_int("GX_BATCH_WINDOW", 16));
        const uint64_t win_rows = sl.full ? sl.o[S] : std::max(maxw, std::min(sl.o[S], win_iters * maxw));
        sl.batch.reserve(std::max<uint64_t>(win_rows * rb, 16));
        sl.h_off.reserve(S + 1);
        sl.d_off.reserve(S + 1);
        for (uint64_t i = 0; i <= S; ++i) sl.h_off.p[i] = (uint32_t)sl.o[i];
        GX_CUDA(cudaMemcpyAsync(sl.d_off.p, sl.h_off.p, (S + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, B));
        sl.counters.reserve(8 * (S + 2));  // S iterations, the cache init, a scratch block
        sl.h_cnt.reserve(8 * (S + 1));
        GX_CUDA(cudaMemsetAsync(sl.counters.p, 0, 8 * (S + 2) * 8, B));
        if (p->digest) {
            sl.digests.reserve(S);
            sl.h_dig.reserve(S);
            GX_CUDA(cudaMemsetAsync(sl.digests.p, 0, S * 8, B));
        }
        while (sl.kev.size() < 3 * S) {
            cudaEvent_t e;
            GX_CUDA(cudaEventCreate(&e));
            sl.kev.push_back(e);
        }
        // device-backed table, whole superbatch resident, changesets: the
        // gathers of all S iterations are ONE launch (see (4)), and when the
        // init rows serve most accesses (few inserts against the init set:
        // papers @5 %, 25K inserts for 5.55M init slots) the switch fans each
        // init row out to the accesses it serves and k_gather_rest copies the
        // rest; with many inserts (cfg1: 540K for 100K slots) most rows would
        // go through the rest copy, and k_gather_sb serves every access.
        // GX_INIT_FAN: 0 off, 1 by that rule (default), 2 always.
        static const bool one_gather = gx::env_int("GX_ONE_GATHER", 1) != 0;
        static const int init_fan = gx::env_int("GX_INIT_FAN", 1);
        const bool single = !fused && !file && sl.full && one_gather && p->f->rows_dev_view != nullptr;
        sl.ifan = single && rb % 16 == 0 && sl.cs.n_init > 0 &&
                  (init_fan == 2 || (init_fan == 1 && 4 * sl.cs.h_in_off[S] <= sl.cs.n_init));
        ctx->launch_stream = B;
        try {
            // (3) switch: the init rows into slots 0..n_init-1 (the inspector
            // resolved every access's serving slot, so no address table here)
            const uint8_t* store = p->f->rows_dev_view;
            sl.ms_storage = 0;
            sl.storage_rows = sl.storage_bytes = 0;
            if (file) {
                // the init rows land in their slots, the misses in this slot's
                // staging rows, both read from storage while B drains
                // (partitioned tables: two all-to-alls with the other ranks)
                const bool f_file = p->f->file != nullptr;
                const uint64_t r0 = f_file ? p->f->file->rows.load() : p->f->xstats.rows_requested;
                const uint64_t b0 = f_file ? p->f->file->bytes.load() : p->f->xstats.bytes_sent;
                sl.cs.init.reserve(1);
                sl.miss_ids.reserve(1);
                // all-fit (fused): each init row also lands in its first batch row
                // (fan-out form: the cache rows then fan out to the other accesses)
                const bool dual = fused;
                sl.ms_storage += fetch_rows(p->f, sl.cs.init.p, sl.cs.n_init, p->cache_rows.p, B,
                                            dual ? sl.batch.p : nullptr, dual ? sl.cs.first_acc.p : nullptr);
                GX_CUDA(cudaEventRecord(sl.ev[4], B));
                sl.stage.reserve(std::max<uint64_t>(n_miss * rb, 16));
                sl.ms_storage += fetch_rows(p->f, sl.miss_ids.p, n_miss, sl.stage.p, B);
                store = sl.stage.p;
                sl.storage_rows = (f_file ? p->f->file->rows.load() : p->f->xstats.rows_requested) - r0;
                sl.storage_bytes = (f_file ? p->f->file->bytes.load() : p->f->xstats.bytes_sent) - b0;
            } else if (fused && sl.cs.fan) {
                // the switch fused with every access: one read of each backing
                // row, written to its slot and to all batch rows of its node
                launch_fan_rows(ctx, sl.cs.init.p, (uint32_t)sl.cs.n_init, p->f->rows_dev_view, rb, p->cache_rows.p,
                                sl.cs.first_acc.p, sl.cs.fan_off.p, sl.cs.fan_list.p, sl.batch.p);
                GX_CUDA(cudaEventRecord(sl.ev[4], B));
            } else if (fused) {
                // the switch fused with every init node's first use: one read of
                // the backing row, written to its slot and to its first batch row
                launch_fill_first(ctx, sl.cs.init.p, sl.cs.first_acc.p, (uint32_t)sl.cs.n_init, p->f->rows_dev_view,
                                  rb, p->cache_rows.p, sl.batch.p);
                GX_CUDA(cudaEventRecord(sl.ev[4], B));
            } else if (sl.ifan) {
                launch_init_fan(ctx, sl.trace.p, sl.acc_slot.p, sl.o[S], sl.cs.init.p, (uint32_t)sl.cs.n_init,
                                p->f->rows_dev_view, rb, p->cache_rows.p, sl.batch.p, sl.ifan_cnt, sl.ifan_off,
                                sl.ifan_list, sl.ifan_rank, sl.ifan_tmp);
                GX_CUDA(cudaEventRecord(sl.ev[4], B));
            } else {
                launch_cache_init(ctx, sl.cs.init.p, (uint32_t)sl.cs.n_init, nullptr, p->f, p->cache_rows.p,
                                  sl.counters.p + 8 * S);
                GX_CUDA(cudaEventRecord(sl.ev[4], B));
            }
            // (4) main loop. Iterations whose changesets are empty do not mutate
            // the cache, so with the whole superbatch resident a run of them is
            // gathered by one launch (segment), then the last one's changeset applied.
            auto empty_cs = [&](uint64_t i) {
                return sl.cs.h_in_off[i + 1] == sl.cs.h_in_off[i] && sl.cs.h_out_off[i + 1] == sl.cs.h_out_off[i];
            };
            uint64_t seg0 = 0;  // first iteration of the current segment (the window's row 0 when not resident)
            auto rows_of = [&](uint64_t i) { return sl.batch.p + (sl.full ? sl.o[i] : sl.o[i] - sl.o[seg0]) * rb; };
            uint64_t nseg = 0;
            // device-backed table, whole superbatch resident, changesets: the
            // gathers of all S iterations are ONE bulk-copy launch (k_gather_sb).
            // The cache keeps its init rows during the launch (the changesets
            // are applied after it, in iteration order, so the cache ends in the
            // reference's state): a hit whose slot still holds its init node
            // reads the cache, every other access the same bytes from the
            // HBM-resident table (a slot is a copy of the table row,
            // feature_cache.hpp:115-126), so iteration i's hits no longer wait
            // for the applies of iterations < i. The per-iteration miss / page
            // counters come from the inspector's resolved slots.
            // GX_ONE_GATHER=0: per-segment gathers + applies.
            if (single) {
                GX_CUDA(cudaEventRecord(sl.kev[0], B));
                if (sl.ifan)  // the init-served accesses were written by the switch
                    launch_gather_rest(ctx, sl.trace.p, sl.ifan_rank.p, sl.o[S], p->f->rows_dev_view, rb, sl.batch.p,
                                       sl.counters.p + 8 * S + 5);
                else if (!launch_gather_superbatch(ctx, sl.trace.p, sl.acc_slot.p, sl.o[S], sl.cs.init.p,
                                                   (uint32_t)sl.cs.n_init, p->cache_rows.p, p->f->rows_dev_view, rb,
                                                   sl.batch.p))
                    launch_gather_resolved(ctx, sl.trace.p, nullptr, sl.o[S], nullptr, p->f->rows_dev_view, rb,
                                           sl.batch.p, sl.counters.p + 8 * (S + 1), nullptr, 0, false, false);
                launch_count_iter_misses(ctx, sl.trace.p, sl.acc_slot.p, sl.d_off.p, (uint32_t)S, maxw, rb,
                                         sl.counters.p);
                GX_CUDA(cudaEventRecord(sl.kev[1], B));
                if (p->digest)
                    for (uint64_t k = 0; k < S; ++k)
                        launch_digest(ctx, rows_of(k), sl.o[k + 1] - sl.o[k], rb, sl.digests.p + k);
                // all changesets at once: each slot takes its last insert's row
                const uint64_t n_in = sl.cs.h_in_off[S];
                if (n_in) {
                    sl.d_in_off.reserve(S + 1);
                    sl.h_in_off32.reserve(S + 1);
                    for (uint64_t i = 0; i <= S; ++i) sl.h_in_off32.p[i] = (uint32_t)sl.cs.h_in_off[i];
                    GX_CUDA(cudaMemcpyAsync(sl.d_in_off.p, sl.h_in_off32.p, (S + 1) * 4, cudaMemcpyHostToDevice, B));
                    if (sl.last_ins_n < p->K + 1) {
                        sl.last_ins.alloc(p->K + 1);
                        GX_CUDA(cudaMemsetAsync(sl.last_ins.p, 0, (p->K + 1) * 4, B));
                        sl.last_ins_n = p->K + 1;
                    }
                    launch_apply_all(ctx, sl.cs.in_pos.p, sl.cs.in_slot.p, sl.d_in_off.p, (uint32_t)S, (uint32_t)n_in,
                                     sl.d_off.p, sl.last_ins.p, sl.batch.p, p->cache_rows.p, rb);
                }
                GX_CUDA(cudaEventRecord(sl.kev[2], B));
            }
            if (fused) {  // one launch: every access that is not a first use
                GX_CUDA(cudaEventRecord(sl.kev[0], B));
                if (sl.cs.fan) {
                    // staged tiers: the filled cache rows fan out to the batch
                    // rows (device-backed tables did this in the switch)
                    if (file)
                        launch_fan_rows(ctx, nullptr, (uint32_t)sl.cs.n_init, p->cache_rows.p, rb, nullptr, nullptr,
                                        sl.cs.fan_off.p, sl.cs.fan_list.p, sl.batch.p);
                } else {
                    launch_gather_resolved(ctx, sl.cs.rest_x.p, sl.cs.rest_slot.p, sl.cs.n_rest, p->cache_rows.p,
                                           store, rb, sl.batch.p, sl.counters.p + 8 * S, nullptr, 0, false, true);
                }
                GX_CUDA(cudaEventRecord(sl.kev[1], B));
                if (p->digest)
                    for (uint64_t k = 0; k < S; ++k)
                        launch_digest(ctx, rows_of(k), sl.o[k + 1] - sl.o[k], rb, sl.digests.p + k);
                GX_CUDA(cudaEventRecord(sl.kev[2], B));
            }
            for (uint64_t i = fused || single ? S : 0; i < S;) {
                uint64_t e = i;  // segment [i, e]
                if (sl.full)
                    while (e + 1 < S && empty_cs(e)) ++e;
                else
                    while (e + 1 < S && empty_cs(e) && sl.o[e + 2] - sl.o[i] <= win_rows) ++e;
                seg0 = i;
                if (e + 1 == S) sl.last_row = sl.full ? sl.o[S - 1] : sl.o[S - 1] - sl.o[i];
                GX_CUDA(cudaEventRecord(sl.kev[3 * nseg], B));
                // a one-iteration segment charges its misses through the kernel's
                // per-warp counters (the iteration's counter block has the same
                // layout); per-miss atomics on one iteration's two counters
                // serialise at L2 (cfg1: 3.4 -> 2.1 ms of gather per superbatch)
                const bool one = e == i;
                launch_gather_resolved(ctx, sl.trace.p + sl.o[i], sl.acc_slot.p + sl.o[i], sl.o[e + 1] - sl.o[i],
                                       p->cache_rows.p, store, rb, rows_of(i), sl.counters.p + 8 * i,
                                       one ? nullptr : sl.d_off.p + i, one ? 0u : (uint32_t)(e - i + 1),
                                       file && n_miss > 0, false);
                GX_CUDA(cudaEventRecord(sl.kev[3 * nseg + 1], B));
                if (p->digest)
                    for (uint64_t k = i; k <= e; ++k)
                        launch_digest(ctx, rows_of(k), sl.o[k + 1] - sl.o[k], rb, sl.digests.p + k);
                if (!empty_cs(e)) {
                    const uint64_t a = sl.cs.h_in_off[e], b = sl.cs.h_out_off[e];
                    launch_apply_slots(ctx, sl.cs.in_ids.p + a, sl.cs.in_pos.p + a, sl.cs.in_slot.p + a,
                                       (uint32_t)(sl.cs.h_in_off[e + 1] - a), sl.cs.out_ids.p + b,
                                       (uint32_t)(sl.cs.h_out_off[e + 1] - b), nullptr, rows_of(e),
                                       p->cache_rows.p, rb);
                }
                GX_CUDA(cudaEventRecord(sl.kev[3 * nseg + 2], B));
                ++nseg;
                i = e + 1;
            }
            sl.nseg = fused || single ? 1 : nseg;
        } catch (...) {
            ctx->launch_stream = nullptr;
            throw;
        }
        ctx->launch_stream = nullptr;
        GX_CUDA(cudaMemcpyAsync(sl.h_cnt.p, sl.counters.p, 8 * (S + 1) * 8, cudaMemcpyDeviceToHost, B));
        if (p->digest) GX_CUDA(cudaMemcpyAsync(sl.h_dig.p, sl.digests.p, S * 8, cudaMemcpyDeviceToHost, B));
        GX_CUDA(cudaEventRecord(sl.ev[5], B));
        sl.launches = gx::g_kernel_launches.load(std::memory_order_relaxed) - launches0;
        // the next submit reuses the context stream's scratch: it may start as
        // soon as the inspector is done; slot reuse is guarded by `pending`
        sl.pending = true;
        sl.ticket = t;
        *ticket = t;
        p->submitted = t + 1;
    });
}

gx_status gx_pipeline_wait(gx_pipeline* p, uint64_t ticket, uint64_t* misses_per_iter, gx_pipeline_stats* stats) {
    return guard([&] {
        PipeSlot& sl = p->slot[ticket & 1];
        if (!sl.pending || ticket + 2 < p->submitted || ticket >= p->submitted)
            fail(GX_INVALID_ARGUMENT, "unknown or already completed pipeline ticket");
        GX_CUDA(cudaEventSynchronize(sl.ev[5]));
        sl.pending = false;
        const uint64_t S = sl.S;
        const unsigned long long* cnt = sl.h_cnt.p;
        uint64_t tm = 0, pm = 0;
        gx_iostats gio{};
        // per iteration (segment-mode gathers): [1] misses, [2] pages; a miss
        // reads one row of row_bytes (feature_cache.hpp:66-71)
        for (uint64_t i = 0; i < S; ++i) {
            if (misses_per_iter) misses_per_iter[i] = cnt[8 * i + 1];
            tm += cnt[8 * i + 1];
            pm += sl.cs.h_misses[i];
            gio.pages_read += cnt[8 * i + 2];
            gio.rows_read += cnt[8 * i + 1];
            gio.bytes_read += cnt[8 * i + 1] * p->f->row_bytes;
        }
        if (p->digest) p->h_digests.assign(sl.h_dig.p, sl.h_dig.p + S);
        if (stats) {
            float ms[5];
            GX_CUDA(cudaEventElapsedTime(&ms[0], sl.ev[0], sl.ev[1]));  // sample
            GX_CUDA(cudaEventElapsedTime(&ms[1], sl.ev[1], sl.ev[2]));  // inspect
            GX_CUDA(cudaEventElapsedTime(&ms[2], sl.ev[3], sl.ev[4]));  // switch (executor stream)
            GX_CUDA(cudaEventElapsedTime(&ms[3], sl.ev[4], sl.ev[5]));  // gather + apply
            stats->sampled_edges = sl.sampled_edges;
            stats->gathered_rows = sl.o[S];
            stats->total_misses = tm;
            stats->predicted_misses = pm;
            stats->init_size = sl.cs.n_init;
            stats->total_in = sl.cs.h_in_off[S];
            stats->total_out = sl.cs.h_out_off[S];
            stats->sample_io = sl.sample_io;
            stats->gather_io = gio;
            stats->ms_sample = ms[0];
            stats->ms_inspect = ms[1];
            stats->ms_switch = ms[2];
            stats->ms_gather = ms[3];
            double gk = 0, ak = 0;
            for (uint64_t i = 0; i < sl.nseg; ++i) {
                float a = 0, b = 0;
                GX_CUDA(cudaEventElapsedTime(&a, sl.kev[3 * i], sl.kev[3 * i + 1]));
                GX_CUDA(cudaEventElapsedTime(&b, sl.kev[3 * i + 1], sl.kev[3 * i + 2]));
                gk += a;
                ak += b;
            }
            stats->ms_gather_kernels = gk;
            stats->ms_apply_kernels = ak;
            stats->kernel_launches = sl.launches;
            stats->gather_launches = sl.nseg;
            stats->fill_rows = sl.cs.n_init;
            // init fan-out: the gather copies only the accesses the init rows
            // do not serve (counted by k_gather_rest in the unused init block)
            stats->gather_kernel_rows = sl.ifan ? cnt[8 * S + 5] : sl.gather_rows;
            stats->fused_fill = sl.fused ? (sl.cs.fan ? 2u : 1u) : (sl.ifan ? 3u : 0u);
            stats->reserved0 = 0;
            stats->ms_storage = sl.ms_storage;
            stats->storage_rows = sl.storage_rows;
            stats->storage_bytes = sl.storage_bytes;
        }
    });
}

gx_status gx_pipeline_batch(gx_pipeline* p, uint64_t ticket, uint64_t i, const void** rows, uint64_t* n_rows,
                            void* host_out) {
    return guard([&] {
        if (!p) fail(GX_INVALID_ARGUMENT, "null pipeline");
        const PipeSlot& sl = p->slot[ticket & 1];
        if (sl.ticket != ticket || sl.pending)
            fail(GX_LOGIC_ERROR, "batches are readable after wait(ticket) until that slot is resubmitted");
        if (i >= sl.S) fail(GX_OUT_OF_RANGE, "iteration index out of range");
        if (!sl.full && i + 1 != sl.S)
            fail(GX_LOGIC_ERROR, "superbatch exceeded GX_BATCH_BUDGET_MB: only the last iteration's rows are resident");
        const uint8_t* src = sl.batch.p + (sl.full ? sl.o[i] : sl.last_row) * p->f->row_bytes;
        const uint64_t n = sl.o[i + 1] - sl.o[i];
        if (rows) *rows = src;
        if (n_rows) *n_rows = n;
        if (host_out && n) {
            GX_CUDA(cudaMemcpyAsync(host_out, src, n * p->f->row_bytes, cudaMemcpyDeviceToHost, p->exec));
            GX_CUDA(cudaStreamSynchronize(p->exec));
        }
    });
}

gx_status gx_pipeline_copy_superbatch(gx_pipeline* p, uint64_t ticket, void* host_out, uint64_t cap,
                                      uint64_t* bytes) {
    return guard([&] {
        if (!p) fail(GX_INVALID_ARGUMENT, "null pipeline");
        const PipeSlot& sl = p->slot[ticket & 1];
        if (sl.ticket != ticket || sl.pending)
            fail(GX_LOGIC_ERROR, "batches are readable after wait(ticket) until that slot is resubmitted");
        if (!sl.full) fail(GX_LOGIC_ERROR, "superbatch exceeded GX_BATCH_BUDGET_MB: not resident");
        const uint64_t n = sl.o[sl.S] * p->f->row_bytes;
        if (bytes) *bytes = n;
        if (!host_out || !n) return;
        if (cap < n) fail(GX_INVALID_ARGUMENT, "host buffer smaller than the superbatch's rows");
        GX_CUDA(cudaMemcpyAsync(host_out, sl.batch.p, n, cudaMemcpyDeviceToHost, p->exec));
        GX_CUDA(cudaStreamSynchronize(p->exec));
    });
}

gx_status gx_pipeline_superbatch(gx_pipeline* p, const uint64_t* seeds_flat, const uint64_t* batch_off,
                                 uint64_t S, uint64_t global_seed, uint64_t first_global_batch,
                                 uint64_t* misses_per_iter, gx_pipeline_stats* stats) {
    uint64_t t = 0;
    gx_status st = gx_pipeline_submit(p, seeds_flat, batch_off, S, global_seed, first_global_batch, &t);
    if (st != GX_OK) return st;
    return gx_pipeline_wait(p, t, misses_per_iter, stats);
}

}  // extern "C"
