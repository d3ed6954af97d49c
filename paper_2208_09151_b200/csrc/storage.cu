// storage.cu -- the backing 'SSD' tier (GX_BACKING_FILE).
//
// The reference reads every missed feature row with one pread of the row's
// bytes (FeatureFile::read_row, graph_store.hpp:308-315) on the calling thread,
// through the page cache (PreadFile opens O_RDONLY, common.hpp:278). Here the
// rows a superbatch misses are known before its executor runs (the inspector
// resolved every access), so they are fetched in bulk:
//   1. the requests (node ids) are sorted by id on the device (CUB radix sort
//      of (id, request index) pairs) and the sorted ids come back to the host;
//   2. a host thread pool reads them as coalesced runs of whole 4 KB pages
//      (O_DIRECT when the filesystem allows it: page-aligned offsets, lengths
//      and buffers; rows that straddle pages are covered by the run) and
//      extracts the rows into a pinned chunk, in sorted order;
//   3. each chunk is copied to HBM on the features' copy stream while the
//      host reads the next one (two pinned + two device landing buffers), and
//      a scatter kernel on the consumer stream moves the rows to their
//      destinations (cache slots for the init set, staging rows for misses).
// The reference's IoStats page accounting is unchanged (the gather kernels
// charge page_count_for_row per miss); physical reads are counted separately
// (gx_storage_stats).
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdlib>
#include <cub/cub.cuh>
#include <thread>

#include "gx_internal.cuh"

namespace gx {

static uint64_t round_down(uint64_t x, uint64_t a) { return x / a * a; }
static uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

RowReader::RowReader(const char* p, uint64_t payload_off, uint64_t row_bytes, uint64_t n_rows)
    : path(p), poff(payload_off), rb(row_bytes), n(n_rows) {
    const bool want_direct = env_int("GX_SSD_DIRECT", 1) != 0;
    if (want_direct) {
        fd = ::open(p, O_RDONLY | O_DIRECT);
        direct = fd >= 0;
        if (direct) {  // some filesystems accept the flag at open but refuse the reads
            void* probe = nullptr;
            if (posix_memalign(&probe, kPage, kPage) != 0) fail(GX_RUNTIME_ERROR, "allocation failed");
            const ssize_t r = ::pread(fd, probe, kPage, 0);
            free(probe);
            if (r < 0) {
                ::close(fd);
                fd = -1;
                direct = false;
            }
        }
    }
    if (fd < 0) fd = ::open(p, O_RDONLY);  // tmpfs / overlay without O_DIRECT: buffered
    if (fd < 0) fail(GX_RUNTIME_ERROR, std::string("cannot open: ") + p);
    const off_t e = ::lseek(fd, 0, SEEK_END);
    if (e < 0) fail(GX_RUNTIME_ERROR, "lseek failed: " + path);
    fsize = (uint64_t)e;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    threads = (unsigned)std::max(1, env_int("GX_SSD_THREADS", (int)std::min(16u, hw)));
    run_cap = std::max<uint64_t>((uint64_t)std::max(4, env_int("GX_SSD_RUN_KB", 512)) << 10,
                                 round_up(rb, kPage) + kPage);
    gap_pages = (uint64_t)std::max(0, env_int("GX_SSD_GAP_PAGES", 8));  // measured: 8 beats 0 on the virtio disk (3.6 vs 2.4 GB/s)
}

RowReader::~RowReader() {
    if (fd >= 0) ::close(fd);
}

// Read [off, off + len) into dst; at least `need` bytes must arrive (a run may
// extend past EOF to the page boundary, O_DIRECT then returns a short read).
void RowReader::pread_full(uint8_t* dst, uint64_t len, uint64_t off, uint64_t need) {
    uint64_t done = 0;
    while (done < len) {
        const ssize_t r = ::pread(fd, dst + done, len - done, (off_t)(off + done));
        if (r < 0) {
            if (errno == EINTR) continue;
            fail(GX_RUNTIME_ERROR, "pread failed: " + path);
        }
        if (r == 0) break;
        done += (uint64_t)r;
        preads.fetch_add(1, std::memory_order_relaxed);
    }
    if (done < need) fail(GX_RUNTIME_ERROR, "truncated feature file: " + path);
    bytes.fetch_add(done, std::memory_order_relaxed);
}

void RowReader::read_range(const uint32_t* sorted, uint64_t lo, uint64_t hi, uint8_t* dst, uint8_t* bounce) {
    uint64_t q = lo;
    while (q < hi) {
        const uint64_t a = poff + (uint64_t)sorted[q] * rb;
        const uint64_t p0 = round_down(a, kPage);
        uint64_t pe = round_up(a + rb, kPage);
        uint64_t q1 = q + 1;
        while (q1 < hi) {
            const uint64_t a1 = poff + (uint64_t)sorted[q1] * rb;
            if (round_down(a1, kPage) > pe + gap_pages * kPage) break;
            const uint64_t ne = std::max(pe, round_up(a1 + rb, kPage));
            if (ne - p0 > run_cap) break;
            pe = ne;
            ++q1;
        }
        const uint64_t last_end = poff + (uint64_t)sorted[q1 - 1] * rb + rb;
        pread_full(bounce, pe - p0, p0, last_end - p0);
        for (uint64_t k = q; k < q1; ++k)
            std::memcpy(dst + (k - lo) * rb, bounce + (poff + (uint64_t)sorted[k] * rb - p0), rb);
        q = q1;
    }
}

void RowReader::read_sorted(const uint32_t* sorted, uint64_t cnt, uint8_t* dst) {
    if (!cnt) return;
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t bounce_bytes = run_cap + 2 * kPage;
    // at least ~256 rows per worker, so small requests stay on one thread
    const unsigned T = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(threads, (cnt + 255) / 256));
    std::vector<uint8_t*> bounce(T, nullptr);
    for (auto& b : bounce)
        if (posix_memalign((void**)&b, kPage, bounce_bytes) != 0) fail(GX_RUNTIME_ERROR, "bounce buffer allocation failed");
    std::vector<std::exception_ptr> errs(T);
    auto work = [&](unsigned t) {
        try {
            const uint64_t lo = cnt * t / T, hi = cnt * (t + 1) / T;
            read_range(sorted, lo, hi, dst + lo * rb, bounce[t]);
        } catch (...) {
            errs[t] = std::current_exception();
        }
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    }
    for (auto b : bounce) free(b);
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    rows.fetch_add(cnt, std::memory_order_relaxed);
    read_ns.fetch_add((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count(),
                      std::memory_order_relaxed);
}

void RowReader::read_rows(const uint64_t* ids, uint64_t cnt, uint8_t* dst) {
    if (!cnt) return;
    std::vector<std::pair<uint32_t, uint64_t>> o(cnt);
    for (uint64_t k = 0; k < cnt; ++k) o[k] = {(uint32_t)ids[k], k};
    std::sort(o.begin(), o.end());
    std::vector<uint32_t> sorted(cnt);
    for (uint64_t k = 0; k < cnt; ++k) sorted[k] = o[k].first;
    std::vector<uint8_t> tmp(cnt * rb);
    read_sorted(sorted.data(), cnt, tmp.data());
    for (uint64_t k = 0; k < cnt; ++k) std::memcpy(dst + o[k].second * rb, tmp.data() + k * rb, rb);
}

StageScratch::~StageScratch() {
    if (copy) cudaStreamSynchronize(copy);
    for (auto& e : ev_h2d)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev_free)
        if (e) cudaEventDestroy(e);
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (copy) cudaStreamDestroy(copy);
}

__global__ void k_iota32(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

// out row dst_idx[q] <- landing row q (one warp per row, 16-byte vectors).
// out2 != nullptr: the row also goes to out2 row idx2[dst_idx[q]] (the
// fused all-fit executor: an init row's slot and its first batch row)
template <int VEC>
__global__ void k_scatter_rows(const uint8_t* __restrict__ land, const uint32_t* __restrict__ dst_idx, uint64_t cnt,
                               uint8_t* __restrict__ out, uint64_t rb, uint8_t* __restrict__ out2,
                               const uint32_t* __restrict__ idx2) {
    using V = typename std::conditional<VEC == 16, uint4, uint32_t>::type;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31, nvec = (uint32_t)(rb / VEC);
    for (uint64_t q = warp; q < cnt; q += nwarps) {
        const uint32_t j = __ldg(dst_idx + q);
        const V* s = reinterpret_cast<const V*>(land + q * rb);
        V* d = reinterpret_cast<V*>(out + (uint64_t)j * rb);
        V* d2 = out2 ? reinterpret_cast<V*>(out2 + (uint64_t)__ldg(idx2 + j) * rb) : nullptr;
        for (uint32_t c = lane; c < nvec; c += 32) {
            const V v = s[c];
            d[c] = v;
            if (d2) d2[c] = v;
        }
    }
}

void launch_scatter_rows(const uint8_t* src, const uint32_t* dst_idx, uint64_t cnt, uint8_t* out, uint64_t rb,
                         int num_sms, cudaStream_t s, uint8_t* out2, const uint32_t* idx2) {
    if (!cnt) return;
    const unsigned blocks = (unsigned)std::min<uint64_t>((cnt * 32 + 255) / 256, (uint64_t)num_sms * 8);
    if (rb % 16 == 0) k_scatter_rows<16><<<blocks, 256, 0, s>>>(src, dst_idx, cnt, out, rb, out2, idx2);
    else k_scatter_rows<4><<<blocks, 256, 0, s>>>(src, dst_idx, cnt, out, rb, out2, idx2);
    GX_CHECK_LAUNCH();
}

static int key_bits(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

double stage_fetch(gx_features* f, const uint32_t* d_ids, uint64_t n, uint8_t* d_out, cudaStream_t s,
                   uint8_t* out2, const uint32_t* idx2) {
    if (!n) return 0.0;
    if (!f->file || !f->ctx) fail(GX_INVALID_ARGUMENT, "stage_fetch needs a GX_BACKING_FILE table with a context");
    gx_ctx* ctx = f->ctx;
    if (!f->stage) f->stage.reset(new StageScratch());
    StageScratch& st = *f->stage;
    if (!st.copy) {
        GX_CUDA(cudaStreamCreateWithFlags(&st.copy, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            GX_CUDA(cudaEventCreateWithFlags(&st.ev_h2d[b], cudaEventDisableTiming));
            GX_CUDA(cudaEventCreateWithFlags(&st.ev_free[b], cudaEventDisableTiming));
        }
        GX_CUDA(cudaEventCreateWithFlags(&st.ev_ready, cudaEventDisableTiming));
    }
    const uint64_t rb = f->row_bytes;
    // (1) sort (id, request index) on the copy stream once the ids are ready on
    // s and the previous call's scatters (which read vals) are done
    GX_CUDA(cudaEventRecord(st.ev_ready, s));
    GX_CUDA(cudaStreamWaitEvent(st.copy, st.ev_ready, 0));
    for (int b = 0; b < 2; ++b) GX_CUDA(cudaStreamWaitEvent(st.copy, st.ev_free[b], 0));  // any earlier consumer
    st.keys.reserve(n);
    st.keys_alt.reserve(n);
    st.vals.reserve(n);
    st.vals_alt.reserve(n);
    GX_CUDA(cudaMemcpyAsync(st.keys.p, d_ids, n * 4, cudaMemcpyDeviceToDevice, st.copy));
    k_iota32<<<ctx->num_sms * 2, 256, 0, st.copy>>>(st.vals.p, n);
    GX_CHECK_LAUNCH();
    cub::DoubleBuffer<uint32_t> dk(st.keys.p, st.keys_alt.p), dv(st.vals.p, st.vals_alt.p);
    size_t tb = 0;
    const int bits = key_bits(f->n);
    GX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, bits, st.copy));
    st.cub_tmp.reserve(tb + 16);
    GX_CUDA(cub::DeviceRadixSort::SortPairs(st.cub_tmp.p, tb, dk, dv, (int)n, 0, bits, st.copy));
    st.h_sorted.reserve(n);
    GX_CUDA(cudaMemcpyAsync(st.h_sorted.p, dk.Current(), n * 4, cudaMemcpyDeviceToHost, st.copy));
    GX_CUDA(cudaStreamSynchronize(st.copy));
    const uint32_t* perm = dv.Current();
    // (2)+(3) chunked host reads, H2D on the copy stream, scatter on s
    const uint64_t chunk_bytes = (uint64_t)std::max(1, env_int("GX_SSD_CHUNK_MB", 64)) << 20;
    const uint64_t rows_per_chunk = std::max<uint64_t>(1, chunk_bytes / rb);
    const uint64_t cbytes = std::min(n, rows_per_chunk) * rb;
    for (int b = 0; b < 2; ++b) {
        if (st.pin[b].n < cbytes) {
            GX_CUDA(cudaStreamSynchronize(st.copy));
            st.pin[b].alloc(cbytes);
        }
        st.land[b].reserve(cbytes);
    }
    double read_ms = 0;
    bool used[2] = {false, false};
    for (uint64_t c0 = 0, j = 0; c0 < n; c0 += rows_per_chunk, ++j) {
        const int b = (int)(j & 1);
        const uint64_t cnt = std::min(rows_per_chunk, n - c0);
        if (used[b]) GX_CUDA(cudaEventSynchronize(st.ev_h2d[b]));  // pinned buffer b drained
        const auto r0 = std::chrono::steady_clock::now();
        f->file->read_sorted(st.h_sorted.p + c0, cnt, st.pin[b].p);
        read_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();
        if (used[b]) GX_CUDA(cudaStreamWaitEvent(st.copy, st.ev_free[b], 0));  // landing b scattered
        GX_CUDA(cudaMemcpyAsync(st.land[b].p, st.pin[b].p, cnt * rb, cudaMemcpyHostToDevice, st.copy));
        GX_CUDA(cudaEventRecord(st.ev_h2d[b], st.copy));
        f->file->h2d.fetch_add(cnt * rb, std::memory_order_relaxed);
        GX_CUDA(cudaStreamWaitEvent(s, st.ev_h2d[b], 0));
        launch_scatter_rows(st.land[b].p, perm + c0, cnt, d_out, rb, ctx->num_sms, s, out2, idx2);
        GX_CUDA(cudaEventRecord(st.ev_free[b], s));
        used[b] = true;
    }
    return read_ms;
}

__global__ void k_miss_flags(const uint32_t* __restrict__ slots, uint64_t n, uint32_t* __restrict__ flags) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        flags[k] = slots[k] == kNever ? 1u : 0u;
}

__global__ void k_miss_write(const uint32_t* __restrict__ ids, uint32_t* __restrict__ slots,
                             const uint32_t* __restrict__ ranks, uint64_t n, uint32_t* __restrict__ miss_ids) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        if (slots[k] == kNever) {
            const uint32_t r = ranks[k];
            miss_ids[r] = ids[k];
            slots[k] = kStageFlag | r;
        }
}

uint64_t stage_misses(gx_ctx* ctx, const uint32_t* ids, uint32_t* slots, uint64_t n, DevBuf<uint32_t>& miss_ids,
                      cudaStream_t s) {
    if (!n) return 0;
    if (n >= kStageFlag) fail(GX_OVERFLOW, "too many accesses for the staging index");
    // per-context scratch (allocated on this context's device, freed with it)
    DevBuf<uint32_t>&flags = ctx->miss_flags, &ranks = ctx->miss_ranks;
    DevBuf<uint8_t>& tmp = ctx->miss_tmp;
    flags.reserve(n);
    ranks.reserve(n);
    const unsigned g = ctx->num_sms * 4;
    k_miss_flags<<<g, 256, 0, s>>>(slots, n, flags.p);
    GX_CHECK_LAUNCH();
    size_t tb = 0;
    GX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags.p, ranks.p, (int)n, s));
    tmp.reserve(tb + 16);
    GX_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flags.p, ranks.p, (int)n, s));
    uint32_t h[2];
    GX_CUDA(cudaMemcpyAsync(&h[0], ranks.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
    GX_CUDA(cudaMemcpyAsync(&h[1], flags.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
    GX_CUDA(cudaStreamSynchronize(s));
    const uint64_t m = (uint64_t)h[0] + h[1];
    if (m) {
        miss_ids.reserve(m);
        k_miss_write<<<g, 256, 0, s>>>(ids, slots, ranks.p, n, miss_ids.p);
        GX_CHECK_LAUNCH();
    }
    return m;
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_features_storage_stats(const gx_features* f, gx_storage_stats* out) {
    return guard([&] {
        if (!f || !out) fail(GX_INVALID_ARGUMENT, "null handle");
        *out = gx_storage_stats{};
        if (!f->file) return;
        const RowReader& r = *f->file;
        out->rows = r.rows.load();
        out->preads = r.preads.load();
        out->bytes = r.bytes.load();
        out->h2d_bytes = r.h2d.load();
        out->read_ms = (double)r.read_ns.load() / 1e6;
        out->threads = r.threads;
        out->direct = r.direct ? 1 : 0;
    });
}

}  // extern "C"
