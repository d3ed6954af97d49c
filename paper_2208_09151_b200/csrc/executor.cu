// executor.cu -- the feature cache of the executor (feature_cache.hpp) on HBM.
//
// Cache rows: K x row_bytes in HBM; address table: i32[N] (node -> slot, -1
// miss); backing store: the whole feature table in HBM or pinned host memory
// read zero-copy over PCIe (gx_backing). The hot kernels are bandwidth-bound
// row copies:
//  * k_gather  (FeatureCache::gather, feature_cache.hpp:58-76): one warp per
//    row, 16-byte vector loads, several rows in flight per warp; hits read the
//    cache slot, misses the backing store, misses charged one row,
//    page_count_for_row pages and row_bytes bytes (graph_store.hpp:308-315).
//  * k_apply_slots (apply_changeset, feature_cache.hpp:89-130) with the slots
//    the inspector precomputed; k_apply (API path) recomputes them from this
//    cache's own free list, exactly as the reference does.
#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <cstdlib>

#include <cub/cub.cuh>

#include "gx_internal.cuh"

struct gx_cache {
    gx_features* f = nullptr;
    gx_ctx* ctx = nullptr;
    uint64_t K = 0;
    gx::DevBuf<uint8_t> rows;        // K * row_bytes
    gx::DevBuf<int32_t> table;       // N
    gx::DevBuf<uint32_t> free_list;  // K (back = top-1 is the next slot handed out)
    uint64_t free_top = 0;
    gx::DevBuf<unsigned long long> counters;  // hits, misses, pages, rows, bytes
    gx::DevBuf<uint32_t> scratch;             // ids / changeset staging
    gx::DevBuf<unsigned int> err;
};

namespace gx {

constexpr int GA_THREADS = 256;
constexpr int GA_ROWS = 4;  // rows in flight per warp

template <int VEC>
struct VecT;
template <>
struct VecT<16> {
    using T = uint4;
};
template <>
struct VecT<4> {
    using T = uint32_t;
};

__device__ __forceinline__ uint4 ld_nc(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_nc(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ void st_na(uint4* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ void st_na(uint32_t* p, const uint32_t& v) { *p = v; }

// Row gather with pre-resolved sources: row k of `out` = cache slot slots[k]
// or, for a miss, row ids[k] of the backing store (slots[k] == kNever) or row
// slots[k] & ~kStageFlag of the staged rows the storage tier delivered.
// A warp moves R rows per step: lanes 0..R-1 fetch the rows' metadata
// (coalesced), the row base pointers are broadcast by shuffles and every lane
// issues R independent 16-byte loads before the R stores, so R x row_bytes per
// warp are in flight with no dependent index chain on the data path.
// counters: [0] hits [1] misses [2] pages [3] rows [4] bytes (misses only,
// graph_store.hpp:308-315).
template <int R>
struct GatherOcc {
    static constexpr int value = R >= 16 ? 2 : (R >= 8 ? 3 : (R >= 4 ? 5 : 8));
};

// Segment mode (the pipeline gathers several iterations per launch when no
// cache mutation separates them): `off` = the iterations' absolute row offsets
// (n + 1 entries, off[0] = this launch's first row) and every miss is charged to
// its own iteration's counters (8 words per iteration: [1] misses, [2] pages;
// hits, rows and bytes follow from the counts on the host). off == nullptr: one
// counter block for the launch ([0] hits, [1] misses, [2] pages, [3] rows, [4] bytes).
struct SegInfo {
    const uint32_t* off;
    uint32_t n;
    unsigned long long* counters;
};

__device__ __forceinline__ void charge_miss_seg(const SegInfo& sg, uint32_t r, uint32_t pages) {
    const uint32_t ra = r + __ldg(sg.off);
    uint32_t lo = 0, hi = sg.n;  // off[lo] <= ra < off[lo + 1]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(sg.off + mid) <= ra) lo = mid;
        else hi = mid;
    }
    atomicAdd(&sg.counters[8 * lo + 1], 1ull);
    atomicAdd(&sg.counters[8 * lo + 2], (unsigned long long)pages);
}

template <int VEC, int R, bool STAGED>
__global__ void __launch_bounds__(GA_THREADS, GatherOcc<R>::value) k_gather_rows(const uint32_t* __restrict__ ids,
                                                               const uint32_t* __restrict__ slots, uint32_t n,
                                                               const uint8_t* __restrict__ cache_rows,
                                                               const uint8_t* __restrict__ store,
                                                               uint32_t row_bytes, uint8_t* __restrict__ out,
                                                               unsigned long long* counters, SegInfo sg) {
    using V = typename VecT<VEC>::T;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nvec = row_bytes / VEC;
    uint32_t hits = 0, misses = 0, pages = 0;
    for (uint32_t r0 = warp * R; r0 < n; r0 += nwarps * R) {
        const uint32_t nr = min(n - r0, (uint32_t)R);
        const uint8_t* src = nullptr;
        if (lane < nr) {
            const uint32_t v = __ldg(ids + r0 + lane);
            const uint32_t s = slots ? __ldg(slots + r0 + lane) : kNever;
            if (STAGED ? s < kStageFlag : s != kNever) {
                src = cache_rows + (uint64_t)s * row_bytes;
                if (!sg.off) ++hits;
            } else {  // miss: backing row v, or staged row (s & ~kStageFlag)
                src = store + (uint64_t)(STAGED ? (s == kNever ? v : (s & ~kStageFlag)) : v) * row_bytes;
                const uint32_t pg =
                    (uint32_t)pages_touched((uint64_t)v * row_bytes, (uint64_t)v * row_bytes + row_bytes);
                if (sg.off) {
                    charge_miss_seg(sg, r0 + lane, pg);
                } else {
                    ++misses;
                    pages += pg;
                }
            }
        }
        V* dst = reinterpret_cast<V*>(out + (uint64_t)r0 * row_bytes);
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < nvec; c0 += 32) {
            const uint32_t c = c0 + lane;
            V tmp[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const V* sq = reinterpret_cast<const V*>(__shfl_sync(0xffffffffu, (unsigned long long)src, q));
                if (q < (int)nr && c < nvec) tmp[q] = ld_nc(sq + c);
            }
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (q < (int)nr && c < nvec) st_na(dst + q * nvec + c, tmp[q]);
        }
    }
    hits = warp_sum(hits);
    misses = warp_sum(misses);
    pages = warp_sum(pages);
    if (lane == 0 && (hits | misses)) {
        atomicAdd(&counters[0], (unsigned long long)hits);
        atomicAdd(&counters[1], (unsigned long long)misses);
        atomicAdd(&counters[2], (unsigned long long)pages);
        atomicAdd(&counters[3], (unsigned long long)misses);
        atomicAdd(&counters[4], (unsigned long long)misses * row_bytes);
    }
}

// STAGED: the store is a staging buffer (storage tier / partition exchange)
// and a miss reads row (slot & ~kStageFlag) of it; otherwise a miss reads row
// ids[k] of the backing table. Separate instantiations: the extra select on
// the (cold) miss path measurably slows the all-hit gather when compiled in
// (4.1 vs 2.9 ms per papers superbatch), so the HBM-backed path never sees it.
template <bool STAGED>
__device__ __forceinline__ const uint8_t* gather_src(const uint32_t* ids, const uint32_t* slots, uint32_t r,
                                                     const uint8_t* cache_rows, const uint8_t* store,
                                                     uint32_t row_bytes, uint32_t& hits, uint32_t& misses,
                                                     uint32_t& pages, const SegInfo& sg) {
    const uint32_t v = __ldg(ids + r);
    const uint32_t s = slots ? __ldg(slots + r) : kNever;
    if (STAGED ? s < kStageFlag : s != kNever) {
        if (!sg.off) ++hits;
        return cache_rows + (uint64_t)s * row_bytes;
    }
    const uint32_t pg = (uint32_t)pages_touched((uint64_t)v * row_bytes, (uint64_t)v * row_bytes + row_bytes);
    if (sg.off) {
        charge_miss_seg(sg, r, pg);
    } else {
        ++misses;
        pages += pg;
    }
    return store + (uint64_t)(STAGED ? (s == kNever ? v : (s & ~kStageFlag)) : v) * row_bytes;
}

// TMA variant of the row gather: every thread moves whole rows with the bulk
// copy engine, global -> its own smem row buffer (cp.async.bulk + mbarrier
// complete_tx) -> global (cp.async.bulk bulk_group). Bytes in flight are
// bounded by shared memory (blockDim x row_bytes per CTA), not registers.
// Requires row_bytes % 16 == 0 and 16-byte aligned rows.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <bool STAGED>
__global__ void __launch_bounds__(128) k_gather_tma(const uint32_t* __restrict__ ids,
                                                    const uint32_t* __restrict__ slots, uint32_t n,
                                                    const uint8_t* __restrict__ cache_rows,
                                                    const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                    uint8_t* __restrict__ out, unsigned long long* counters, SegInfo sg) {
    extern __shared__ __align__(128) unsigned char sbuf[];
    __shared__ __align__(8) unsigned long long bars[128];
    const uint32_t tid = threadIdx.x;
    const uint32_t bar = smem_u32(&bars[tid]);
    const uint32_t buf = smem_u32(sbuf + (size_t)tid * row_bytes);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t phase = 0;
    uint32_t hits = 0, misses = 0, pages = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + tid; r < n; r += gridDim.x * blockDim.x) {
        const uint8_t* src = gather_src<STAGED>(ids, slots, r, cache_rows, store, row_bytes, hits, misses, pages, sg);
        // the previous row's store must have finished reading the buffer
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(buf),
            "l"(src), "r"(row_bytes), "r"(bar)
            : "memory");
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar),
            "r"(phase)
            : "memory");
        phase ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (uint64_t)r * row_bytes),
                     "r"(buf), "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    hits = warp_sum(hits);
    misses = warp_sum(misses);
    pages = warp_sum(pages);
    if ((tid & 31) == 0 && (hits | misses)) {
        atomicAdd(&counters[0], (unsigned long long)hits);
        atomicAdd(&counters[1], (unsigned long long)misses);
        atomicAdd(&counters[2], (unsigned long long)pages);
        atomicAdd(&counters[3], (unsigned long long)misses);
        atomicAdd(&counters[4], (unsigned long long)misses * row_bytes);
    }
}

// 2-deep per-thread pipeline: the load of row j+1 is in flight while row j is
// stored, so each thread keeps two rows moving.

__device__ __forceinline__ void bulk_load(uint32_t buf, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(buf),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}
#ifndef GX_STORE_EVICT_FIRST
#define GX_STORE_EVICT_FIRST 1
#endif
// Gathered rows are written once and not read again by this step: with an L2
// evict-first policy they do not push the cache rows out of L2 (a small cache,
// e.g. cfg1's 51 MB, then stays L2-resident across iterations).
__device__ __forceinline__ void bulk_store(void* dst, uint32_t buf, uint32_t bytes) {
#if GX_STORE_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst), "r"(buf),
                 "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(buf), "r"(bytes) : "memory");
#endif
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// DSTIDX: row k goes to batch row ids[k] (the fused all-fit gather: a dense
// list of the accesses that are not an init node's first use).
template <bool STAGED, bool DSTIDX = false>
__global__ void __launch_bounds__(128) k_gather_tma2(const uint32_t* __restrict__ ids,
                                                     const uint32_t* __restrict__ slots, uint32_t n,
                                                     const uint8_t* __restrict__ cache_rows,
                                                     const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                     uint8_t* __restrict__ out, unsigned long long* counters, SegInfo sg) {
    extern __shared__ __align__(128) unsigned char sbuf[];
    __shared__ __align__(8) unsigned long long bars[2 * 128];
    const uint32_t tid = threadIdx.x;
    const uint32_t bar0 = smem_u32(&bars[2 * tid]), bar1 = bar0 + 8;
    const uint32_t buf0 = smem_u32(sbuf + (size_t)(2 * tid) * row_bytes), buf1 = buf0 + row_bytes;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t hits = 0, misses = 0, pages = 0;
    const uint32_t step = gridDim.x * blockDim.x;
    uint32_t r = blockIdx.x * blockDim.x + tid;
    uint32_t ph0 = 0, ph1 = 0;
    if (r < n) bulk_load(buf0, gather_src<STAGED>(ids, slots, r, cache_rows, store, row_bytes, hits, misses, pages, sg), row_bytes, bar0);
    for (uint32_t j = 0; r < n; ++j) {
        const uint32_t nx = r + step;
        const bool odd = j & 1;
        if (nx < n) {  // prefetch the next row into the other buffer
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bulk_load(odd ? buf0 : buf1, gather_src<STAGED>(ids, slots, nx, cache_rows, store, row_bytes, hits, misses, pages, sg),
                      row_bytes, odd ? bar0 : bar1);
        }
        const uint64_t dr = DSTIDX ? (uint64_t)__ldg(ids + r) : (uint64_t)r;
        if (odd) {
            bar_wait(bar1, ph1);
            ph1 ^= 1;
            bulk_store(out + dr * row_bytes, buf1, row_bytes);
        } else {
            bar_wait(bar0, ph0);
            ph0 ^= 1;
            bulk_store(out + dr * row_bytes, buf0, row_bytes);
        }
        r = nx;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    hits = warp_sum(hits);
    misses = warp_sum(misses);
    pages = warp_sum(pages);
    if ((tid & 31) == 0 && (hits | misses)) {
        atomicAdd(&counters[0], (unsigned long long)hits);
        atomicAdd(&counters[1], (unsigned long long)misses);
        atomicAdd(&counters[2], (unsigned long long)pages);
        atomicAdd(&counters[3], (unsigned long long)misses);
        atomicAdd(&counters[4], (unsigned long long)misses * row_bytes);
    }
}

// One launch over a whole resident superbatch with changesets (the pipeline's
// device-backed executor): the cache holds exactly its init rows for the
// duration of the launch (the changesets are applied after it), so an access
// whose resolved slot still holds its init node (slot < n_init and
// init[slot] == node) reads the cache slot -- a small, TLB-friendly region --
// and every other access (misses, nodes inserted by a changeset) reads the
// same bytes from the HBM-resident table. No counting here: the per-iteration
// miss counters come from k_count_iter_misses over the same resolved slots.
__global__ void __launch_bounds__(128) k_gather_sb(const uint32_t* __restrict__ ids,
                                                   const uint32_t* __restrict__ slots, uint32_t n,
                                                   const uint32_t* __restrict__ init, uint32_t n_init,
                                                   const uint8_t* __restrict__ cache_rows,
                                                   const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                   uint8_t* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char sbuf[];
    __shared__ __align__(8) unsigned long long bars[2 * 128];
    const uint32_t tid = threadIdx.x;
    const uint32_t bar0 = smem_u32(&bars[2 * tid]), bar1 = bar0 + 8;
    const uint32_t buf0 = smem_u32(sbuf + (size_t)(2 * tid) * row_bytes), buf1 = buf0 + row_bytes;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto src = [&](uint32_t r) -> const uint8_t* {
        const uint32_t v = __ldg(ids + r), sl = __ldg(slots + r);
        if (sl < n_init && __ldg(init + sl) == v) return cache_rows + (uint64_t)sl * row_bytes;
        return store + (uint64_t)v * row_bytes;
    };
    const uint32_t step = gridDim.x * blockDim.x;
    uint32_t r = blockIdx.x * blockDim.x + tid;
    uint32_t ph0 = 0, ph1 = 0;
    if (r < n) bulk_load(buf0, src(r), row_bytes, bar0);
    for (uint32_t j = 0; r < n; ++j) {
        const uint32_t nx = r + step;
        const bool odd = j & 1;
        if (nx < n) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bulk_load(odd ? buf0 : buf1, src(nx), row_bytes, odd ? bar0 : bar1);
        }
        if (odd) {
            bar_wait(bar1, ph1);
            ph1 ^= 1;
            bulk_store(out + (uint64_t)r * row_bytes, buf1, row_bytes);
        } else {
            bar_wait(bar0, ph0);
            ph0 ^= 1;
            bulk_store(out + (uint64_t)r * row_bytes, buf0, row_bytes);
        }
        r = nx;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// D-stage ring of bulk copies per thread: D-1 row loads stay in flight while
// the previous row's bulk store drains; a buffer is refilled once its store has
// read shared memory (wait_group.read 1 = all but the newest store).
template <int D>
__global__ void __launch_bounds__(256) k_gather_ring(const uint32_t* __restrict__ ids,
                                                     const uint32_t* __restrict__ slots, uint32_t n,
                                                     const uint8_t* __restrict__ cache_rows,
                                                     const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                     uint8_t* __restrict__ out, unsigned long long* counters, SegInfo sg) {
    extern __shared__ __align__(128) unsigned char sbuf[];
    __shared__ __align__(8) unsigned long long bars[D * 256];
    const uint32_t tid = threadIdx.x;
    const uint32_t bar_base = smem_u32(&bars[D * tid]);
    const uint32_t buf_base = smem_u32(sbuf + (size_t)(D * tid) * row_bytes);
#pragma unroll
    for (int k = 0; k < D; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_base + 8 * k));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    uint32_t hits = 0, misses = 0, pages = 0;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t r0 = (uint64_t)blockIdx.x * blockDim.x + tid;
#pragma unroll
    for (int k = 0; k < D - 1; ++k) {
        const uint64_t r = r0 + k * step;
        if (r < n)
            bulk_load(buf_base + k * row_bytes,
                      gather_src<false>(ids, slots, (uint32_t)r, cache_rows, store, row_bytes, hits, misses, pages, sg),
                      row_bytes, bar_base + 8 * k);
    }
    uint32_t b = 0, par = 0;  // buffer of row j, and its barrier parity ((j / D) & 1)
    for (uint64_t r = r0; r < n; r += step) {
        bar_wait(bar_base + 8 * b, par);
        bulk_store(out + r * row_bytes, buf_base + b * row_bytes, row_bytes);
        const uint64_t rn = r + (D - 1) * step;
        const uint32_t bn = b == 0 ? D - 1 : b - 1;  // (j + D - 1) % D
        if (rn < n) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            bulk_load(buf_base + bn * row_bytes,
                      gather_src<false>(ids, slots, (uint32_t)rn, cache_rows, store, row_bytes, hits, misses, pages, sg),
                      row_bytes, bar_base + 8 * bn);
        }
        if (++b == D) {
            b = 0;
            par ^= 1;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    hits = warp_sum(hits);
    misses = warp_sum(misses);
    pages = warp_sum(pages);
    if ((tid & 31) == 0 && (hits | misses)) {
        atomicAdd(&counters[0], (unsigned long long)hits);
        atomicAdd(&counters[1], (unsigned long long)misses);
        atomicAdd(&counters[2], (unsigned long long)pages);
        atomicAdd(&counters[3], (unsigned long long)misses);
        atomicAdd(&counters[4], (unsigned long long)misses * row_bytes);
    }
}

// Fused cache fill for an all-fit superbatch (the "switch" and the first use of
// every init node in one pass): init slot r <- backing row init[r], and the
// same bytes to the batch row of the slot's first use, first_acc[r]. R rows
// in flight per warp, 16-byte loads, two 16-byte stores per load.
template <int R>
__global__ void __launch_bounds__(GA_THREADS, GatherOcc<R>::value) k_fill_first(const uint32_t* __restrict__ init,
                                                               const uint32_t* __restrict__ first_acc, uint32_t n,
                                                               const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                               uint8_t* __restrict__ cache_rows,
                                                               uint8_t* __restrict__ batch) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nvec = row_bytes / 16;
    for (uint32_t r0 = warp * R; r0 < n; r0 += nwarps * R) {
        const uint32_t nr = min(n - r0, (uint32_t)R);
        const uint8_t* src = nullptr;
        uint8_t* dst2 = nullptr;
        if (lane < nr) {
            src = store + (uint64_t)__ldg(init + r0 + lane) * row_bytes;
            dst2 = batch + (uint64_t)__ldg(first_acc + r0 + lane) * row_bytes;
        }
        uint4* dst1 = reinterpret_cast<uint4*>(cache_rows + (uint64_t)r0 * row_bytes);
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < nvec; c0 += 32) {
            const uint32_t c = c0 + lane;
            uint4 tmp[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const uint4* sq = reinterpret_cast<const uint4*>(__shfl_sync(0xffffffffu, (unsigned long long)src, q));
                if (q < (int)nr && c < nvec) tmp[q] = ld_nc(sq + c);
            }
#pragma unroll
            for (int q = 0; q < R; ++q) {
                uint4* dq = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, (unsigned long long)dst2, q));
                if (q < (int)nr && c < nvec) {
                    st_na(dst1 + q * nvec + c, tmp[q]);
                    st_na(dq + c, tmp[q]);
                }
            }
        }
    }
}

// Fan-out executor for an all-fit superbatch: every init row is read ONCE and
// written to its cache slot, to the batch row of its first use first[r] and to
// the batch rows of its other accesses list[off[r - 1] .. off[r]), so no access
// re-reads the cache: (3w + 12) bytes per init row + (w + 4) per other access
// instead of (3w + 8) per init row + (2w + 8) per other access (fill + gather).
// A warp takes R consecutive slots: their lists are one contiguous run, so one
// coalesced load brings the first 32 destinations of all R slots into lanes.
// Measured and removed: a bulk-copy form (lanes issue cp.async.bulk stores of
// their destinations from smem row buffers, the next group's loads in flight:
// 2.94 vs 2.85 ms), 64-register builds, L2 evict-first stores, prefetching the
// next group's offsets and list window (2.85-2.93 ms).
template <int R>
__global__ void __launch_bounds__(GA_THREADS, GatherOcc<R>::value) k_fan_rows(
    const uint32_t* __restrict__ idx, uint32_t n, const uint8_t* __restrict__ src, uint32_t row_bytes,
    uint8_t* __restrict__ cache_rows, const uint32_t* __restrict__ first, const uint32_t* __restrict__ off,
    const uint32_t* __restrict__ list, uint8_t* __restrict__ batch) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nvec = row_bytes / 16;
    for (uint32_t r0 = warp * R; r0 < n; r0 += nwarps * R) {
        const uint32_t nr = min(n - r0, (uint32_t)R);
        // lanes < nr: source row and first-use row of slot r0 + lane;
        // lanes <= nr: range ends (slot s: [off[s - 1], off[s]))
        const uint8_t* sp = nullptr;
        uint8_t* fp = nullptr;
        if (lane < nr) {
            sp = src + (uint64_t)(idx ? __ldg(idx + r0 + lane) : r0 + lane) * row_bytes;
            if (first) fp = batch + (uint64_t)__ldg(first + r0 + lane) * row_bytes;
        }
        const uint32_t o = lane <= nr && r0 + lane ? __ldg(off + r0 + lane - 1) : 0u;
        const uint32_t base = __shfl_sync(0xffffffffu, o, 0), end = __shfl_sync(0xffffffffu, o, nr);
        // rows to read: all (a first use or a cache slot to write), else only
        // slots with other accesses (staged tiers: the slots are already filled)
        const uint32_t o_next = __shfl_down_sync(0xffffffffu, o, 1);
        const uint32_t need = __ballot_sync(0xffffffffu, lane < nr && (first || cache_rows || o_next > o));
        const uint32_t d = base + lane < end ? __ldg(list + base + lane) : 0u;
#pragma unroll 1
        for (uint32_t c0 = 0; c0 < nvec; c0 += 32) {
            const uint32_t c = c0 + lane;
            uint4 tmp[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const uint4* sq = reinterpret_cast<const uint4*>(__shfl_sync(0xffffffffu, (unsigned long long)sp, q));
                if (((need >> q) & 1) && c < nvec) tmp[q] = ld_nc(sq + c);
            }
#pragma unroll
            for (int q = 0; q < R; ++q) {
                if (q >= (int)nr) break;
                uint4* fq = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, (unsigned long long)fp, q));
                if (c < nvec) {
                    if (cache_rows) st_na(reinterpret_cast<uint4*>(cache_rows + (uint64_t)(r0 + q) * row_bytes) + c, tmp[q]);
                    if (fq) st_na(fq + c, tmp[q]);
                }
                const uint32_t b = __shfl_sync(0xffffffffu, o, q), e = __shfl_sync(0xffffffffu, o, q + 1);
                for (uint32_t j = b; j < e; ++j) {
                    const uint32_t v = __shfl_sync(0xffffffffu, d, (j - base) & 31);
                    const uint32_t x = j - base < 32 ? v : __ldg(list + j);
                    if (c < nvec) st_na(reinterpret_cast<uint4*>(batch + (uint64_t)x * row_bytes) + c, tmp[q]);
                }
            }
        }
    }
}

void launch_fan_rows(gx_ctx* ctx, const uint32_t* idx, uint32_t n, const uint8_t* src, uint64_t rb,
                     uint8_t* cache_rows, const uint32_t* first, const uint32_t* off, const uint32_t* list,
                     uint8_t* batch) {
    if (!n) return;
    if (rb % 16) fail(GX_INVALID_ARGUMENT, "fan-out fill needs 16-byte rows");
    static const int rr = env_int("GX_FAN_R", 16);  // slots per warp: 4, 8 or 16 (16: 2.83 vs 2.89 ms for 8, r02z_ab_fan_r.txt)
    auto go = [&](auto kfn, int R) {
        int bps = 0;
        GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, GA_THREADS, 0));
        const uint64_t warps_needed = (n + R - 1) / R;
        const uint64_t blocks = std::min<uint64_t>((warps_needed * 32 + GA_THREADS - 1) / GA_THREADS,
                                                   (uint64_t)ctx->num_sms * std::max(bps, 1));
        kfn<<<(unsigned)blocks, GA_THREADS, 0, lstream(ctx)>>>(idx, n, src, (uint32_t)rb, cache_rows, first, off,
                                                               list, batch);
        GX_CHECK_LAUNCH();
    };
    if (rr == 4) go(k_fan_rows<4>, 4);
    else if (rr == 16) go(k_fan_rows<16>, 16);
    else go(k_fan_rows<8>, 8);
}

static int gather_smem_budget(uint64_t rb);

// Bulk-copy form of the fused fill: each thread moves whole rows through its
// own two smem buffers (load of row j+1 in flight while row j is stored), and
// every row is stored twice from the same buffer (cache slot, batch row).
__global__ void __launch_bounds__(128) k_fill_first_tma(const uint32_t* __restrict__ init,
                                                        const uint32_t* __restrict__ first_acc, uint32_t n,
                                                        const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                        uint8_t* __restrict__ cache_rows, uint8_t* __restrict__ batch) {
    extern __shared__ __align__(128) unsigned char sbuf[];
    __shared__ __align__(8) unsigned long long bars[2 * 128];
    const uint32_t tid = threadIdx.x;
    const uint32_t bar0 = smem_u32(&bars[2 * tid]), bar1 = bar0 + 8;
    const uint32_t buf0 = smem_u32(sbuf + (size_t)(2 * tid) * row_bytes), buf1 = buf0 + row_bytes;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint32_t step = gridDim.x * blockDim.x;
    uint32_t r = blockIdx.x * blockDim.x + tid;
    uint32_t ph0 = 0, ph1 = 0;
    if (r < n) bulk_load(buf0, store + (uint64_t)__ldg(init + r) * row_bytes, row_bytes, bar0);
    for (uint32_t j = 0; r < n; ++j, r += step) {
        const uint32_t nx = r + step;
        const bool odd = j & 1;
        if (nx < n) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            bulk_load(odd ? buf0 : buf1, store + (uint64_t)__ldg(init + nx) * row_bytes, row_bytes, odd ? bar0 : bar1);
        }
        const uint64_t x = __ldg(first_acc + r);
        const uint32_t buf = odd ? buf1 : buf0;
        if (odd) {
            bar_wait(bar1, ph1);
            ph1 ^= 1;
        } else {
            bar_wait(bar0, ph0);
            ph0 ^= 1;
        }
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(cache_rows + (uint64_t)r * row_bytes),
                     "r"(buf), "r"(row_bytes) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(batch + x * row_bytes),
                     "r"(buf), "r"(row_bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// launch configuration of a dynamic-smem kernel for one row size on one device
struct LaunchCfg {
    uint64_t rb = 0;  // row size the entry was set up for (0 = not yet)
    int tpb = 0, bps = 0;
};

void launch_fill_first(gx_ctx* ctx, const uint32_t* init, const uint32_t* first_acc, uint32_t n,
                       const uint8_t* store, uint64_t rb, uint8_t* cache_rows, uint8_t* batch) {
    if (!n) return;
    if (rb % 16) fail(GX_INVALID_ARGUMENT, "fused fill needs 16-byte rows");
    static const int tma = env_int("GX_FILL_TMA", 0);  // bulk-copy form: 1.85 vs 1.67 ms (LDG/STG) at papers shape
    if (tma && (uint64_t)2 * 32 * rb <= (uint64_t)gather_smem_budget(rb)) {
        static PerDevice<LaunchCfg> cfg_dev;  // the smem attribute is per device
        auto lk = cfg_dev.lock();
        LaunchCfg& cf = cfg_dev.at(ctx->device);
        if (cf.rb != rb) {
            cf.tpb = (int)std::min<uint64_t>(128, gather_smem_budget(rb) / (2 * rb)) & ~31;
            const int smem = cf.tpb * 2 * (int)rb;
            GX_CUDA(cudaFuncSetAttribute(k_fill_first_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cf.bps, k_fill_first_tma, cf.tpb, smem));
            cf.bps = std::max(cf.bps, 1);
            cf.rb = rb;
        }
        const int tpb = cf.tpb, bpsm = cf.bps;
        const uint64_t blocks = std::min<uint64_t>((n + tpb - 1) / tpb, (uint64_t)ctx->num_sms * bpsm);
        k_fill_first_tma<<<(unsigned)blocks, tpb, (size_t)tpb * 2 * rb, lstream(ctx)>>>(init, first_acc, n, store,
                                                                                      (uint32_t)rb, cache_rows, batch);
        GX_CHECK_LAUNCH();
        return;
    }
    static const int rr = env_int("GX_FILL_R", 8);  // rows in flight per warp: 4, 8 or 16
    auto go = [&](auto kfn, int R) {
        int bps = 0;
        GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, GA_THREADS, 0));
        const uint64_t warps_needed = (n + R - 1) / R;
        const uint64_t blocks = std::min<uint64_t>((warps_needed * 32 + GA_THREADS - 1) / GA_THREADS,
                                                   (uint64_t)ctx->num_sms * std::max(bps, 1));
        kfn<<<(unsigned)blocks, GA_THREADS, 0, lstream(ctx)>>>(init, first_acc, n, store, (uint32_t)rb, cache_rows,
                                                               batch);
        GX_CHECK_LAUNCH();
    };
    if (rr == 4) go(k_fill_first<4>, 4);
    else if (rr == 16) go(k_fill_first<16>, 16);
    else go(k_fill_first<8>, 8);
}

// Address-table resolution for the API path: slots[k] = table[ids[k]] (or kNever).
__global__ void k_resolve(const uint32_t* __restrict__ ids, uint64_t n, const int32_t* __restrict__ table,
                          uint32_t* __restrict__ slots) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t s = table[ids[k]];
        slots[k] = s >= 0 ? (uint32_t)s : kNever;
    }
}

template <int VEC>
__device__ __forceinline__ void warp_copy_row(const uint8_t* src, uint8_t* dst, uint64_t row_bytes) {
    using V = typename VecT<VEC>::T;
    const uint32_t nvec = (uint32_t)(row_bytes / VEC);
    const V* s = reinterpret_cast<const V*>(src);
    V* d = reinterpret_cast<V*>(dst);
    for (uint32_t c = threadIdx.x & 31; c < nvec; c += 32) d[c] = s[c];
}

// Changeset application with precomputed slots (pipeline path).
template <int VEC>
__global__ void k_apply_slots(const uint32_t* __restrict__ in_ids, const uint32_t* __restrict__ in_pos,
                              const uint32_t* __restrict__ in_slot, uint32_t n_in,
                              const uint32_t* __restrict__ out_ids, uint32_t n_out, int32_t* table,
                              const uint8_t* __restrict__ batch, uint8_t* cache_rows, uint64_t row_bytes) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t m = max(n_in, n_out);
    for (uint64_t k = warp; k < m; k += nwarps) {
        if (table && k < n_out && lane == 0) table[out_ids[k]] = -1;
        if (k < n_in) {
            const uint32_t s = in_slot[k];
            warp_copy_row<VEC>(batch + (uint64_t)in_pos[k] * row_bytes, cache_rows + (uint64_t)s * row_bytes,
                               row_bytes);
            if (table && lane == 0) table[in_ids[k]] = (int32_t)s;
        }
    }
}

// API-path validation (feature_cache.hpp:96-112): any violation -> logic_error.
__global__ void k_apply_validate(const uint32_t* ids, uint32_t n_ids, const uint32_t* in_ids,
                                 const uint32_t* in_pos, uint32_t n_in, const uint32_t* out_ids,
                                 uint32_t n_out, const int32_t* table, uint64_t N, unsigned int* err) {
    const uint32_t G = gridDim.x * blockDim.x;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_in; k += G) {
        const uint32_t v = in_ids[k], p = in_pos[k];
        if (p >= n_ids || ids[p] != v) atomicOr(err, 1u);
        else if (v >= N) atomicOr(err, 2u);
        else if (table[v] >= 0) atomicOr(err, 1u);
    }
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_out; k += G) {
        const uint32_t v = out_ids[k];
        if (v >= N || table[v] < 0) atomicOr(err, 1u);
    }
}

// API-path mutation: freed[k] = table[out[k]]; in[k] -> freed[k] or the free
// list back; surplus freed slots are pushed back in order.
template <int VEC>
__global__ void k_apply(const uint32_t* __restrict__ in_ids, const uint32_t* __restrict__ in_pos,
                        uint32_t n_in, const uint32_t* __restrict__ out_ids, uint32_t n_out, int32_t* table,
                        uint32_t* free_list, uint64_t top, const uint8_t* __restrict__ batch,
                        uint8_t* cache_rows, uint64_t row_bytes) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t m = max(n_in, n_out);
    for (uint64_t k = warp; k < m; k += nwarps) {
        int32_t freed = -1;
        if (k < n_out) freed = table[out_ids[k]];
        __syncwarp();
        if (k < n_out && lane == 0) {
            table[out_ids[k]] = -1;
            if (k >= n_in) free_list[top + (k - n_in)] = (uint32_t)freed;
        }
        if (k < n_in) {
            const uint32_t s = k < n_out ? (uint32_t)freed : free_list[top - 1 - (k - n_out)];
            warp_copy_row<VEC>(batch + (uint64_t)in_pos[k] * row_bytes, cache_rows + (uint64_t)s * row_bytes,
                               row_bytes);
            if (lane == 0) table[in_ids[k]] = (int32_t)s;
        }
    }
}

// Changesets with duplicate ids (API path). The reference accepts them and
// runs its loops in order (feature_cache.hpp:103-129): a duplicated out id
// frees the same slot twice, a duplicated in id is rewritten by its later
// entry. One warp replays exactly that sequence (rows lane-strided, so a
// later copy into the same slot lands after the earlier one).
template <int VEC>
__global__ void k_apply_serial(const uint32_t* __restrict__ in_ids, const uint32_t* __restrict__ in_pos,
                               uint32_t n_in, const uint32_t* __restrict__ out_ids, uint32_t n_out, int32_t* table,
                               uint32_t* free_list, uint64_t top, const uint8_t* __restrict__ batch,
                               uint8_t* cache_rows, uint64_t row_bytes, uint32_t* freed) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t k = lane; k < n_out; k += 32) freed[k] = (uint32_t)table[out_ids[k]];  // pre-update state
    __syncwarp();
    for (uint32_t k = lane; k < n_out; k += 32) table[out_ids[k]] = -1;
    __syncwarp();
    uint64_t t = top;
    for (uint32_t k = 0; k < n_in; ++k) {
        const uint32_t s = k < n_out ? freed[k] : free_list[--t];
        warp_copy_row<VEC>(batch + (uint64_t)in_pos[k] * row_bytes, cache_rows + (uint64_t)s * row_bytes, row_bytes);
        if (lane == 0) table[in_ids[k]] = (int32_t)s;
        __syncwarp();
    }
    for (uint32_t k = n_in + lane; k < n_out; k += 32) free_list[t + (k - n_in)] = freed[k];
}

__global__ void k_iota_desc(uint32_t* p, uint64_t n, uint64_t K) {
    // free list [K-1, K-2, ..., K-n]: back() pops ascending from K-n
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)(K - 1 - i);
}

__global__ void k_reset_table(const uint32_t* nodes, uint64_t n, int32_t* table) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        table[nodes[i]] = -1;
}

__global__ void k_resident(const int32_t* table, uint64_t N, uint32_t* out, uint64_t cap, unsigned int* cnt) {
    // compaction in id order via a two-level approach is not needed for a test
    // hook: emit (unordered, at most cap) and let the host sort.
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < N;
         v += (uint64_t)gridDim.x * blockDim.x)
        if (table[v] >= 0) {
            const unsigned int k = atomicAdd(cnt, 1u);
            if (k < cap) out[k] = (uint32_t)v;
        }
}

static bool vec16(uint64_t row_bytes) { return row_bytes % 16 == 0; }


// digest = sum over u32 words x of (word[x] + 1) * mix64(x)  (mod 2^64)
__global__ void k_digest(const uint32_t* __restrict__ w, uint64_t nwords, unsigned long long* out) {
    unsigned long long acc = 0;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < nwords;
         x += (uint64_t)gridDim.x * blockDim.x)
        acc += ((unsigned long long)w[x] + 1ull) * mix64(x);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

void launch_digest(gx_ctx* ctx, const uint8_t* batch, uint64_t rows, uint64_t row_bytes,
                   unsigned long long* out) {
    const uint64_t nw = rows * row_bytes / 4;
    if (!nw) return;
    k_digest<<<ctx->num_sms * 4, 256, 0, lstream(ctx)>>>(reinterpret_cast<const uint32_t*>(batch), nw, out);
    GX_CHECK_LAUNCH();
}

// Launchers shared with the pipeline.
template <int VEC, int R, bool STAGED = false>
static void gather_rows_launch(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, uint64_t n,
                               const uint8_t* cache_rows, const uint8_t* store, uint64_t rb, uint8_t* out,
                               unsigned long long* counters, SegInfo sg = {nullptr, 0, nullptr}) {
    static const int bps = [] {
        int b = 0;
        GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_gather_rows<VEC, R, STAGED>, GA_THREADS, 0));
        return std::max(b, 1);
    }();
    const uint64_t warps_needed = (n + R - 1) / R;
    const uint64_t blocks_needed = (warps_needed * 32 + GA_THREADS - 1) / GA_THREADS;
    const uint64_t blocks = std::min<uint64_t>(blocks_needed, (uint64_t)ctx->num_sms * bps);
    k_gather_rows<VEC, R, STAGED><<<(unsigned)blocks, GA_THREADS, 0, lstream(ctx)>>>(
        ids, slots, (uint32_t)n, cache_rows, store, (uint32_t)rb, out, counters, sg);
    GX_CHECK_LAUNCH();
}

static int gather_variant() {
    static const int R = [] {
        const char* e = std::getenv("GX_GATHER_R");
        const int r = e ? std::atoi(e) : 1;
        return (r == 0 || r == 1 || r == 2 || r == 4 || r == 8) ? r : 1;
    }();
    return R;
}
// shared memory per CTA for the bulk-copy row buffers: three full warps with
// two rows in flight each (96 KB at 512-byte rows -> two CTAs per SM; 192 KB at
// 1 KB rows -> one; measured at friendster shape: 0.98 vs 0.88 of peak against
// a fixed 96 KB, whose 48-thread CTAs leave half a warp idle)
static int gather_smem_budget(uint64_t rb = 512) {
    static const int knob = env_int("GX_GATHER_SMEM_KB", 0);
    if (knob > 0) return std::min(std::max(knob, 16), 200) * 1024;
    return (int)std::min<uint64_t>(200 * 1024, std::max<uint64_t>(16 * 1024, 96 * 2 * rb));
}

// the pipeline may fuse the fill with the first uses only when the gather that
// will serve the rest is the bulk-copy kernel (its DSTIDX instantiation)
bool gather_can_skip_first(uint64_t rb) {
    static const bool on = env_int("GX_FUSED_FILL", 1) != 0;
    return on && vec16(rb) && gather_variant() == 1 && (uint64_t)2 * 32 * rb <= (uint64_t)gather_smem_budget(rb);
}

void launch_gather_resolved(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, uint64_t n,
                            const uint8_t* cache_rows, const uint8_t* store, uint64_t rb, uint8_t* out,
                            unsigned long long* counters, const uint32_t* seg_off, uint32_t nseg, bool staged,
                            bool skip_first) {
    if (!n) return;
    const SegInfo sg{seg_off, seg_off ? nseg : 0u, counters};
    // Variant (tuning knob GX_GATHER_R): 1 = TMA bulk, 2 rows in flight per
    // thread (default); 0 = TMA bulk, 1 row per thread; 2/4/8 = LDG/STG with
    // that many rows per warp. TMA needs 16-byte rows whose buffers fit smem.
    const int R = gather_variant();
    const int budget = gather_smem_budget(rb);
    static const int ring = env_int("GX_GATHER_D", 0);  // 3/4/6: k_gather_ring<D> (experimental)
    static std::mutex cfg_mu;  // launch-config caches below are shared by every context / host thread
    std::lock_guard<std::mutex> cfg_lock(cfg_mu);
    const int dev = ctx->device;  // dynamic-smem attributes are per device
    if (!staged && vec16(rb) && R == 1 && (ring == 3 || ring == 4 || ring == 6) &&
        (uint64_t)ring * 32 * rb <= (uint64_t)budget) {
        static std::map<int, LaunchCfg> ring_cfg;  // per device
        LaunchCfg& cf = ring_cfg[dev];
        auto kfn = ring == 3 ? k_gather_ring<3> : ring == 4 ? k_gather_ring<4> : k_gather_ring<6>;
        if (cf.rb != rb) {
            cf.rb = rb;
            cf.tpb = (int)std::min<uint64_t>(256, budget / (ring * rb)) & ~31;
            const int smem = cf.tpb * ring * (int)rb;
            GX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cf.bps, kfn, cf.tpb, smem));
            cf.bps = std::max(cf.bps, 1);
        }
        const int tpb = cf.tpb, bpsm = cf.bps;
        static const int ctas_knob = env_int("GX_GATHER_CTAS", 0);
        const uint64_t cap = ctas_knob > 0 ? (uint64_t)ctas_knob : (uint64_t)ctx->num_sms * bpsm;
        const uint64_t blocks = std::min<uint64_t>((n + tpb - 1) / tpb, cap);
        kfn<<<(unsigned)blocks, tpb, (size_t)tpb * ring * rb, lstream(ctx)>>>(ids, slots, (uint32_t)n, cache_rows,
                                                                            store, (uint32_t)rb, out,
                                                                            counters, sg);
        GX_CHECK_LAUNCH();
        return;
    }
    const int depth = R == 1 ? 2 : 1;
    if (skip_first && (staged || !gather_can_skip_first(rb)))
        fail(GX_LOGIC_ERROR, "the fused all-fit gather needs the bulk-copy kernel");
    if (vec16(rb) && R <= 1 && (uint64_t)depth * 32 * rb <= (uint64_t)budget) {
        // launch config per (depth, staged), cached for the last row size
        static std::map<int, std::array<LaunchCfg, 6>> tma_cfg;  // per device
        std::array<LaunchCfg, 6>& cfs = tma_cfg[dev];
        const bool skip = skip_first && depth == 2 && !staged;
        const int d = skip ? 4 : (depth - 1) + 2 * (int)staged;
        using KFn = void (*)(const uint32_t*, const uint32_t*, uint32_t, const uint8_t*, const uint8_t*, uint32_t,
                             uint8_t*, unsigned long long*, SegInfo);
        const KFn kfn = skip ? (KFn)k_gather_tma2<false, true>
                        : depth == 2 ? (staged ? (KFn)k_gather_tma2<true> : (KFn)k_gather_tma2<false>)
                                     : (staged ? (KFn)k_gather_tma<true> : (KFn)k_gather_tma<false>);
        LaunchCfg& cf = cfs[d];
        if (cf.rb != rb) {  // threads per CTA: one (or two) row buffers per thread
            cf.tpb = (int)std::min<uint64_t>(128, budget / (depth * rb)) & ~31;
            const int smem = cf.tpb * depth * (int)rb;
            GX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cf.bps, kfn, cf.tpb, smem));
            cf.bps = std::max(cf.bps, 1);
            cf.rb = rb;
        }
        static const int ctas_knob = env_int("GX_GATHER_CTAS", 0);  // cap on CTAs (0 = all resident)
        const uint64_t cap = ctas_knob > 0 ? (uint64_t)ctas_knob : (uint64_t)ctx->num_sms * cf.bps;
        const uint64_t blocks = std::min<uint64_t>((n + cf.tpb - 1) / cf.tpb, cap);
        kfn<<<(unsigned)blocks, cf.tpb, (size_t)cf.tpb * depth * rb, lstream(ctx)>>>(
            ids, slots, (uint32_t)n, cache_rows, store, (uint32_t)rb, out, counters, sg);
        GX_CHECK_LAUNCH();
    } else if (vec16(rb)) {
        if (staged) gather_rows_launch<16, 4, true>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
        else if (R == 2) gather_rows_launch<16, 2>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
        else if (R == 8) gather_rows_launch<16, 8>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
        else gather_rows_launch<16, 4>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
    } else if (staged) {
        gather_rows_launch<4, 4, true>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
    } else {
        gather_rows_launch<4, 4>(ctx, ids, slots, n, cache_rows, store, rb, out, counters, sg);
    }
}

void launch_gather(gx_ctx* ctx, const uint32_t* ids, uint64_t n, const int32_t* table, const uint8_t* cache_rows,
                   gx_features* f, uint8_t* out, unsigned long long* counters) {
    if (!n) {
        if (f->backing == GX_BACKING_PARTITIONED) {  // still take part in the exchange
            ctx->stage_ids.reserve(1);
            fetch_rows(f, ctx->stage_ids.p, 0, nullptr, lstream(ctx));
        }
        return;
    }
    DevBuf<uint32_t>& slots = ctx->resolve_slots;  // API path only
    slots.reserve(n);
    k_resolve<<<ctx->num_sms * 4, 256, 0, lstream(ctx)>>>(ids, n, table, slots.p);
    GX_CHECK_LAUNCH();
    const uint8_t* store = f->rows_dev_view;
    if (staged_backing(f)) {  // misses come from the storage tier / the owning ranks
        const uint64_t m = stage_misses(ctx, ids, slots.p, n, ctx->stage_ids, lstream(ctx));
        ctx->stage_rows.reserve(std::max<uint64_t>(m * f->row_bytes, 16));
        ctx->stage_ids.reserve(1);
        fetch_rows(f, ctx->stage_ids.p, m, ctx->stage_rows.p, lstream(ctx));
        store = ctx->stage_rows.p;
    }
    launch_gather_resolved(ctx, ids, slots.p, n, cache_rows, store, f->row_bytes, out, counters, nullptr, 0,
                           staged_backing(f));
}

void launch_apply_slots(gx_ctx* ctx, const uint32_t* in_ids, const uint32_t* in_pos, const uint32_t* in_slot,
                        uint32_t n_in, const uint32_t* out_ids, uint32_t n_out, int32_t* table,
                        const uint8_t* batch, uint8_t* cache_rows, uint64_t row_bytes) {
    const uint32_t m = std::max(n_in, n_out);
    if (!m) return;
    const unsigned blocks = (unsigned)std::min<uint64_t>(((uint64_t)m * 32 + 255) / 256, ctx->num_sms * 8);
    if (vec16(row_bytes))
        k_apply_slots<16><<<blocks, 256, 0, lstream(ctx)>>>(in_ids, in_pos, in_slot, n_in, out_ids, n_out, table,
                                                           batch, cache_rows, row_bytes);
    else
        k_apply_slots<4><<<blocks, 256, 0, lstream(ctx)>>>(in_ids, in_pos, in_slot, n_in, out_ids, n_out, table,
                                                          batch, cache_rows, row_bytes);
    GX_CHECK_LAUNCH();
}

// FeatureCache ctor prefetch (feature_cache.hpp:30-36): cache slot k <- row
// init[k] of the store, i.e. an all-miss gather into the slot array (the TMA
// gather kernel), plus the address table when the caller keeps one.
__global__ void k_set_table(const uint32_t* __restrict__ init, uint32_t n, int32_t* table) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        table[init[k]] = (int32_t)k;
}

// Per-iteration miss and page counts of a resolved access list (slot kNever =
// miss; a miss charges page_count_for_row, feature_cache.hpp:66-71): grid
// (chunks, iterations), one block reduction and two atomics per block.
__global__ void k_count_iter_misses(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ slots,
                                    const uint32_t* __restrict__ off, uint32_t S, uint64_t rb,
                                    unsigned long long* __restrict__ counters) {
    __shared__ unsigned long long red[2][32];
    for (uint32_t i = blockIdx.y; i < S; i += gridDim.y) {
        unsigned long long m = 0, pg = 0;
        for (uint32_t x = off[i] + blockIdx.x * blockDim.x + threadIdx.x; x < off[i + 1]; x += gridDim.x * blockDim.x) {
            if (__ldg(slots + x) == kNever) {
                const uint64_t v = __ldg(ids + x);
                ++m;
                pg += pages_touched(v * rb, v * rb + rb);
            }
        }
        m = warp_sum(m);
        pg = warp_sum(pg);
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = m;
            red[1][threadIdx.x >> 5] = pg;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tm = 0, tp = 0;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) {
                tm += red[0][w];
                tp += red[1][w];
            }
            if (tm) {
                atomicAdd(&counters[8 * i + 1], tm);
                atomicAdd(&counters[8 * i + 2], tp);
            }
        }
        __syncthreads();
    }
}

void launch_count_iter_misses(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, const uint32_t* d_off,
                              uint32_t S, uint64_t maxw, uint64_t rb, unsigned long long* counters) {
    if (!S) return;
    const dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((maxw + 1023) / 1024, 16)),
                    (unsigned)std::min<uint32_t>(S, 65535));
    k_count_iter_misses<<<grid, 256, 0, lstream(ctx)>>>(ids, slots, d_off, S, rb, counters);
    GX_CHECK_LAUNCH();
}

bool launch_gather_superbatch(gx_ctx* ctx, const uint32_t* ids, const uint32_t* slots, uint64_t n,
                              const uint32_t* init, uint32_t n_init, const uint8_t* cache_rows, const uint8_t* store,
                              uint64_t rb, uint8_t* out) {
    const int budget = gather_smem_budget(rb);
    if (!vec16(rb) || 2ull * 32 * rb > (uint64_t)budget) return false;  // the caller falls back
    if (!n) return true;
    static std::mutex mu;
    static std::map<int, LaunchCfg> cfgs;  // per device
    std::lock_guard<std::mutex> lk(mu);
    LaunchCfg& cf = cfgs[ctx->device];
    if (cf.rb != rb) {
        cf.tpb = (int)std::min<uint64_t>(128, budget / (2 * rb)) & ~31;
        const int smem = cf.tpb * 2 * (int)rb;
        GX_CUDA(cudaFuncSetAttribute(k_gather_sb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cf.bps, k_gather_sb, cf.tpb, smem));
        cf.bps = std::max(cf.bps, 1);
        cf.rb = rb;
    }
    const uint64_t blocks = std::min<uint64_t>((n + cf.tpb - 1) / cf.tpb, (uint64_t)ctx->num_sms * cf.bps);
    k_gather_sb<<<(unsigned)blocks, cf.tpb, (size_t)cf.tpb * 2 * rb, lstream(ctx)>>>(
        ids, slots, (uint32_t)n, init, n_init, cache_rows, store, (uint32_t)rb, out);
    GX_CHECK_LAUNCH();
    return true;
}

// Changeset regime, device-backed table, whole superbatch resident: the switch
// fanned out to every access its init rows serve (the all-fit fan-out,
// generalised). Access x is init-served when its serving slot s = acc_slot[x]
// is an init slot still holding init[s] == trace[x] -- a slot is a copy of the
// table row (feature_cache.hpp:115-126), so an init node evicted and later
// re-inserted into its own slot serves the same bytes. Each init row is read
// once and written to its slot and to the batch rows of those accesses; the
// other accesses (misses, hits on inserted nodes) are copied from the table by
// k_gather_rest; the changesets' rows land in their slots afterwards
// (launch_apply_all), so the cache ends in the reference's state.
__device__ __forceinline__ bool init_served(uint32_t s, uint32_t v, const uint32_t* __restrict__ init,
                                            uint32_t n_init) {
    return s < n_init && __ldg(init + s) == v;
}

// rank[x] = x's index in its init slot's list (ticket of a per-slot count),
// kNever when x is not init-served
__global__ void __launch_bounds__(256) k_ifan_rank(const uint32_t* __restrict__ trace,
                                                   const uint32_t* __restrict__ acc_slot, uint32_t A,
                                                   const uint32_t* __restrict__ init, uint32_t n_init,
                                                   uint32_t* cnt, uint32_t* rank) {
    const uint64_t G = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x0 < A; x0 += 4 * G) {
        uint32_t s[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t x = x0 + j * G;
            s[j] = x < A ? __ldg(acc_slot + x) : kNever;
            v[j] = x < A ? __ldg(trace + x) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = init_served(s[j], v[j], init, n_init) ? atomicAdd(&cnt[s[j]], 1u) : kNever;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (x0 + j * G < A) rank[x0 + j * G] = v[j];
    }
}

// list[start[s] + rank[x]] = x for every init-served access (no atomics)
__global__ void __launch_bounds__(256) k_ifan_place(const uint32_t* __restrict__ acc_slot,
                                                    const uint32_t* __restrict__ rank, uint32_t A,
                                                    const uint32_t* __restrict__ start, uint32_t* list) {
    const uint64_t G = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x0 < A; x0 += 4 * G) {
        uint32_t s[4], r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t x = x0 + j * G;
            r[j] = x < A ? __ldg(rank + x) : kNever;
            s[j] = r[j] != kNever ? __ldg(acc_slot + x) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (r[j] != kNever) r[j] += __ldg(start + s[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (r[j] != kNever) list[r[j]] = (uint32_t)(x0 + j * G);
    }
}

// every access that is not init-served: its row from the table. A warp takes
// 32 consecutive accesses and copies the selected rows 4 at a time (16 bytes
// per lane per row).
__global__ void __launch_bounds__(256) k_gather_rest(const uint32_t* __restrict__ trace,
                                                     const uint32_t* __restrict__ rank, uint32_t A,
                                                     const uint8_t* __restrict__ store, uint32_t row_bytes,
                                                     uint8_t* __restrict__ out, unsigned long long* nrows) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t nvec = row_bytes / 16;
    uint32_t copied = 0;
    for (uint64_t b0 = warp * 32; b0 < A; b0 += nwarps * 32) {
        const uint64_t x = b0 + lane;
        uint32_t v = 0;
        bool rest = false;
        if (x < A) {
            v = __ldg(trace + x);
            rest = __ldg(rank + x) == kNever;
        }
        uint32_t m = __ballot_sync(0xffffffffu, rest);
        copied += __popc(m);
        while (m) {
            uint32_t q[4];
            int k = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                q[j] = 0;
                if (m) {
                    q[j] = __ffs(m) - 1;
                    m &= m - 1;
                    k = j + 1;
                }
            }
            uint32_t vq[4];  // (shuffles before the lane-dependent copy loop: rows < 512 B idle lanes)
#pragma unroll
            for (int j = 0; j < 4; ++j) vq[j] = __shfl_sync(0xffffffffu, v, q[j]);
            for (uint32_t c = lane; c < nvec; c += 32) {
                uint4 t[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < k) t[j] = ld_nc(reinterpret_cast<const uint4*>(store + (uint64_t)vq[j] * row_bytes) + c);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j < k) st_na(reinterpret_cast<uint4*>(out + (b0 + q[j]) * row_bytes) + c, t[j]);
            }
        }
    }
    if (lane == 0 && copied) atomicAdd(nrows, (unsigned long long)copied);
}

void launch_init_fan(gx_ctx* ctx, const uint32_t* trace, const uint32_t* acc_slot, uint64_t A, const uint32_t* init,
                     uint32_t n_init, const uint8_t* store, uint64_t rb, uint8_t* cache_rows, uint8_t* batch,
                     DevBuf<uint32_t>& cnt, DevBuf<uint32_t>& off, DevBuf<uint32_t>& list, DevBuf<uint32_t>& rank,
                     DevBuf<uint8_t>& tmp) {
    if (rb % 16) fail(GX_INVALID_ARGUMENT, "init fan-out needs 16-byte rows");
    if (!n_init) return;
    cudaStream_t st = lstream(ctx);
    cnt.reserve(n_init + 1);
    off.reserve(n_init + 1);
    list.reserve(std::max<uint64_t>(A, 1));
    rank.reserve(std::max<uint64_t>(A, 1));
    GX_CUDA(cudaMemsetAsync(cnt.p, 0, (n_init + 1) * sizeof(uint32_t), st));
    const unsigned g = std::min<uint64_t>((A + 1023) / 1024 + 1, (uint64_t)ctx->num_sms * 8);
    k_ifan_rank<<<g, 256, 0, st>>>(trace, acc_slot, (uint32_t)A, init, n_init, cnt.p, rank.p);
    GX_CHECK_LAUNCH();
    size_t tb = 0;
    GX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, (int)(n_init + 1), st));
    tmp.reserve(std::max<size_t>(tb, 16));
    GX_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, (int)(n_init + 1), st));
    k_ifan_place<<<g, 256, 0, st>>>(acc_slot, rank.p, (uint32_t)A, off.p, list.p);
    GX_CHECK_LAUNCH();
    // off = list starts (n_init + 1 entries); k_fan_rows reads slot s as
    // [o[s - 1], o[s]) with o[-1] = 0, i.e. o = off + 1
    launch_fan_rows(ctx, init, n_init, store, rb, cache_rows, nullptr, off.p + 1, list.p, batch);
}

void launch_gather_rest(gx_ctx* ctx, const uint32_t* trace, const uint32_t* rank, uint64_t A, const uint8_t* store,
                        uint64_t rb, uint8_t* batch, unsigned long long* nrows) {
    if (!A) return;
    const unsigned g = (unsigned)std::min<uint64_t>((A + 255) / 256, (uint64_t)ctx->num_sms * 8);
    k_gather_rest<<<g, 256, 0, lstream(ctx)>>>(trace, rank, (uint32_t)A, store, (uint32_t)rb, batch, nrows);
    GX_CHECK_LAUNCH();
}

// All changesets of a superbatch applied at once, in effect (the pipeline's
// one-launch executor; nothing reads the cache in between): a slot ends with
// the row of its LAST insert (feature_cache.hpp:114-129 applied in iteration
// order), so pass 1 records each slot's last inserting iteration (+1), pass 2
// copies only those rows (batch row o[i] + pos -> slot), pass 3 clears the
// marks. Insert k's iteration comes from the insert offsets in_off[S + 1].
__device__ __forceinline__ uint32_t iter_of_insert(const uint32_t* in_off, uint32_t S, uint32_t k) {
    uint32_t lo = 0, hi = S;  // in_off[lo] <= k < in_off[lo + 1]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(in_off + mid) <= k) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_apply_last(const uint32_t* __restrict__ in_slot, const uint32_t* __restrict__ in_off, uint32_t S,
                             uint32_t n, uint32_t* __restrict__ last) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        atomicMax(&last[__ldg(in_slot + k)], iter_of_insert(in_off, S, k) + 1);
}

template <int VEC>
__global__ void k_apply_copy(const uint32_t* __restrict__ in_pos, const uint32_t* __restrict__ in_slot,
                             const uint32_t* __restrict__ in_off, uint32_t S, uint32_t n,
                             const uint32_t* __restrict__ bat_off, const uint32_t* __restrict__ last,
                             const uint8_t* __restrict__ batch, uint8_t* __restrict__ cache_rows, uint32_t rb) {
    using V = typename VecT<VEC>::T;
    const uint32_t lane = threadIdx.x & 31, nv = rb / VEC;
    for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t i = iter_of_insert(in_off, S, k), sl = __ldg(in_slot + k);
        if (__ldg(last + sl) != i + 1) continue;  // a later iteration overwrites this slot
        const V* src = reinterpret_cast<const V*>(batch + (uint64_t)(__ldg(bat_off + i) + __ldg(in_pos + k)) * rb);
        V* dst = reinterpret_cast<V*>(cache_rows + (uint64_t)sl * rb);
        for (uint32_t c = lane; c < nv; c += 32) dst[c] = src[c];
    }
}

__global__ void k_apply_clear(const uint32_t* __restrict__ in_slot, uint32_t n, uint32_t* __restrict__ last) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        last[__ldg(in_slot + k)] = 0;
}

void launch_apply_all(gx_ctx* ctx, const uint32_t* in_pos, const uint32_t* in_slot, const uint32_t* in_off,
                      uint32_t S, uint32_t n, const uint32_t* bat_off, uint32_t* last, const uint8_t* batch,
                      uint8_t* cache_rows, uint64_t rb) {
    if (!n) return;
    const unsigned g = std::min<unsigned>((n + 255) / 256, ctx->num_sms * 8);
    k_apply_last<<<g, 256, 0, lstream(ctx)>>>(in_slot, in_off, S, n, last);
    GX_CHECK_LAUNCH();
    const unsigned gw = std::min<unsigned>((n + 7) / 8, ctx->num_sms * 16);  // a warp per insert
    if (vec16(rb))
        k_apply_copy<16><<<gw, 256, 0, lstream(ctx)>>>(in_pos, in_slot, in_off, S, n, bat_off, last, batch, cache_rows,
                                                      (uint32_t)rb);
    else
        k_apply_copy<4><<<gw, 256, 0, lstream(ctx)>>>(in_pos, in_slot, in_off, S, n, bat_off, last, batch, cache_rows,
                                                     (uint32_t)rb);
    GX_CHECK_LAUNCH();
    k_apply_clear<<<g, 256, 0, lstream(ctx)>>>(in_slot, n, last);
    GX_CHECK_LAUNCH();
}

void launch_cache_init(gx_ctx* ctx, const uint32_t* init, uint32_t n, int32_t* table, gx_features* f,
                       uint8_t* cache_rows, unsigned long long* counters) {
    if (staged_backing(f)) {
        // the storage tier / the owners write the init rows straight into their slots
        fetch_rows(f, init, n, cache_rows, lstream(ctx));
    } else if (!n) {
        return;
    } else if (vec16(f->row_bytes)) {
        // one large all-miss gather: the 8-rows-per-warp LDG/STG kernel measured
        // faster than the bulk-copy kernel here (1.05 vs 1.35 ms, 6.2M x 512 B rows)
        gather_rows_launch<16, 8>(ctx, init, nullptr, n, nullptr, f->rows_dev_view, f->row_bytes, cache_rows,
                                  counters);
    } else {
        launch_gather_resolved(ctx, init, nullptr, n, nullptr, f->rows_dev_view, f->row_bytes, cache_rows, counters);
    }
    if (table) {
        k_set_table<<<ctx->num_sms * 4, 256, 0, lstream(ctx)>>>(init, n, table);
        GX_CHECK_LAUNCH();
    }
}

void launch_reset_table(gx_ctx* ctx, const uint32_t* nodes, uint64_t n, int32_t* table) {
    if (!n) return;
    k_reset_table<<<ctx->num_sms * 4, 256, 0, lstream(ctx)>>>(nodes, n, table);
    GX_CHECK_LAUNCH();
}

static void upload_u32(gx_ctx* ctx, gx::DevBuf<uint32_t>& buf, uint64_t off, const uint64_t* h, uint64_t n) {
    if (!n) return;
    std::vector<uint32_t> t(n);
    for (uint64_t i = 0; i < n; ++i) t[i] = (uint32_t)h[i];
    GX_CUDA(cudaMemcpyAsync(buf.p + off, t.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    GX_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_batch_create(gx_ctx* ctx, gx_batch** out) {
    return guard([&] {
        auto b = new gx_batch();
        b->ctx = ctx;
        *out = b;
    });
}
void gx_batch_destroy(gx_batch* b) { delete b; }
uint64_t gx_batch_rows(const gx_batch* b) { return b ? b->rows : 0; }
void* gx_batch_device_ptr(const gx_batch* b) { return b ? b->data.p : nullptr; }
gx_status gx_batch_upload(gx_batch* b, const void* rows, uint64_t n, uint64_t row_bytes) {
    return guard([&] {
        b->rows = n;
        b->row_bytes = row_bytes;
        b->data.reserve(std::max<uint64_t>(n * row_bytes, 16));
        if (n) GX_CUDA(cudaMemcpy(b->data.p, rows, n * row_bytes, cudaMemcpyHostToDevice));
    });
}

gx_status gx_batch_copy_to_host(const gx_batch* b, void* out) {
    return guard([&] {
        if (b->rows) GX_CUDA(cudaMemcpy(out, b->data.p, b->rows * b->row_bytes, cudaMemcpyDeviceToHost));
    });
}

gx_status gx_cache_create(gx_features* f, const uint64_t* init, uint64_t n_init, uint64_t K, gx_iostats* io,
                          gx_cache** out) {
    return guard([&] {
        if (n_init > K) fail(GX_INVALID_ARGUMENT, "init set larger than feature cache capacity");
        // reference order (feature_cache.hpp:30-36): per id, range then duplicate
        {
            std::vector<uint8_t> seen;
            std::vector<uint64_t> sorted;
            for (uint64_t k = 0; k < n_init; ++k)
                if (init[k] >= f->n) {
                    // a duplicate strictly before the first out-of-range id wins
                    std::vector<uint64_t> pre(init, init + k);
                    std::sort(pre.begin(), pre.end());
                    if (std::adjacent_find(pre.begin(), pre.end()) != pre.end())
                        fail(GX_INVALID_ARGUMENT, "duplicate init id");
                    fail(GX_OUT_OF_RANGE, "init id out of range");
                }
            sorted.assign(init, init + n_init);
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                fail(GX_INVALID_ARGUMENT, "duplicate init id");
        }
        if (K >= 0x7FFFFFFFull) fail(GX_INVALID_ARGUMENT, "cache capacity exceeds 2^31 - 1 slots");
        if (!f->ctx) fail(GX_INVALID_ARGUMENT, "feature table was opened without a context");
        gx_ctx* ctx = f->ctx;
        auto c = new gx_cache();
        try {
            c->f = f;
            c->ctx = ctx;
            c->K = K;
            c->rows.alloc(std::max<uint64_t>(K * f->row_bytes, 16));
            c->table.alloc(std::max<uint64_t>(f->n, 1));
            GX_CUDA(cudaMemsetAsync(c->table.p, 0xff, std::max<uint64_t>(f->n, 1) * 4, ctx->stream));
            c->free_list.alloc(std::max<uint64_t>(K, 1));
            c->free_top = K - n_init;
            if (c->free_top)
                k_iota_desc<<<ctx->num_sms, 256, 0, ctx->stream>>>(c->free_list.p, c->free_top, K);
            GX_CHECK_LAUNCH();
            c->counters.alloc(8);
            c->err.alloc(1);
            c->scratch.alloc(std::max<uint64_t>(n_init, 1));
            upload_u32(ctx, c->scratch, 0, init, n_init);
            GX_CUDA(cudaMemsetAsync(c->counters.p, 0, 8 * 8, ctx->stream));
            launch_cache_init(ctx, c->scratch.p, (uint32_t)n_init, c->table.p, f, c->rows.p, c->counters.p);
            unsigned long long pg = 0;
            GX_CUDA(cudaMemcpyAsync(&pg, c->counters.p + 2, 8, cudaMemcpyDeviceToHost, ctx->stream));
            GX_CUDA(cudaStreamSynchronize(ctx->stream));
            if (staged_backing(f)) {  // the staged tiers do not run the gather's counters
                pg = 0;
                for (uint64_t k = 0; k < n_init; ++k)
                    pg += pages_touched(init[k] * f->row_bytes, init[k] * f->row_bytes + f->row_bytes);
            }
            if (io) {
                io->rows_read += n_init;
                io->pages_read += pg;
                io->bytes_read += n_init * f->row_bytes;
            }
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void gx_cache_destroy(gx_cache* c) { delete c; }
uint64_t gx_cache_num_entries(const gx_cache* c) { return c ? c->K : 0; }

gx_status gx_cache_gather(gx_cache* c, const uint64_t* ids, uint64_t n, gx_batch* out, uint64_t* hits,
                          uint64_t* misses, gx_iostats* io) {
    return guard([&] {
        gx_ctx* ctx = c->ctx;
        for (uint64_t k = 0; k < n; ++k)
            if (ids[k] >= c->f->n) fail(GX_OUT_OF_RANGE, "gather id out of range");
        c->scratch.reserve(std::max<uint64_t>(n, 1));
        upload_u32(ctx, c->scratch, 0, ids, n);
        out->ctx = ctx;
        out->rows = n;
        out->row_bytes = c->f->row_bytes;
        out->data.reserve(std::max<uint64_t>(n * c->f->row_bytes, 16));
        GX_CUDA(cudaMemsetAsync(c->counters.p, 0, 8 * 8, ctx->stream));
        launch_gather(ctx, c->scratch.p, n, c->table.p, c->rows.p, c->f, out->data.p, c->counters.p);
        unsigned long long cnt[5];
        GX_CUDA(cudaMemcpyAsync(cnt, c->counters.p, 5 * 8, cudaMemcpyDeviceToHost, ctx->stream));
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (hits) *hits = cnt[0];
        if (misses) *misses = cnt[1];
        if (io) {
            io->pages_read += cnt[2];
            io->rows_read += cnt[3];
            io->bytes_read += cnt[4];
        }
    });
}

gx_status gx_cache_apply(gx_cache* c, const gx_batch* batch, const uint64_t* ids, uint64_t n_ids,
                         const uint64_t* in_ids, const uint64_t* in_pos, uint64_t n_in, const uint64_t* out_ids,
                         uint64_t n_out) {
    return guard([&] {
        gx_ctx* ctx = c->ctx;
        if (!batch || batch->rows != n_ids || (n_ids && batch->row_bytes != c->f->row_bytes))
            fail(GX_INVALID_ARGUMENT, "batch buffer does not match ids");
        // stage ids | in_ids | in_pos | out_ids as u32 (positions beyond u32 are invalid anyway)
        for (uint64_t k = 0; k < n_in; ++k)
            if (in_pos[k] >= n_ids) fail(GX_LOGIC_ERROR, "changeset position does not match ids");
        for (uint64_t k = 0; k < n_out; ++k)
            if (out_ids[k] >= c->f->n) fail(GX_LOGIC_ERROR, "evicted node is not cached");
        for (uint64_t k = 0; k < n_in; ++k)
            if (in_ids[k] >= c->f->n) fail(GX_LOGIC_ERROR, "changeset position does not match ids");
        // duplicate ids inside the changeset take the exact sequential replay
        // (k_apply_serial); the parallel kernel assumes distinct in and out ids
        auto has_dup = [](const uint64_t* v, uint64_t n) {
            if (n < 2) return false;
            std::vector<uint64_t> t(v, v + n);
            std::sort(t.begin(), t.end());
            return std::adjacent_find(t.begin(), t.end()) != t.end();
        };
        const bool dup = has_dup(in_ids, n_in) || has_dup(out_ids, n_out);
        const uint64_t tot = n_ids + 2 * n_in + n_out + (dup ? n_out : 0);
        c->scratch.reserve(std::max<uint64_t>(tot, 1));
        upload_u32(ctx, c->scratch, 0, ids, n_ids);
        upload_u32(ctx, c->scratch, n_ids, in_ids, n_in);
        upload_u32(ctx, c->scratch, n_ids + n_in, in_pos, n_in);
        upload_u32(ctx, c->scratch, n_ids + 2 * n_in, out_ids, n_out);
        const uint32_t* d_ids = c->scratch.p;
        const uint32_t* d_in = c->scratch.p + n_ids;
        const uint32_t* d_pos = c->scratch.p + n_ids + n_in;
        const uint32_t* d_out = c->scratch.p + n_ids + 2 * n_in;
        GX_CUDA(cudaMemsetAsync(c->err.p, 0, 4, ctx->stream));
        if (n_in || n_out) {
            k_apply_validate<<<ctx->num_sms, 256, 0, ctx->stream>>>(d_ids, (uint32_t)n_ids, d_in, d_pos,
                                                                    (uint32_t)n_in, d_out, (uint32_t)n_out,
                                                                    c->table.p, c->f->n, c->err.p);
            GX_CHECK_LAUNCH();
        }
        unsigned int e = 0;
        GX_CUDA(cudaMemcpyAsync(&e, c->err.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (e) fail(GX_LOGIC_ERROR, "invalid changeset for the current cache state");
        if (n_in > n_out + c->free_top) fail(GX_LOGIC_ERROR, "changeset overflows cache capacity");
        const uint32_t m = (uint32_t)std::max(n_in, n_out);
        if (m && dup) {
            uint32_t* freed = c->scratch.p + n_ids + 2 * n_in + n_out;
            if (vec16(c->f->row_bytes))
                k_apply_serial<16><<<1, 32, 0, ctx->stream>>>(d_in, d_pos, (uint32_t)n_in, d_out, (uint32_t)n_out,
                                                             c->table.p, c->free_list.p, c->free_top, batch->data.p,
                                                             c->rows.p, c->f->row_bytes, freed);
            else
                k_apply_serial<4><<<1, 32, 0, ctx->stream>>>(d_in, d_pos, (uint32_t)n_in, d_out, (uint32_t)n_out,
                                                            c->table.p, c->free_list.p, c->free_top, batch->data.p,
                                                            c->rows.p, c->f->row_bytes, freed);
            GX_CHECK_LAUNCH();
        } else if (m) {
            const unsigned blocks = (unsigned)std::min<uint64_t>(((uint64_t)m * 32 + 255) / 256, ctx->num_sms * 8);
            if (vec16(c->f->row_bytes))
                k_apply<16><<<blocks, 256, 0, ctx->stream>>>(d_in, d_pos, (uint32_t)n_in, d_out, (uint32_t)n_out,
                                                             c->table.p, c->free_list.p, c->free_top,
                                                             batch->data.p, c->rows.p, c->f->row_bytes);
            else
                k_apply<4><<<blocks, 256, 0, ctx->stream>>>(d_in, d_pos, (uint32_t)n_in, d_out, (uint32_t)n_out,
                                                            c->table.p, c->free_list.p, c->free_top,
                                                            batch->data.p, c->rows.p, c->f->row_bytes);
            GX_CHECK_LAUNCH();
        }
        if (n_in > n_out) c->free_top -= (n_in - n_out);
        else c->free_top += (n_out - n_in);
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

gx_status gx_cache_contains(const gx_cache* c, uint64_t v, int* out) {
    return guard([&] {
        if (v >= c->f->n) fail(GX_OUT_OF_RANGE, "node id out of range");
        int32_t s;
        GX_CUDA(cudaMemcpy(&s, c->table.p + v, 4, cudaMemcpyDeviceToHost));
        *out = s >= 0;
    });
}

gx_status gx_cache_cached_row(const gx_cache* c, uint64_t v, void* out) {
    return guard([&] {
        if (v >= c->f->n) fail(GX_OUT_OF_RANGE, "node id out of range");
        int32_t s;
        GX_CUDA(cudaMemcpy(&s, c->table.p + v, 4, cudaMemcpyDeviceToHost));
        if (s < 0) fail(GX_LOGIC_ERROR, "cached_row on a miss");
        GX_CUDA(cudaMemcpy(out, c->rows.p + (uint64_t)s * c->f->row_bytes, c->f->row_bytes,
                           cudaMemcpyDeviceToHost));
    });
}

gx_status gx_cache_resident_set(const gx_cache* c, uint64_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        gx_ctx* ctx = c->ctx;
        // more residents than slots is possible after a changeset with
        // duplicate out ids (two nodes share a freed slot, as in the reference):
        // size by the count and retry once
        uint64_t cap = std::max<uint64_t>(c->K, 1);
        DevBuf<uint32_t> tmp(cap);
        DevBuf<unsigned int> cnt(1);
        unsigned int hc = 0;
        for (int pass = 0; pass < 2; ++pass) {
            GX_CUDA(cudaMemsetAsync(cnt.p, 0, 4, ctx->stream));
            k_resident<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(c->table.p, c->f->n, tmp.p, cap, cnt.p);
            GX_CHECK_LAUNCH();
            GX_CUDA(cudaMemcpyAsync(&hc, cnt.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
            GX_CUDA(cudaStreamSynchronize(ctx->stream));
            if (hc <= cap) break;
            cap = hc;
            tmp.alloc(cap);
        }
        std::vector<uint32_t> h(hc);
        if (hc) GX_CUDA(cudaMemcpy(h.data(), tmp.p, hc * 4, cudaMemcpyDeviceToHost));
        std::sort(h.begin(), h.end());
        *n = hc;
        for (uint64_t i = 0; i < hc && i < cap; ++i) out[i] = h[i];
    });
}

gx_status gx_features_read_rows(gx_features* f, const uint64_t* ids, uint64_t n, void* out, gx_iostats* io) {
    return guard([&] {
        gx_ctx* ctx = f->ctx;
        for (uint64_t k = 0; k < n; ++k)
            if (ids[k] >= f->n) fail(GX_OUT_OF_RANGE, "feature row id out of range");
        if (f->backing == GX_BACKING_PARTITIONED)
            fail(GX_INVALID_ARGUMENT, "read_rows on a partitioned table: rows are served collectively (cache/pipeline)");
        if (f->backing == GX_BACKING_FILE) {  // straight from storage into the caller's buffer
            f->file->read_rows(ids, n, (uint8_t*)out);
            if (io) {
                for (uint64_t k = 0; k < n; ++k)
                    io->pages_read += pages_touched(ids[k] * f->row_bytes, ids[k] * f->row_bytes + f->row_bytes);
                io->rows_read += n;
                io->bytes_read += n * f->row_bytes;
            }
            return;
        }
        DevBuf<uint32_t> d(std::max<uint64_t>(n, 1));
        upload_u32(ctx, d, 0, ids, n);
        DevBuf<uint8_t> o(std::max<uint64_t>(n * f->row_bytes, 16));
        DevBuf<unsigned long long> cnt(8);
        GX_CUDA(cudaMemsetAsync(cnt.p, 0, 64, ctx->stream));
        // every row is a backing-store read: the all-miss form (no slots, no
        // address table), charging pages like FeatureFile::read_row
        const cudaStream_t saved = ctx->launch_stream;
        ctx->launch_stream = nullptr;
        launch_gather_resolved(ctx, d.p, nullptr, n, nullptr, f->rows_dev_view, f->row_bytes, o.p, cnt.p);
        ctx->launch_stream = saved;
        unsigned long long h[5];
        GX_CUDA(cudaMemcpyAsync(h, cnt.p, 40, cudaMemcpyDeviceToHost, ctx->stream));
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
        if (n) GX_CUDA(cudaMemcpy(out, o.p, n * f->row_bytes, cudaMemcpyDeviceToHost));
        if (io) {
            io->pages_read += h[2];
            io->rows_read += h[3];
            io->bytes_read += h[4];
        }
    });
}

}  // extern "C"
