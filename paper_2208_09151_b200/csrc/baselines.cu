// baselines.cu -- comparison cache policies of `gx simulate` (baselines.hpp).
//
// simulate_policy (baselines.hpp:64-143) over a trace of S distinct-id lists:
//  * none          every access misses;
//  * static_degree a fixed resident set: the K nodes of highest out-degree,
//                  ties by lower id (static_degree_set, baselines.hpp:50-62) --
//                  out-degrees by a histogram over the CSC indices, the set by
//                  a stable CUB radix sort of (~degree, id), misses by a
//                  per-iteration count of non-resident ids;
//  * belady        the inspector (precompute over the same trace);
//  * lru           (baselines.hpp:104-128) as LRU stack distances: access t of
//                  node v, previous access p, hits iff fewer than K distinct
//                  nodes were accessed in (p, t). That count is
//                  D(t) = t - p - 1 - C(t), C(t) = #{u < t : prev[u] > p}
//                  (every access in (p, t) whose own previous access also lies
//                  in (p, t) repeats a node already counted), and C is a
//                  per-element inversion count over prev[] -- a bottom-up merge
//                  sort whose merge step adds, for each element of a right run,
//                  the left-run elements above it. prev[] comes from a stable
//                  CUB radix sort of (node, time). Exact for any trace (also
//                  repeats inside one list, which the reference counts as hits).
#include <cub/cub.cuh>

#include "gx_internal.cuh"

namespace gx {

__global__ void k_outdeg_hist(const uint32_t* __restrict__ indices, uint64_t E, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&out[indices[i]], 1u);
}

__global__ void k_deg_keys(const uint32_t* __restrict__ deg, uint64_t n, uint32_t* __restrict__ keys,
                           uint32_t* __restrict__ ids) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        keys[v] = ~deg[v];  // descending degree; the stable sort keeps ids ascending within a degree
        ids[v] = (uint32_t)v;
    }
}

__global__ void k_mark(const uint32_t* __restrict__ ids, uint64_t k, uint32_t* __restrict__ bits) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
        atomicOr(&bits[ids[i] >> 5], 1u << (ids[i] & 31));
}

// misses[i] = |{x in list i : not resident}|; err bit 1: an id >= N
__global__ void k_count_misses(const uint32_t* __restrict__ trace, const uint64_t* __restrict__ off, uint32_t S,
                               uint64_t N, const uint32_t* __restrict__ bits, unsigned long long* __restrict__ misses,
                               unsigned int* err) {
    for (uint32_t i = blockIdx.y; i < S; i += gridDim.y) {
        unsigned long long c = 0;
        for (uint64_t x = off[i] + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < off[i + 1];
             x += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t v = trace[x];
            if (v >= N) {
                atomicOr(err, 1u);
                continue;
            }
            if (!((bits[v >> 5] >> (v & 31)) & 1u)) ++c;
        }
        c = warp_sum(c);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&misses[i], c);
    }
}

// prev1[t] = 1 + previous access time of the same node, 0 = first access
__global__ void k_lru_prev(const uint32_t* __restrict__ node_sorted, const uint32_t* __restrict__ time_sorted,
                           uint64_t A, uint32_t* __restrict__ prev1) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < A; s += (uint64_t)gridDim.x * blockDim.x)
        prev1[time_sorted[s]] = (s > 0 && node_sorted[s - 1] == node_sorted[s]) ? time_sorted[s - 1] + 1 : 0u;
}

__global__ void k_lru_pack(const uint32_t* __restrict__ prev1, uint64_t A, unsigned long long* __restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < A; t += (uint64_t)gridDim.x * blockDim.x)
        out[t] = ((unsigned long long)prev1[t] << 32) | t;
}

// number of x in sorted run [p, p + n) with x < key
__device__ __forceinline__ uint64_t count_below(const unsigned long long* __restrict__ p, uint64_t n,
                                                unsigned long long key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (p[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// one merge level of width w over packed (prev1 << 32 | time) keys (all
// distinct): every element lands at its merged position; a right-run element
// adds the left-run elements with a larger prev1 to C[time]
__global__ void k_lru_merge(const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out,
                            uint64_t A, uint64_t w, uint32_t* __restrict__ C) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < A; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t base = i / (2 * w) * (2 * w);
        const uint64_t lmid = min(base + w, A), rend = min(base + 2 * w, A);
        const unsigned long long x = in[i];
        uint64_t pos;
        if (i < lmid) {
            pos = base + (i - base) + count_below(in + lmid, rend - lmid, x);
        } else {
            const uint64_t nl = lmid - base;
            pos = base + (i - lmid) + count_below(in + base, nl, x);
            const uint32_t v = (uint32_t)(x >> 32);
            if (v) {  // a repeat: left elements with prev1 > v (keys >= (v + 1) << 32)
                const uint64_t le = count_below(in + base, nl, (unsigned long long)(v + 1) << 32);
                C[(uint32_t)x] += (uint32_t)(nl - le);
            }
        }
        out[pos] = x;
    }
}

__global__ void k_lru_misses(const uint32_t* __restrict__ prev1, const uint32_t* __restrict__ C,
                             const uint64_t* __restrict__ off, uint32_t S, uint64_t K,
                             unsigned long long* __restrict__ misses) {
    for (uint32_t i = blockIdx.y; i < S; i += gridDim.y) {
        unsigned long long c = 0;
        for (uint64_t t = off[i] + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < off[i + 1];
             t += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t p1 = prev1[t];
            const bool hit = p1 && (t - p1 - C[t]) < K;  // distinct nodes in (p, t) = t - p - 1 - C
            c += hit ? 0 : 1;
        }
        c = warp_sum(c);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&misses[i], c);
    }
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_static_degree_set(gx_graph* g, uint64_t K, uint64_t* out) {
    return guard([&] {
        if (!g) fail(GX_INVALID_ARGUMENT, "null graph");
        require_whole_csc(g, "static_degree policy");
        const uint64_t n = g->n;
        if (K > n) fail(GX_INVALID_ARGUMENT, "static set larger than node count");
        gx_ctx* ctx = g->ctx;
        cudaStream_t st = ctx->stream;
        const unsigned grid = ctx->num_sms * 4;
        DevBuf<uint32_t> deg(n + 1), keys(n + 1), keys2(n + 1), ids(n + 1), ids2(n + 1);
        GX_CUDA(cudaMemsetAsync(deg.p, 0, (n + 1) * 4, st));
        if (g->e) {
            k_outdeg_hist<<<grid, 256, 0, st>>>(g->indices.p, g->e, deg.p);
            GX_CHECK_LAUNCH();
        }
        if (n) {
            k_deg_keys<<<grid, 256, 0, st>>>(deg.p, n, keys.p, ids.p);
            GX_CHECK_LAUNCH();
        }
        cub::DoubleBuffer<uint32_t> dk(keys.p, keys2.p), dv(ids.p, ids2.p);
        size_t tb = 0;
        GX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, 32, st));
        DevBuf<uint8_t> tmp(tb + 16);
        GX_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)n, 0, 32, st));
        std::vector<uint32_t> h(K);
        if (K) GX_CUDA(cudaMemcpyAsync(h.data(), dv.Current(), K * 4, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < K; ++i) out[i] = h[i];
    });
}

gx_status gx_simulate_static_degree(gx_graph* g, const uint64_t* ids_flat, const uint64_t* offsets, uint64_t S,
                                    uint64_t K, uint64_t* misses) {
    return guard([&] {
        if (!g) fail(GX_INVALID_ARGUMENT, "null graph");
        require_whole_csc(g, "static_degree policy");
        const uint64_t n = g->n;
        if (K > n) fail(GX_INVALID_ARGUMENT, "static set larger than node count");
        gx_ctx* ctx = g->ctx;
        cudaStream_t st = ctx->stream;
        std::vector<uint64_t> set(K);
        const gx_status s = gx_static_degree_set(g, K, set.data());
        if (s != GX_OK) fail(s, gx_last_error());
        const uint64_t A = S ? offsets[S] : 0;
        DevBuf<uint32_t> bits((n + 31) / 32 + 1), dset(std::max<uint64_t>(K, 1)), trace(std::max<uint64_t>(A, 1));
        DevBuf<uint64_t> doff(S + 1);
        DevBuf<unsigned long long> dm(std::max<uint64_t>(S, 1));
        DevBuf<unsigned int> err(1);
        std::vector<uint32_t> h32(std::max(K, A));
        for (uint64_t i = 0; i < K; ++i) h32[i] = (uint32_t)set[i];
        GX_CUDA(cudaMemsetAsync(bits.p, 0, bits.bytes(), st));
        if (K) GX_CUDA(cudaMemcpyAsync(dset.p, h32.data(), K * 4, cudaMemcpyHostToDevice, st));
        if (K) {
            k_mark<<<ctx->num_sms, 256, 0, st>>>(dset.p, K, bits.p);
            GX_CHECK_LAUNCH();
        }
        GX_CUDA(cudaStreamSynchronize(st));
        bool bad = false;
        for (uint64_t x = 0; x < A; ++x) {
            if (ids_flat[x] >= n) bad = true;
            h32[x] = (uint32_t)std::min<uint64_t>(ids_flat[x], 0xFFFFFFFFull);
        }
        if (bad) fail(GX_OUT_OF_RANGE, "trace id out of range");
        if (A) GX_CUDA(cudaMemcpyAsync(trace.p, h32.data(), A * 4, cudaMemcpyHostToDevice, st));
        if (S) GX_CUDA(cudaMemcpyAsync(doff.p, offsets, (S + 1) * 8, cudaMemcpyHostToDevice, st));
        GX_CUDA(cudaMemsetAsync(dm.p, 0, std::max<uint64_t>(S, 1) * 8, st));
        GX_CUDA(cudaMemsetAsync(err.p, 0, 4, st));
        if (S && A) {
            dim3 grid(16, (unsigned)std::min<uint64_t>(S, 65535));
            k_count_misses<<<grid, 256, 0, st>>>(trace.p, doff.p, (uint32_t)S, n, bits.p, dm.p, err.p);
            GX_CHECK_LAUNCH();
        }
        std::vector<unsigned long long> hm(std::max<uint64_t>(S, 1));
        unsigned int he = 0;
        GX_CUDA(cudaMemcpyAsync(hm.data(), dm.p, std::max<uint64_t>(S, 1) * 8, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaMemcpyAsync(&he, err.p, 4, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        if (he) fail(GX_OUT_OF_RANGE, "trace id out of range");
        for (uint64_t i = 0; i < S; ++i) misses[i] = hm[i];
    });
}

gx_status gx_simulate_lru(gx_ctx* ctx, const uint64_t* ids_flat, const uint64_t* offsets, uint64_t S, uint64_t N,
                          uint64_t K, uint64_t* misses) {
    return guard([&] {
        if (!ctx) fail(GX_INVALID_ARGUMENT, "null context");
        const uint64_t A = S ? offsets[S] : 0;
        if (A >= 0xFFFFFFFFull) fail(GX_INVALID_ARGUMENT, "trace longer than 2^32 - 1 accesses");
        std::vector<uint32_t> h32(std::max<uint64_t>(A, 1));
        for (uint64_t x = 0; x < A; ++x) {
            if (ids_flat[x] >= N) fail(GX_OUT_OF_RANGE, "trace id out of range");
            h32[x] = (uint32_t)ids_flat[x];
        }
        for (uint64_t i = 0; i < S; ++i) misses[i] = 0;
        if (!A) return;
        cudaStream_t st = ctx->stream;
        const unsigned grid = ctx->num_sms * 8;
        DevBuf<uint32_t> node(A), node2(A), tm(A), tm2(A), prev1(A), C(A);
        DevBuf<unsigned long long> ka(A), kb(A);
        DevBuf<uint64_t> doff(S + 1);
        DevBuf<unsigned long long> dm(S);
        GX_CUDA(cudaMemcpyAsync(node.p, h32.data(), A * 4, cudaMemcpyHostToDevice, st));
        for (uint64_t x = 0; x < A; ++x) h32[x] = (uint32_t)x;
        GX_CUDA(cudaMemcpyAsync(tm.p, h32.data(), A * 4, cudaMemcpyHostToDevice, st));
        GX_CUDA(cudaMemcpyAsync(doff.p, offsets, (S + 1) * 8, cudaMemcpyHostToDevice, st));
        int bits = 1;
        while (bits < 32 && (1ull << bits) < N) ++bits;
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, node.p, node2.p, tm.p, tm2.p, (int64_t)A, 0, bits, st);
        DevBuf<uint8_t> tmp(std::max<size_t>(tmp_bytes, 1));
        GX_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, node.p, node2.p, tm.p, tm2.p, (int64_t)A, 0, bits,
                                                st));
        k_lru_prev<<<grid, 256, 0, st>>>(node2.p, tm2.p, A, prev1.p);
        GX_CHECK_LAUNCH();
        k_lru_pack<<<grid, 256, 0, st>>>(prev1.p, A, ka.p);
        GX_CHECK_LAUNCH();
        GX_CUDA(cudaMemsetAsync(C.p, 0, A * 4, st));
        unsigned long long *in = ka.p, *out = kb.p;
        for (uint64_t w = 1; w < A; w <<= 1) {
            k_lru_merge<<<grid, 256, 0, st>>>(in, out, A, w, C.p);
            GX_CHECK_LAUNCH();
            std::swap(in, out);
        }
        GX_CUDA(cudaMemsetAsync(dm.p, 0, S * 8, st));
        dim3 g2(16, (unsigned)std::min<uint64_t>(S, 65535));
        k_lru_misses<<<g2, 256, 0, st>>>(prev1.p, C.p, doff.p, (uint32_t)S, K, dm.p);
        GX_CHECK_LAUNCH();
        std::vector<unsigned long long> hm(S);
        GX_CUDA(cudaMemcpyAsync(hm.data(), dm.p, S * 8, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < S; ++i) misses[i] = hm[i];
    });
}

}  // extern "C"
