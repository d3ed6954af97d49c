// ncache.cu -- the static neighbor cache (neighbor_cache.hpp) on the device.
//
// In the reference the cache holds in-neighbour lists in host memory so the
// sampler skips their preads; the sampled output never changes, only IoStats
// (a cached list charges nothing, sampler.hpp:91-97). Here the CSC is already
// HBM-resident, so the cache is a per-node bit the sampler consults when it
// charges IoStats, plus the reference's address_table / cache_array for the
// byte-exact ncache.bin (persist/load, neighbor_cache.hpp:118-148).
//
// build_neighbor_cache (neighbor_cache.hpp:88-116) on the device:
//   out-degrees: a histogram over the CSC indices (compute_out_degrees);
//   score = out/in (in-degree 0 excluded); order = score descending, id
//   ascending -- a stable CUB radix sort of (~bits(score), id) over the ids in
//   ascending order; greedy admission within the byte budget with skipping:
//   chunks that fit whole are admitted by a block scan, the tail by one warp
//   (ballot over 32 candidates against the remaining budget, which only
//   shrinks); regions = [count, neighbours...] laid out in admission order.
#include <cub/cub.cuh>

#include "gx_internal.cuh"

struct gx_ncache {
    gx_ctx* ctx = nullptr;
    uint64_t n = 0;
    uint64_t n_cells = 0, n_cached = 0;
    gx::DevBuf<uint32_t> bits;     // (n + 31) / 32 words: bit v = node v cached
    gx::DevBuf<int64_t> addr;      // address_table (i64, -1 = miss)
    gx::DevBuf<uint64_t> cells;    // cache_array
};

namespace gx {

static const char kNcMagic[8] = {'G', 'X', 'N', 'C', 'A', 'C', 'H', '1'};

__global__ void k_out_degree(const uint32_t* __restrict__ indices, uint64_t E, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&out[indices[i]], 1u);
}

// key = ~bits(out/in) (non-negative doubles order like their bit patterns, so
// the complement sorts descending); in-degree 0 -> excluded (key = ~0, last)
__global__ void k_score_keys(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ outdeg, uint64_t n,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ ids,
                             unsigned int* __restrict__ n_elig) {
    uint32_t c = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t in = indptr[v + 1] - indptr[v];
        unsigned long long k = ~0ull;
        if (in) {
            const double s = (double)outdeg[v] / (double)in;
            // 0 <= s: sign bit clear, so dropping the complement's top bit keeps
            // every eligible key below the excluded ones (score 0.0 included)
            k = ~(unsigned long long)__double_as_longlong(s) & 0x7FFFFFFFFFFFFFFFull;
            ++c;
        }
        keys[v] = k;
        ids[v] = (uint32_t)v;
    }
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(n_elig, c);
}

__global__ void k_region_cells(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ order, uint64_t m,
                               uint64_t* __restrict__ cells) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = order[i];
        cells[i] = 1 + indptr[v + 1] - indptr[v];
    }
}

// Greedy admission (neighbor_cache.hpp:104-114): walk the order, admit a node
// when its region fits the remaining budget, skip it otherwise. One CTA:
// while whole 1024-candidate chunks fit they are admitted by a block scan;
// from the first chunk that does not, warp 0 walks on with ballots.
__global__ void __launch_bounds__(1024) k_greedy(const uint64_t* __restrict__ cells, uint64_t m, uint64_t budget_cells,
                                                 uint8_t* __restrict__ admit, unsigned long long* out_used) {
    __shared__ unsigned long long scan[33];
    __shared__ unsigned long long s_used;
    __shared__ int s_stop;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        s_used = 0;
        s_stop = 0;
    }
    __syncthreads();
    uint64_t i0 = 0;
    for (; i0 < m; i0 += blockDim.x) {
        const uint64_t i = i0 + tid;
        const unsigned long long c = i < m ? cells[i] : 0ull;
        unsigned long long tot;
        block_excl_scan(c, scan, tot);
        const unsigned long long used = s_used;
        if (used + tot > budget_cells) break;  // uniform: every thread sees the same tot
        if (i < m) admit[i] = 1;
        __syncthreads();
        if (tid == 0) s_used = used + tot;
        __syncthreads();
    }
    __syncthreads();
    if (tid >= 32) return;
    unsigned long long left = budget_cells - s_used;
    for (uint64_t b = i0; b < m && left >= 2; b += 32) {  // a region is at least 2 cells
        const uint64_t i = b + tid;
        const unsigned long long c = i < m ? cells[i] : ~0ull;
        uint32_t decided = 0;  // lanes already visited in this group
        while (true) {
            const uint32_t fit = __ballot_sync(0xffffffffu, c <= left) & ~decided;
            if (!fit) break;
            const int lane = __ffs(fit) - 1;  // the next candidate that fits, in order
            const unsigned long long cl = __shfl_sync(0xffffffffu, c, lane);
            if (tid == (uint32_t)lane) admit[i] = 1;
            left -= cl;
            decided |= (2u << lane) - 1;  // candidates up to it are settled (smaller ones skipped)
        }
    }
    if (tid == 0) *out_used = budget_cells - left;
}

__global__ void k_fill_regions(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ indices,
                               const uint32_t* __restrict__ adm_ids, const uint64_t* __restrict__ off, uint64_t na,
                               int64_t* __restrict__ addr, uint64_t* __restrict__ cells, uint32_t* __restrict__ bits) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t k = warp; k < na; k += nw) {
        const uint32_t v = adm_ids[k];
        const uint64_t lo = indptr[v], deg = indptr[v + 1] - lo, o = off[k];
        if (lane == 0) {
            addr[v] = (int64_t)o;
            cells[o] = deg;
            atomicOr(&bits[v >> 5], 1u << (v & 31));
        }
        for (uint64_t j = lane; j < deg; j += 32) cells[o + 1 + j] = indices[lo + j];
    }
}

__global__ void k_bits_from_addr(const int64_t* __restrict__ addr, uint64_t n, uint32_t* __restrict__ bits,
                                 unsigned long long* __restrict__ cnt) {
    uint32_t c = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        if (addr[v] >= 0) {
            atomicOr(&bits[v >> 5], 1u << (v & 31));
            ++c;
        }
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

// IoStats of the admitted lists' reads (read_in_neighbors, graph_store.hpp:145-154)
__global__ void k_list_io(const uint64_t* __restrict__ indptr, const uint32_t* __restrict__ ids, uint64_t na,
                          unsigned long long* io) {
    unsigned long long pages = 0, bytes = 0;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < na; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = ids[k];
        pages += pages_touched(8 * indptr[v], 8 * indptr[v + 1]);
        bytes += 8 * (indptr[v + 1] - indptr[v]);
    }
    pages = warp_sum(pages);
    bytes = warp_sum(bytes);
    if ((threadIdx.x & 31) == 0 && (pages | bytes)) {
        atomicAdd(&io[0], pages);
        atomicAdd(&io[1], bytes);
    }
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_ncache_build(gx_graph* g, uint64_t budget_bytes, gx_iostats* io, gx_ncache** out) {
    return guard([&] {
        if (!g) fail(GX_INVALID_ARGUMENT, "null graph");
        require_whole_csc(g, "build_neighbor_cache");
        const uint64_t n = g->n, E = g->e;
        if (budget_bytes < n * 8) fail(GX_INVALID_ARGUMENT, "neighbor cache budget is smaller than the address table");
        gx_ctx* ctx = g->ctx;
        cudaStream_t st = ctx->stream;
        const unsigned grid = ctx->num_sms * 4;
        auto nc = std::make_unique<gx_ncache>();
        nc->ctx = ctx;
        nc->n = n;
        DevBuf<uint32_t> outdeg(std::max<uint64_t>(n, 1));
        GX_CUDA(cudaMemsetAsync(outdeg.p, 0, std::max<uint64_t>(n, 1) * 4, st));
        if (E) {
            k_out_degree<<<grid, 256, 0, st>>>(g->indices.p, E, outdeg.p);
            GX_CHECK_LAUNCH();
        }
        DevBuf<unsigned long long> keys(std::max<uint64_t>(n, 1)), keys2(std::max<uint64_t>(n, 1));
        DevBuf<uint32_t> ids(std::max<uint64_t>(n, 1)), ids2(std::max<uint64_t>(n, 1));
        DevBuf<unsigned int> n_elig(1);
        GX_CUDA(cudaMemsetAsync(n_elig.p, 0, 4, st));
        if (n) {
            k_score_keys<<<grid, 256, 0, st>>>(g->indptr.p, outdeg.p, n, keys.p, ids.p, n_elig.p);
            GX_CHECK_LAUNCH();
        }
        cub::DoubleBuffer<unsigned long long> dk(keys.p, keys2.p);
        cub::DoubleBuffer<uint32_t> dv(ids.p, ids2.p);
        size_t tb = 0;
        GX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, 64, st));
        DevBuf<uint8_t> tmp(tb + 16);
        GX_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, (int)n, 0, 64, st));
        unsigned int h_elig = 0;
        GX_CUDA(cudaMemcpyAsync(&h_elig, n_elig.p, 4, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        const uint64_t m = h_elig;  // eligible nodes lead the order
        const uint32_t* order = dv.Current();
        DevBuf<uint64_t> cells(std::max<uint64_t>(m, 1));
        DevBuf<uint8_t> admit(std::max<uint64_t>(m, 1));
        GX_CUDA(cudaMemsetAsync(admit.p, 0, std::max<uint64_t>(m, 1), st));
        DevBuf<unsigned long long> used(1);
        GX_CUDA(cudaMemsetAsync(used.p, 0, 8, st));
        if (m) {
            k_region_cells<<<grid, 256, 0, st>>>(g->indptr.p, order, m, cells.p);
            GX_CHECK_LAUNCH();
            k_greedy<<<1, 1024, 0, st>>>(cells.p, m, (budget_bytes - n * 8) / 8, admit.p, used.p);
            GX_CHECK_LAUNCH();
        }
        // admitted ids (admission order) and their region offsets
        DevBuf<uint32_t> adm(std::max<uint64_t>(m, 1));
        DevBuf<unsigned int> na_d(1);
        DevBuf<uint64_t> adm_cells(std::max<uint64_t>(m, 1)), off(std::max<uint64_t>(m, 1));
        size_t t2 = 0, t3 = 0, t4 = 0;
        GX_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, order, admit.p, adm.p, na_d.p, (int)m, st));
        GX_CUDA(cub::DeviceSelect::Flagged(nullptr, t3, cells.p, admit.p, adm_cells.p, na_d.p, (int)m, st));
        GX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t4, adm_cells.p, off.p, (int)m, st));
        tmp.reserve(std::max({t2, t3, t4}) + 16);
        unsigned int h_na = 0;
        unsigned long long h_used = 0;
        if (m) {
            GX_CUDA(cub::DeviceSelect::Flagged(tmp.p, t2, order, admit.p, adm.p, na_d.p, (int)m, st));
            GX_CUDA(cub::DeviceSelect::Flagged(tmp.p, t3, cells.p, admit.p, adm_cells.p, na_d.p, (int)m, st));
            GX_CUDA(cudaMemcpyAsync(&h_na, na_d.p, 4, cudaMemcpyDeviceToHost, st));
            GX_CUDA(cudaMemcpyAsync(&h_used, used.p, 8, cudaMemcpyDeviceToHost, st));
            GX_CUDA(cudaStreamSynchronize(st));
            if (h_na) GX_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, t4, adm_cells.p, off.p, (int)h_na, st));
        }
        nc->n_cached = h_na;
        nc->n_cells = h_used;
        nc->bits.alloc((n + 31) / 32 + 1);
        GX_CUDA(cudaMemsetAsync(nc->bits.p, 0, nc->bits.bytes(), st));
        nc->addr.alloc(std::max<uint64_t>(n, 1));
        GX_CUDA(cudaMemsetAsync(nc->addr.p, 0xff, std::max<uint64_t>(n, 1) * 8, st));
        nc->cells.alloc(std::max<uint64_t>(h_used, 1));
        DevBuf<unsigned long long> lio(2);
        GX_CUDA(cudaMemsetAsync(lio.p, 0, 16, st));
        if (h_na) {
            k_fill_regions<<<grid, 256, 0, st>>>(g->indptr.p, g->indices.p, adm.p, off.p, h_na, nc->addr.p,
                                                 nc->cells.p, nc->bits.p);
            GX_CHECK_LAUNCH();
            k_list_io<<<grid, 256, 0, st>>>(g->indptr.p, adm.p, h_na, lio.p);
            GX_CHECK_LAUNCH();
        }
        unsigned long long h_lio[2] = {0, 0};
        GX_CUDA(cudaMemcpyAsync(h_lio, lio.p, 16, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        if (io) {  // compute_out_degrees (graph_store.hpp:164-185) + one read per admitted list
            io->bytes_read += E * 8 + h_lio[1];
            io->pages_read += pages_touched(0, E * 8) + h_lio[0];
            io->neighbor_lists_read += h_na;
        }
        *out = nc.release();
    });
}

gx_status gx_ncache_write(const gx_ncache* c, const char* path) {
    return guard([&] {
        if (!c) fail(GX_INVALID_ARGUMENT, "null handle");
        FILE* fp = std::fopen(path, "wb");
        if (!fp) fail(GX_RUNTIME_ERROR, std::string("cannot open: ") + path);
        auto put = [&](const void* p, size_t nb) {
            if (nb && std::fwrite(p, 1, nb, fp) != nb) {
                std::fclose(fp);
                fail(GX_RUNTIME_ERROR, std::string("short write: ") + path);
            }
        };
        const uint32_t ver = 1;
        put(kNcMagic, 8);
        put(&ver, 4);
        put(&c->n, 8);
        put(&c->n_cells, 8);
        const uint64_t CH = 1ull << 24;
        std::vector<uint64_t> buf(std::min<uint64_t>(std::max(c->n, c->n_cells), CH) + 1);
        for (uint64_t o = 0; o < c->n; o += CH) {
            const uint64_t k = std::min(CH, c->n - o);
            GX_CUDA(cudaMemcpy(buf.data(), c->addr.p + o, k * 8, cudaMemcpyDeviceToHost));
            put(buf.data(), k * 8);
        }
        for (uint64_t o = 0; o < c->n_cells; o += CH) {
            const uint64_t k = std::min(CH, c->n_cells - o);
            GX_CUDA(cudaMemcpy(buf.data(), c->cells.p + o, k * 8, cudaMemcpyDeviceToHost));
            put(buf.data(), k * 8);
        }
        if (std::fclose(fp) != 0) fail(GX_RUNTIME_ERROR, std::string("close failed: ") + path);
    });
}

gx_status gx_ncache_open(gx_graph* g, const char* path, gx_iostats* io, gx_ncache** out) {
    return guard([&] {
        if (!g) fail(GX_INVALID_ARGUMENT, "null graph");
        FILE* fp = std::fopen(path, "rb");
        if (!fp) fail(GX_RUNTIME_ERROR, std::string("cannot open: ") + path);
        std::unique_ptr<FILE, int (*)(FILE*)> guard_fp(fp, std::fclose);
        auto get = [&](void* p, size_t nb) {
            if (nb && std::fread(p, 1, nb, fp) != nb) fail(GX_RUNTIME_ERROR, std::string("truncated file: ") + path);
        };
        char mg[8];
        get(mg, 8);
        if (std::memcmp(mg, kNcMagic, 8) != 0)
            fail(GX_RUNTIME_ERROR, std::string("bad magic in ") + path + " (expected GXNCACH1)");
        uint32_t ver = 0;
        get(&ver, 4);
        if (ver != 1) fail(GX_RUNTIME_ERROR, "unsupported neighbor cache version: " + std::to_string(ver));
        uint64_t nodes = 0, ncells = 0;
        get(&nodes, 8);
        get(&ncells, 8);
        if (nodes != g->n) fail(GX_INVALID_ARGUMENT, "neighbor cache and graph disagree on node count");
        auto nc = std::make_unique<gx_ncache>();
        nc->ctx = g->ctx;
        nc->n = nodes;
        nc->n_cells = ncells;
        nc->addr.alloc(std::max<uint64_t>(nodes, 1));
        nc->cells.alloc(std::max<uint64_t>(ncells, 1));
        const uint64_t CH = 1ull << 24;
        std::vector<uint64_t> buf(std::min<uint64_t>(std::max(nodes, ncells), CH) + 1);
        for (uint64_t o = 0; o < nodes; o += CH) {
            const uint64_t k = std::min(CH, nodes - o);
            get(buf.data(), k * 8);
            GX_CUDA(cudaMemcpy(nc->addr.p + o, buf.data(), k * 8, cudaMemcpyHostToDevice));
        }
        for (uint64_t o = 0; o < ncells; o += CH) {
            const uint64_t k = std::min(CH, ncells - o);
            get(buf.data(), k * 8);
            GX_CUDA(cudaMemcpy(nc->cells.p + o, buf.data(), k * 8, cudaMemcpyHostToDevice));
        }
        gx_ctx* ctx = g->ctx;
        nc->bits.alloc((nodes + 31) / 32 + 1);
        GX_CUDA(cudaMemsetAsync(nc->bits.p, 0, nc->bits.bytes(), ctx->stream));
        DevBuf<unsigned long long> cnt(1);
        GX_CUDA(cudaMemsetAsync(cnt.p, 0, 8, ctx->stream));
        if (nodes) {
            k_bits_from_addr<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(nc->addr.p, nodes, nc->bits.p, cnt.p);
            GX_CHECK_LAUNCH();
        }
        unsigned long long h = 0;
        GX_CUDA(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
        nc->n_cached = h;
        if (io) {  // load_neighbor_cache charges the file's bytes (neighbor_cache.hpp:140-144)
            const uint64_t bytes = 8 + 4 + 16 + nodes * 8 + ncells * 8;
            io->bytes_read += bytes;
            io->pages_read += pages_touched(0, bytes);
        }
        *out = nc.release();
    });
}

void gx_ncache_destroy(gx_ncache* c) { delete c; }
uint64_t gx_ncache_cached_nodes(const gx_ncache* c) { return c ? c->n_cached : 0; }
uint64_t gx_ncache_bytes_used(const gx_ncache* c) { return c ? (c->n + c->n_cells) * 8 : 0; }

gx_status gx_ncache_contains(const gx_ncache* c, uint64_t v, int* out) {
    return guard([&] {
        if (!c) fail(GX_INVALID_ARGUMENT, "null handle");
        if (v >= c->n) fail(GX_OUT_OF_RANGE, "node id out of range");
        int64_t a = -1;
        GX_CUDA(cudaMemcpy(&a, c->addr.p + v, 8, cudaMemcpyDeviceToHost));
        *out = a >= 0;
    });
}

gx_status gx_graph_set_neighbor_cache(gx_graph* g, const gx_ncache* c) {
    return guard([&] {
        if (!g) fail(GX_INVALID_ARGUMENT, "null graph");
        if (c && c->n != g->n) fail(GX_INVALID_ARGUMENT, "neighbor cache and graph disagree on node count");
        g->ncache_bits = c ? c->bits.p : nullptr;
    });
}

}  // extern "C"
