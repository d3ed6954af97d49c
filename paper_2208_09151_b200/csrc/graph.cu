// graph.cu -- HBM-resident CSC graph and feature table: loaders for the
// reference's on-disk formats, writers, and a bit-exact device generator.
//
// Formats: docs/FORMATS.md; GraphFile::open (graph_store.hpp:108-133),
// persist_graph (:83-98), FeatureFile::open (:282-302), FeatureWriter (:237-269).
// Generator: generate_edges (graphgen.hpp:55-70) + build_csc (graph_store.hpp:
// 53-81) + feature_value (graphgen.hpp:74-77). The dataset generator is input
// synthesis, not the hot path; it uses CUB for sort/unique/scan.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <fcntl.h>
#include <unistd.h>

#include <cuda_fp16.h>

#include "gx_internal.cuh"

namespace gx {

static const char kGraphMagic[8] = {'G', 'X', 'G', 'R', 'A', 'P', 'H', '1'};
static const char kFeatMagic[8] = {'G', 'X', 'F', 'E', 'A', 'T', '0', '1'};

struct File {
    int fd = -1;
    std::string path;
    explicit File(const char* p, int flags = O_RDONLY, int mode = 0644) : path(p) {
        fd = ::open(p, flags, mode);
        if (fd < 0) fail(GX_RUNTIME_ERROR, std::string("cannot open: ") + p);
    }
    ~File() {
        if (fd >= 0) ::close(fd);
    }
    uint64_t size() const {
        off_t e = ::lseek(fd, 0, SEEK_END);
        if (e < 0) fail(GX_RUNTIME_ERROR, "lseek failed: " + path);
        return (uint64_t)e;
    }
    void read_at(void* dst, size_t n, uint64_t off) const {
        size_t done = 0;
        while (done < n) {
            ssize_t r = ::pread(fd, (char*)dst + done, n - done, (off_t)(off + done));
            if (r < 0) fail(GX_RUNTIME_ERROR, "pread failed: " + path);
            if (r == 0) fail(GX_RUNTIME_ERROR, "truncated file: " + path);
            done += (size_t)r;
        }
    }
    void write_all(const void* src, size_t n) const {
        size_t done = 0;
        while (done < n) {
            ssize_t r = ::write(fd, (const char*)src + done, n - done);
            if (r <= 0) fail(GX_RUNTIME_ERROR, "short write: " + path);
            done += (size_t)r;
        }
    }
};

static uint64_t get_u64(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}
static uint32_t get_u32(const unsigned char* p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
    return v;
}

__global__ void k_narrow_ids(const uint64_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n,
                             uint64_t N, unsigned int* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = in[i];
        if (v >= N) atomicOr(bad, 1u);
        out[i] = (uint32_t)v;
    }
}
__global__ void k_widen_ids(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// Upload u64 host ids into a u32 device array (chunked through pinned memory).
static void upload_ids(gx_ctx* ctx, const uint64_t* h, uint64_t n, uint32_t* d, uint64_t N,
                       const File* f = nullptr, uint64_t file_off = 0) {
    const uint64_t CH = 1ull << 24;  // 16M ids per chunk
    PinBuf<uint64_t> pin;
    pin.alloc(std::min(n, CH) + 1);
    DevBuf<uint64_t> tmp(std::min(n, CH) + 1);
    DevBuf<unsigned int> bad(1);
    GX_CUDA(cudaMemsetAsync(bad.p, 0, 4, ctx->stream));
    for (uint64_t o = 0; o < n; o += CH) {
        const uint64_t c = std::min(CH, n - o);
        if (f) f->read_at(pin.p, c * 8, file_off + o * 8);
        else std::memcpy(pin.p, h + o, c * 8);
        GX_CUDA(cudaMemcpyAsync(tmp.p, pin.p, c * 8, cudaMemcpyHostToDevice, ctx->stream));
        k_narrow_ids<<<ctx->num_sms * 4, 256, 0, ctx->stream>>>(tmp.p, d + o, c, N, bad.p);
        GX_CHECK_LAUNCH();
        GX_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    unsigned int hb = 0;
    GX_CUDA(cudaMemcpy(&hb, bad.p, 4, cudaMemcpyDeviceToHost));
    if (hb) fail(GX_RUNTIME_ERROR, "graph contains out-of-range neighbor id");
}

static void check_nodes_u32(uint64_t n) {
    if (n >= 0xFFFFFFFFull) fail(GX_OVERFLOW, "num_nodes exceeds the u32 device id range");
}

// ---------------------------------------------------------------------------
// R-MAT generator (graphgen.hpp:32-70): attempt t consumes draws
// [t*scale, (t+1)*scale) of SplitMix64(edge_seed); accepted iff both
// endpoints < N; the first `target` accepted attempts are the edge list.
// ---------------------------------------------------------------------------
__global__ void k_rmat(uint64_t seed, unsigned scale, uint64_t N, double ta, double tab, double tabc,
                       uint64_t t0, uint64_t cnt, unsigned long long* keys, uint8_t* ok) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < cnt;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = t0 + k;
        uint64_t s = 0, d = 0;
        uint64_t ctr = seed + (t * scale + 1) * kGamma;  // state after the first next()
        for (unsigned lv = 0; lv < scale; ++lv) {
            uint64_t z = ctr;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            z ^= z >> 31;
            ctr += kGamma;
            const double r = (double)(z >> 11) * 0x1.0p-53;
            s <<= 1;
            d <<= 1;
            if (r < ta) {
            } else if (r < tab) {
                d |= 1;
            } else if (r < tabc) {
                s |= 1;
            } else {
                s |= 1;
                d |= 1;
            }
        }
        const bool acc = s < N && d < N;
        ok[k] = acc;
        keys[k] = acc ? ((d << 32) | s) : ~0ull;
    }
}

__global__ void k_indptr_from_sorted(const unsigned long long* __restrict__ keys, uint64_t E, uint64_t N,
                                     uint64_t* indptr, uint32_t* indices) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[e];
        const uint64_t d = k >> 32;
        indices[e] = (uint32_t)k;
        const uint64_t prev = e ? (keys[e - 1] >> 32) : (uint64_t)-1;
        if (e == 0) {
            for (uint64_t v = 0; v <= d; ++v) indptr[v] = 0;
        } else if (d != prev) {
            for (uint64_t v = prev + 1; v <= d; ++v) indptr[v] = e;
        }
        if (e == E - 1)
            for (uint64_t v = d + 1; v <= N; ++v) indptr[v] = E;
    }
}

__global__ void k_fill_u64(uint64_t* p, uint64_t n, uint64_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

static void generate_rmat(gx_graph* g, uint64_t N, double avg, double a, double b, double c,
                          uint64_t seed) {
    gx_ctx* ctx = g->ctx;
    cudaStream_t st = ctx->stream;
    if (N < 1) fail(GX_INVALID_ARGUMENT, "num_nodes must be >= 1");
    if (avg < 0) fail(GX_INVALID_ARGUMENT, "avg_degree must be >= 0");
    const double d = 1.0 - a - b - c;
    const double ssum = a + b + c + d;
    if (ssum < 0.999 || ssum > 1.001) fail(GX_INVALID_ARGUMENT, "quadrant probabilities must sum to 1");
    check_nodes_u32(N);
    unsigned scale = 0;
    while ((1ull << scale) < N) ++scale;
    const uint64_t target = (uint64_t)(avg * (double)N);
    const double ta = a, tab = a + b, tabc = a + b + c;
    DevBuf<unsigned long long> keys(std::max<uint64_t>(target, 1));
    uint64_t have = 0, t0 = 0;
    const uint64_t CH = 1ull << 26;
    DevBuf<unsigned long long> ck(CH), ckout(CH);
    DevBuf<uint8_t> ok(CH);
    DevBuf<uint64_t> nsel(1);
    size_t tmp_bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp_bytes, ck.p, ok.p, ckout.p, nsel.p, (int)CH, st);
    DevBuf<uint8_t> tmp(tmp_bytes + 1);
    while (have < target) {
        // expected acceptance is high; size the chunk to what is still needed
        const uint64_t cnt = CH;
        k_rmat<<<ctx->num_sms * 8, 256, 0, st>>>(seed, scale, N, ta, tab, tabc, t0, cnt, ck.p, ok.p);
        GX_CHECK_LAUNCH();
        GX_CUDA(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, ck.p, ok.p, ckout.p, nsel.p, (int)cnt, st));
        uint64_t ns = 0;
        GX_CUDA(cudaMemcpyAsync(&ns, nsel.p, 8, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        const uint64_t take = std::min(ns, target - have);
        GX_CUDA(cudaMemcpyAsync(keys.p + have, ckout.p, take * 8, cudaMemcpyDeviceToDevice, st));
        have += take;
        t0 += cnt;
    }
    ck.release();
    ckout.release();
    ok.release();
    tmp.release();
    // build_csc: sort (dst, src), unique
    const uint64_t M = target;
    int end_bit = 32;
    while (end_bit < 64 && (1ull << (end_bit - 32)) < N) ++end_bit;
    DevBuf<unsigned long long> alt(std::max<uint64_t>(M, 1));
    if (M > 0) {
        if (M > 0x7FFFFFFFull) fail(GX_INVALID_ARGUMENT, "generator: more than 2^31 edges unsupported");
        cub::DoubleBuffer<unsigned long long> db(keys.p, alt.p);
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int)M, 0, end_bit, st);
        DevBuf<uint8_t> t2(tb + 1);
        GX_CUDA(cub::DeviceRadixSort::SortKeys(t2.p, tb, db, (int)M, 0, end_bit, st));
        unsigned long long* sorted = db.Current();
        unsigned long long* other = sorted == keys.p ? alt.p : keys.p;
        size_t tu = 0;
        cub::DeviceSelect::Unique(nullptr, tu, sorted, other, nsel.p, (int)M, st);
        DevBuf<uint8_t> t3(tu + 1);
        GX_CUDA(cub::DeviceSelect::Unique(t3.p, tu, sorted, other, nsel.p, (int)M, st));
        uint64_t E = 0;
        GX_CUDA(cudaMemcpyAsync(&E, nsel.p, 8, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        g->n = N;
        g->e = E;
        g->indptr.alloc(N + 1);
        g->indices.alloc(std::max<uint64_t>(E, 1));
        k_indptr_from_sorted<<<ctx->num_sms * 8, 256, 0, st>>>(other, E, N, g->indptr.p, g->indices.p);
        GX_CHECK_LAUNCH();
    } else {
        g->n = N;
        g->e = 0;
        g->indptr.alloc(N + 1);
        g->indices.alloc(1);
        k_fill_u64<<<ctx->num_sms, 256, 0, st>>>(g->indptr.p, N + 1, 0);
        GX_CHECK_LAUNCH();
    }
    GX_CUDA(cudaStreamSynchronize(st));
}

// feature_value (graphgen.hpp:74-77) for a whole table.
// Rows [node0, node0 + n) of the table; fp16 extension: __float2half_rn of the value.
template <class T>
__global__ void k_features(T* out, uint64_t n, uint32_t dim, uint64_t vseed, uint64_t node0) {
    const uint64_t total = n * dim;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / dim;
        const uint32_t col = (uint32_t)(i - r * dim);
        const uint64_t h = mix64(vseed ^ mix64((node0 + r) * 0x10001ULL + col));
        const float v = (float)(h >> 40) * 0x1.0p-24f;
        if constexpr (sizeof(T) == 2) out[i] = __float2half_rn(v);
        else out[i] = v;
    }
}

void launch_features(uint8_t* out, uint64_t n, uint32_t dim, uint32_t sw, uint64_t vseed, uint64_t node0,
                     int num_sms, cudaStream_t s) {
    if (!n) return;
    if (sw == 2) k_features<__half><<<num_sms * 8, 256, 0, s>>>((__half*)out, n, dim, vseed, node0);
    else k_features<float><<<num_sms * 8, 256, 0, s>>>((float*)out, n, dim, vseed, node0);
    GX_CHECK_LAUNCH();
}

static void features_alloc(gx_features* f, int backing) {
    const uint64_t bytes = f->n * f->row_bytes;
    f->backing = backing;
    if (backing == GX_BACKING_DEVICE) {
        f->dev.alloc(std::max<uint64_t>(bytes, 16));
        f->rows_dev_view = f->dev.p;
    } else if (backing == GX_BACKING_HOST) {
        f->host.alloc(std::max<uint64_t>(bytes, 16), cudaHostAllocMapped | cudaHostAllocPortable);
        uint8_t* dp = nullptr;
        GX_CUDA(cudaHostGetDevicePointer((void**)&dp, f->host.p, 0));
        f->rows_dev_view = dp;
    } else {
        fail(GX_INVALID_ARGUMENT, "unknown backing mode");
    }
}

}  // namespace gx

using namespace gx;

extern "C" {

gx_status gx_graph_open(gx_ctx* ctx, const char* path, gx_graph** out) {
    return guard([&] {
        File f(path);
        const uint64_t fsz = f.size();
        unsigned char hdr[36];
        if (fsz < 8 || (f.read_at(hdr, 8, 0), std::memcmp(hdr, kGraphMagic, 8) != 0))
            fail(GX_RUNTIME_ERROR, std::string("bad magic in ") + path + " (expected GXGRAPH1)");
        if (fsz < 36) fail(GX_RUNTIME_ERROR, std::string("truncated file: ") + path);
        f.read_at(hdr, 36, 0);
        const uint32_t ver = get_u32(hdr + 8);
        const uint64_t n = get_u64(hdr + 12), e = get_u64(hdr + 20), ioff = get_u64(hdr + 28);
        if (ver != 1) fail(GX_RUNTIME_ERROR, "unsupported graph version: " + std::to_string(ver));
        if (fsz < 36 + (n + 1) * 8) fail(GX_RUNTIME_ERROR, std::string("truncated file: ") + path);
        std::vector<uint64_t> ip(n + 1);
        f.read_at(ip.data(), (n + 1) * 8, 36);
        if (ip.front() != 0 || ip.back() != e)
            fail(GX_RUNTIME_ERROR, std::string("graph file indptr is inconsistent: ") + path);
        if (fsz < ioff + e * 8) fail(GX_RUNTIME_ERROR, std::string("truncated graph file: ") + path);
        check_nodes_u32(n);
        auto g = new gx_graph();
        try {
            g->ctx = ctx;
            g->n = n;
            g->e = e;
            g->indptr.alloc(n + 1);
            g->indices.alloc(std::max<uint64_t>(e, 1));
            GX_CUDA(cudaMemcpy(g->indptr.p, ip.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
            if (e) upload_ids(ctx, nullptr, e, g->indices.p, n, &f, ioff);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

gx_status gx_graph_from_csc(gx_ctx* ctx, uint64_t n, const uint64_t* indptr, const uint64_t* indices,
                            gx_graph** out) {
    return guard([&] {
        check_nodes_u32(n);
        if (indptr[0] != 0) fail(GX_INVALID_ARGUMENT, "indptr[0] must be 0");
        for (uint64_t v = 0; v < n; ++v)
            if (indptr[v + 1] < indptr[v]) fail(GX_INVALID_ARGUMENT, "indptr must be non-decreasing");
        const uint64_t e = indptr[n];
        auto g = new gx_graph();
        try {
            g->ctx = ctx;
            g->n = n;
            g->e = e;
            g->indptr.alloc(n + 1);
            g->indices.alloc(std::max<uint64_t>(e, 1));
            GX_CUDA(cudaMemcpy(g->indptr.p, indptr, (n + 1) * 8, cudaMemcpyHostToDevice));
            if (e) upload_ids(ctx, indices, e, g->indices.p, n);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

gx_status gx_graph_generate_rmat(gx_ctx* ctx, uint64_t n, double avg, double a, double b, double c,
                                 uint64_t seed, gx_graph** out) {
    return guard([&] {
        auto g = new gx_graph();
        g->ctx = ctx;
        try {
            generate_rmat(g, n, avg, a, b, c, seed);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}

void gx_graph_destroy(gx_graph* g) { delete g; }
uint64_t gx_graph_num_nodes(const gx_graph* g) { return g ? g->n : 0; }
uint64_t gx_graph_num_edges(const gx_graph* g) { return g ? g->e : 0; }

gx_status gx_graph_in_degree(const gx_graph* g, uint64_t v, uint64_t* deg) {
    return guard([&] {
        if (v >= g->n) fail(GX_OUT_OF_RANGE, "node id out of range");
        uint64_t ip[2];
        GX_CUDA(cudaMemcpy(ip, g->indptr.p + v, 16, cudaMemcpyDeviceToHost));
        *deg = ip[1] - ip[0];
    });
}

gx_status gx_graph_copy_csc(const gx_graph* g, uint64_t* indptr, uint64_t* indices) {
    return guard([&] {
        require_whole_csc(g, "copy_csc");
        GX_CUDA(cudaMemcpy(indptr, g->indptr.p, (g->n + 1) * 8, cudaMemcpyDeviceToHost));
        const uint64_t CH = 1ull << 24;
        DevBuf<uint64_t> tmp(std::min(g->e, CH) + 1);
        for (uint64_t o = 0; o < g->e; o += CH) {
            const uint64_t c = std::min(CH, g->e - o);
            k_widen_ids<<<g->ctx->num_sms * 4, 256, 0, g->ctx->stream>>>(g->indices.p + o, tmp.p, c);
            GX_CHECK_LAUNCH();
            GX_CUDA(cudaMemcpyAsync(indices + o, tmp.p, c * 8, cudaMemcpyDeviceToHost, g->ctx->stream));
            GX_CUDA(cudaStreamSynchronize(g->ctx->stream));
        }
    });
}

gx_status gx_graph_write(const gx_graph* g, const char* path) {
    return guard([&] {
        require_whole_csc(g, "persist_graph");
        File f(path, O_WRONLY | O_CREAT | O_TRUNC);
        unsigned char hdr[36];
        std::memcpy(hdr, kGraphMagic, 8);
        const uint32_t ver = 1;
        const uint64_t hb = 36, ipb = (g->n + 1) * 8;
        const uint64_t ioff = (hb + ipb + kPage - 1) / kPage * kPage;
        std::memcpy(hdr + 8, &ver, 4);
        std::memcpy(hdr + 12, &g->n, 8);
        std::memcpy(hdr + 20, &g->e, 8);
        std::memcpy(hdr + 28, &ioff, 8);
        f.write_all(hdr, 36);
        std::vector<uint64_t> ip(g->n + 1);
        GX_CUDA(cudaMemcpy(ip.data(), g->indptr.p, ipb, cudaMemcpyDeviceToHost));
        f.write_all(ip.data(), ipb);
        std::vector<char> zeros(ioff - hb - ipb, 0);
        if (!zeros.empty()) f.write_all(zeros.data(), zeros.size());
        const uint64_t CH = 1ull << 24;
        DevBuf<uint64_t> tmp(std::min(g->e, CH) + 1);
        PinBuf<uint64_t> pin;
        pin.alloc(std::min(g->e, CH) + 1);
        for (uint64_t o = 0; o < g->e; o += CH) {
            const uint64_t c = std::min(CH, g->e - o);
            k_widen_ids<<<g->ctx->num_sms * 4, 256, 0, g->ctx->stream>>>(g->indices.p + o, tmp.p, c);
            GX_CHECK_LAUNCH();
            GX_CUDA(cudaMemcpyAsync(pin.p, tmp.p, c * 8, cudaMemcpyDeviceToHost, g->ctx->stream));
            GX_CUDA(cudaStreamSynchronize(g->ctx->stream));
            f.write_all(pin.p, c * 8);
        }
    });
}

// ---- row-partitioned CSC --------------------------------------

namespace gx {
GraphParts::~GraphParts() {
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
}
}  // namespace gx

// bounds[q] = the first node whose list starts at or after E*q/P (lower bound
// on indptr), so every rank owns about E/P edges and no list is split
__global__ void k_part_bounds(const uint64_t* __restrict__ indptr, uint64_t N, uint64_t E, int P,
                              uint64_t* __restrict__ bounds) {
    const int q = threadIdx.x;
    if (q > P) return;
    if (q == 0 || q == P) {
        bounds[q] = q == 0 ? 0 : N;
        return;
    }
    const uint64_t want = (uint64_t)((unsigned __int128)E * (unsigned)q / (unsigned)P);
    uint64_t lo = 0, hi = N;  // first v in [0, N] with indptr[v] >= want
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (indptr[mid] < want) lo = mid + 1;
        else hi = mid;
    }
    bounds[q] = lo;
}

static void part_bounds(const gx_graph* g, int P, uint64_t* nb, uint64_t* eb) {
    if (P < 1 || P > kMaxParts) fail(GX_INVALID_ARGUMENT, "partition count must be in [1, " +
                                                           std::to_string(kMaxParts) + "]");
    DevBuf<uint64_t> d(P + 1);
    k_part_bounds<<<1, 32, 0, g->ctx->stream>>>(g->indptr.p, g->n, g->e, P, d.p);
    GX_CHECK_LAUNCH();
    GX_CUDA(cudaMemcpyAsync(nb, d.p, (P + 1) * 8, cudaMemcpyDeviceToHost, g->ctx->stream));
    GX_CUDA(cudaStreamSynchronize(g->ctx->stream));
    for (int q = 0; q <= P; ++q)
        GX_CUDA(cudaMemcpy(eb + q, g->indptr.p + nb[q], 8, cudaMemcpyDeviceToHost));
}

gx_status gx_graph_partition_bounds(const gx_graph* g, int P, uint64_t* node_bounds) {
    return guard([&] {
        std::vector<uint64_t> eb(P + 1);
        if (g->part.P) {
            if (P != g->part.P) fail(GX_INVALID_ARGUMENT, "graph is already partitioned differently");
            std::copy(g->part.node_bounds, g->part.node_bounds + P + 1, node_bounds);
            return;
        }
        part_bounds(g, P, node_bounds, eb.data());
    });
}

gx_status gx_graph_partition(gx_graph* g, int P, int rank) {
    return guard([&] {
        if (g->part.P) fail(GX_LOGIC_ERROR, "graph is already partitioned");
        if (rank < 0 || rank >= P) fail(GX_INVALID_ARGUMENT, "rank out of range");
        GraphParts& pt = g->part;
        GX_CUDA(cudaSetDevice(g->ctx->device));
        part_bounds(g, P, pt.node_bounds, pt.ebound);
        const uint64_t lo = pt.ebound[rank], hi = pt.ebound[rank + 1];
        DevBuf<uint32_t> mine(std::max<uint64_t>(hi - lo, 1));
        if (hi > lo)
            GX_CUDA(cudaMemcpyAsync(mine.p, g->indices.p + lo, (hi - lo) * 4, cudaMemcpyDeviceToDevice,
                                    g->ctx->stream));
        GX_CUDA(cudaStreamSynchronize(g->ctx->stream));
        g->indices = std::move(mine);   // the other ranks' share is freed
        pt.P = P;
        pt.rank = rank;
        pt.ptr[rank] = g->indices.p;
        pt.attached = P == 1;
    });
}

gx_status gx_graph_ipc_handle(const gx_graph* g, void* handle, uint64_t* edge_lo, uint64_t* edge_hi) {
    return guard([&] {
        if (!g->part.P) fail(GX_LOGIC_ERROR, "graph is not partitioned");
        static_assert(sizeof(cudaIpcMemHandle_t) == GX_IPC_HANDLE_BYTES, "IPC handle size");
        GX_CUDA(cudaSetDevice(g->ctx->device));
        cudaIpcMemHandle_t h;
        GX_CUDA(cudaIpcGetMemHandle(&h, g->indices.p));
        std::memcpy(handle, &h, sizeof(h));
        *edge_lo = g->part.ebound[g->part.rank];
        *edge_hi = g->part.ebound[g->part.rank + 1];
    });
}

gx_status gx_graph_attach_peers(gx_graph* g, const void* handles, const uint64_t* lohi) {
    return guard([&] {
        GraphParts& pt = g->part;
        if (!pt.P) fail(GX_LOGIC_ERROR, "graph is not partitioned");
        if (pt.attached) fail(GX_LOGIC_ERROR, "peers are already attached");
        GX_CUDA(cudaSetDevice(g->ctx->device));  // the mappings belong to this graph's device
        for (int q = 0; q < pt.P; ++q)
            if (lohi[2 * q] != pt.ebound[q] || lohi[2 * q + 1] != pt.ebound[q + 1])
                fail(GX_INVALID_ARGUMENT, "peer " + std::to_string(q) + " holds a different edge range");
        std::vector<void*> opened;
        try {
            for (int q = 0; q < pt.P; ++q) {
                if (q == pt.rank) continue;
                cudaIpcMemHandle_t h;
                std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)q * GX_IPC_HANDLE_BYTES, sizeof(h));
                void* p = nullptr;
                GX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
                opened.push_back(p);
                pt.ptr[q] = static_cast<const uint32_t*>(p);
            }
        } catch (...) {
            for (void* p : opened) cudaIpcCloseMemHandle(p);
            throw;
        }
        pt.ipc_opened = std::move(opened);
        pt.attached = true;
    });
}

gx_status gx_graph_attach_local(gx_graph* g, gx_graph* const* parts, int P) {
    return guard([&] {
        GraphParts& pt = g->part;
        if (!pt.P) fail(GX_LOGIC_ERROR, "graph is not partitioned");
        if (pt.attached && P > 1) fail(GX_LOGIC_ERROR, "peers are already attached");
        if (P != pt.P) fail(GX_INVALID_ARGUMENT, "partition count mismatch");
        for (int q = 0; q < P; ++q) {
            const GraphParts& o = parts[q]->part;
            if (o.P != P || o.rank != q || parts[q]->n != g->n || parts[q]->e != g->e ||
                o.ebound[q] != pt.ebound[q] || o.ebound[q + 1] != pt.ebound[q + 1])
                fail(GX_INVALID_ARGUMENT, "part " + std::to_string(q) + " is not rank " + std::to_string(q) +
                                              " of the same partition");
            pt.ptr[q] = parts[q]->indices.p;
        }
        pt.attached = true;
    });
}

gx_status gx_graph_partition_info(const gx_graph* g, int* nranks, int* rank, int* attached) {
    return guard([&] {
        *nranks = g->part.P;
        *rank = g->part.rank;
        *attached = g->part.attached ? 1 : 0;
    });
}

gx_status gx_features_open(gx_ctx* ctx, const char* path, int backing, gx_features** out) {
    return guard([&] {
        File f(path);
        const uint64_t fsz = f.size();
        unsigned char hdr[36];
        if (fsz < 8 || (f.read_at(hdr, 8, 0), std::memcmp(hdr, kFeatMagic, 8) != 0))
            fail(GX_RUNTIME_ERROR, std::string("bad magic in ") + path + " (expected GXFEAT01)");
        if (fsz < 36) fail(GX_RUNTIME_ERROR, std::string("truncated file: ") + path);
        f.read_at(hdr, 36, 0);
        const uint32_t ver = get_u32(hdr + 8);
        if (ver != 1) fail(GX_RUNTIME_ERROR, "unsupported feature version: " + std::to_string(ver));
        auto ft = new gx_features();
        try {
            ft->ctx = ctx;
            ft->n = get_u64(hdr + 12);
            ft->dim = get_u32(hdr + 20);
            ft->scalar_width = get_u32(hdr + 24);
            const uint64_t poff = get_u64(hdr + 28);
            // scalar_width 4 is the reference format (graph_store.hpp:295-296);
            // 2 is this framework's fp16 extension (cfg4, MAG240M-shape).
            if (ft->scalar_width != 4 && ft->scalar_width != 2)
                fail(GX_RUNTIME_ERROR, std::string("unsupported scalar width in ") + path);
            ft->row_bytes = (uint64_t)ft->dim * ft->scalar_width;
            if (fsz < poff + ft->n * ft->row_bytes)
                fail(GX_RUNTIME_ERROR, std::string("truncated feature file: ") + path);
            if (backing == GX_BACKING_FILE) {  // the storage tier: rows stay in the file
                check_nodes_u32(ft->n);
                ft->backing = GX_BACKING_FILE;
                ft->file.reset(new RowReader(path, poff, ft->row_bytes, ft->n));
                *out = ft;
                return;
            }
            if (!ctx) fail(GX_INVALID_ARGUMENT, "a device or host backed table needs a context");
            features_alloc(ft, backing);
            const uint64_t bytes = ft->n * ft->row_bytes;
            if (backing == GX_BACKING_HOST) {
                if (bytes) f.read_at(ft->host.p, bytes, poff);
            } else {
                const uint64_t CH = 1ull << 28;
                PinBuf<uint8_t> pin;
                pin.alloc(std::min(bytes, CH) + 1);
                for (uint64_t o = 0; o < bytes; o += CH) {
                    const uint64_t c = std::min(CH, bytes - o);
                    f.read_at(pin.p, c, poff + o);
                    GX_CUDA(cudaMemcpy(ft->dev.p + o, pin.p, c, cudaMemcpyHostToDevice));
                }
            }
        } catch (...) {
            delete ft;
            throw;
        }
        *out = ft;
    });
}

gx_status gx_features_from_host(gx_ctx* ctx, uint64_t n, uint32_t dim, uint32_t sw, const void* rows,
                                int backing, gx_features** out) {
    return guard([&] {
        if (backing == GX_BACKING_FILE)
            fail(GX_INVALID_ARGUMENT, "GX_BACKING_FILE tables are opened from features.bin (gx_features_open)");
        if (sw != 4 && sw != 2) fail(GX_INVALID_ARGUMENT, "scalar_width must be 4 or 2");
        if (dim < 1) fail(GX_INVALID_ARGUMENT, "dim must be >= 1");
        check_nodes_u32(n);
        auto ft = new gx_features();
        try {
            ft->ctx = ctx;
            ft->n = n;
            ft->dim = dim;
            ft->scalar_width = sw;
            ft->row_bytes = (uint64_t)dim * sw;
            features_alloc(ft, backing);
            const uint64_t bytes = n * ft->row_bytes;
            if (bytes) {
                if (backing == GX_BACKING_HOST) std::memcpy(ft->host.p, rows, bytes);
                else GX_CUDA(cudaMemcpy(ft->dev.p, rows, bytes, cudaMemcpyHostToDevice));
            }
        } catch (...) {
            delete ft;
            throw;
        }
        *out = ft;
    });
}

gx_status gx_features_generate(gx_ctx* ctx, uint64_t n, uint32_t dim, uint64_t vseed, gx_features** out) {
    return guard([&] {
        if (dim < 1) fail(GX_INVALID_ARGUMENT, "dim must be >= 1");
        check_nodes_u32(n);
        auto ft = new gx_features();
        try {
            ft->ctx = ctx;
            ft->n = n;
            ft->dim = dim;
            ft->scalar_width = 4;
            ft->row_bytes = (uint64_t)dim * 4;
            features_alloc(ft, GX_BACKING_DEVICE);
            launch_features(ft->dev.p, n, dim, 4, vseed, 0, ctx->num_sms, ctx->stream);
            GX_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete ft;
            throw;
        }
        *out = ft;
    });
}

gx_status gx_features_write(const gx_features* f, const char* path) {
    return guard([&] {
        if (!f) fail(GX_INVALID_ARGUMENT, "null handle");
        if (f->backing == GX_BACKING_FILE) fail(GX_INVALID_ARGUMENT, "table is already file backed");
        // FeatureWriter (graph_store.hpp:237-250): magic, u32 version, u64 n,
        // u32 dim, u32 scalar_width, u64 payload offset (4096), zero padding
        File out(path, O_WRONLY | O_CREAT | O_TRUNC);
        unsigned char hdr[kPage] = {};
        std::memcpy(hdr, kFeatMagic, 8);
        const uint32_t ver = 1;
        const uint64_t poff = kPage;
        std::memcpy(hdr + 8, &ver, 4);
        std::memcpy(hdr + 12, &f->n, 8);
        std::memcpy(hdr + 20, &f->dim, 4);
        std::memcpy(hdr + 24, &f->scalar_width, 4);
        std::memcpy(hdr + 28, &poff, 8);
        out.write_all(hdr, kPage);
        const uint64_t bytes = f->n * f->row_bytes;
        if (f->backing == GX_BACKING_HOST) {
            if (bytes) out.write_all(f->host.p, bytes);
            return;
        }
        const uint64_t CH = 1ull << 28;
        PinBuf<uint8_t> pin;
        pin.alloc(std::min(bytes, CH) + 1);
        for (uint64_t o = 0; o < bytes; o += CH) {
            const uint64_t c = std::min(CH, bytes - o);
            GX_CUDA(cudaMemcpy(pin.p, f->dev.p + o, c, cudaMemcpyDeviceToHost));
            out.write_all(pin.p, c);
        }
    });
}

gx_status gx_features_generate_fp16(gx_ctx* ctx, uint64_t n, uint32_t dim, uint64_t vseed, gx_features** out) {
    return guard([&] {
        if (dim < 1) fail(GX_INVALID_ARGUMENT, "dim must be >= 1");
        check_nodes_u32(n);
        auto ft = new gx_features();
        try {
            ft->ctx = ctx;
            ft->n = n;
            ft->dim = dim;
            ft->scalar_width = 2;
            ft->row_bytes = (uint64_t)dim * 2;
            features_alloc(ft, GX_BACKING_DEVICE);
            launch_features(ft->dev.p, n, dim, 2, vseed, 0, ctx->num_sms, ctx->stream);
            GX_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete ft;
            throw;
        }
        *out = ft;
    });
}

void gx_features_destroy(gx_features* f) { delete f; }
uint64_t gx_features_num_nodes(const gx_features* f) { return f ? f->n : 0; }
uint32_t gx_features_dim(const gx_features* f) { return f ? f->dim : 0; }
uint64_t gx_features_row_bytes(const gx_features* f) { return f ? f->row_bytes : 0; }

}  // extern "C"
