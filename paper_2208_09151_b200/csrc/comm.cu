// comm.cu -- the row-partitioned feature table and its exchange.
//
// The reference keeps the whole table in one features.bin and reads each miss
// with a pread (feature_cache.hpp:58-76, graph_store.hpp:308-315). Across the
// GPUs of one box the table is row-partitioned instead: rank r of P owns rows
// [N*r/P, N*(r+1)/P) in its HBM. A rank's storage requests (its cache init and
// its changeset misses -- known as soon as its inspector has run) are served in
// ONE variable all-to-all per request set:
//   1. owner of every request + a stable counting sort by owner (CUB radix sort
//      of (owner, request index) pairs, log2(P) key bits) -> per-owner runs of
//      local row ids;
//   2. counts all-to-all, then ids all-to-all (grouped send/recv);
//   3. each owner gathers the requested rows from its partition with the row
//      gather kernel (all-miss, no accounting) into a send buffer;
//   4. rows all-to-all back; a scatter kernel places row q at request perm[q].
// The transport is NCCL (grouped ncclSend/ncclRecv on the caller's stream; over
// NVLink/NVSwitch on a B200 box), or an in-process hub (one host thread per rank,
// peer copies through the CUDA runtime) that lets the single-GPU test suite run
// P ranks against the oracle. libnccl.so.2 is resolved at run time so the
// library loads (and its CPU tests run) where NCCL is absent, and so the process
// shares the NCCL torch.distributed already loaded.
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cub/cub.cuh>
#include <mutex>

#include "gx_internal.cuh"

namespace gx {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch loaded, if any
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = dlerror() ? dlerror() : "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        if (api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.GroupStart && api.GroupEnd)
            api.h = h;
        else
            err = "libnccl.so.2 lacks send/recv";
    });
    if (!api.h) fail(GX_RUNTIME_ERROR, "NCCL unavailable: " + err);
    return api;
}

#define GX_NCCL(call)                                                                                  \
    do {                                                                                               \
        ncclResult_t _r = (call);                                                                      \
        if (_r != ncclSuccess)                                                                         \
            ::gx::fail(GX_RUNTIME_ERROR, std::string("NCCL: ") + #call + ": " +                         \
                                             (nccl().GetErrorString ? nccl().GetErrorString(_r) : "")); \
    } while (0)

// ---------------------------------------------------------------------------
// transports
// ---------------------------------------------------------------------------
struct Transport {
    int rank = 0, size = 1;
    virtual ~Transport() = default;
    // recv[p] = what rank p sent to this rank (send[q] goes to rank q)
    virtual void counts(const uint64_t* send, uint64_t* recv, cudaStream_t s) = 0;
    // bytes: send + soff[p] (scnt[p]) -> rank p; recv + roff[p] (rcnt[p]) <- rank p; on stream s
    virtual void alltoallv(const uint8_t* send, const uint64_t* soff, const uint64_t* scnt, uint8_t* recv,
                           const uint64_t* roff, const uint64_t* rcnt, cudaStream_t s) = 0;
};

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    DevBuf<unsigned long long> dsend, drecv;
    PinBuf<unsigned long long> hbuf;
    ~NcclTransport() override {
        if (comm) nccl().CommDestroy(comm);
    }
    void counts(const uint64_t* send, uint64_t* recv, cudaStream_t s) override {
        auto& N = nccl();
        dsend.reserve(size);
        drecv.reserve(size);
        hbuf.reserve(size);
        std::memcpy(hbuf.p, send, size * 8);
        GX_CUDA(cudaMemcpyAsync(dsend.p, hbuf.p, size * 8, cudaMemcpyHostToDevice, s));
        GX_NCCL(N.GroupStart());
        for (int p = 0; p < size; ++p) {
            GX_NCCL(N.Send(dsend.p + p, 1, ncclUint64, p, comm, s));
            GX_NCCL(N.Recv(drecv.p + p, 1, ncclUint64, p, comm, s));
        }
        GX_NCCL(N.GroupEnd());
        GX_CUDA(cudaMemcpyAsync(hbuf.p, drecv.p, size * 8, cudaMemcpyDeviceToHost, s));
        GX_CUDA(cudaStreamSynchronize(s));
        std::memcpy(recv, hbuf.p, size * 8);
    }
    void alltoallv(const uint8_t* send, const uint64_t* soff, const uint64_t* scnt, uint8_t* recv,
                   const uint64_t* roff, const uint64_t* rcnt, cudaStream_t s) override {
        auto& N = nccl();
        GX_NCCL(N.GroupStart());
        for (int p = 0; p < size; ++p) {
            if (scnt[p]) GX_NCCL(N.Send(send + soff[p], scnt[p], ncclUint8, p, comm, s));
            if (rcnt[p]) GX_NCCL(N.Recv(recv + roff[p], rcnt[p], ncclUint8, p, comm, s));
        }
        GX_NCCL(N.GroupEnd());
    }
};

// In-process hub: P ranks on P host threads. Each exchange posts the rank's
// buffers, meets the others at a barrier, pulls its pieces from every peer
// with cudaMemcpyAsync (UVA; the contexts may share a GPU), then waits until
// every peer has pulled from it before its send buffer may be reused.
struct LocalHub {
    int P;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const uint8_t*> send;
    std::vector<const uint64_t*> soff, scnt;
    std::vector<std::vector<uint64_t>> cnt;
    std::vector<cudaEvent_t> ready, done;
    explicit LocalHub(int p) : P(p), send(p), soff(p), scnt(p), cnt(p, std::vector<uint64_t>(p)), ready(p), done(p) {
        for (int r = 0; r < P; ++r) {
            GX_CUDA(cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming));
            GX_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
        }
    }
    ~LocalHub() {
        for (int r = 0; r < P; ++r) {
            cudaEventDestroy(ready[r]);
            cudaEventDestroy(done[r]);
        }
    }
    bool broken = false;  // a rank failed inside an exchange: the others fail too
    void barrier(int rank) {
        std::unique_lock<std::mutex> lk(m);
        if (broken) fail(GX_RUNTIME_ERROR, "exchange aborted: another rank failed");
        const uint64_t g = gen;
        if (++arrived == P) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            static const int secs = env_int("GX_LOCAL_HUB_TIMEOUT_S", 120);
            if (!cv.wait_for(lk, std::chrono::seconds(secs), [&] { return gen != g || broken; })) {
                broken = true;
                cv.notify_all();
                fail(GX_RUNTIME_ERROR, "exchange timed out: rank " + std::to_string(rank) +
                                           " waited for the other ranks");
            }
            if (gen == g) fail(GX_RUNTIME_ERROR, "exchange aborted: another rank failed");
        }
    }
    void abort() {
        std::lock_guard<std::mutex> lk(m);
        broken = true;
        cv.notify_all();
    }
};

struct LocalTransport : Transport {
    std::shared_ptr<LocalHub> hub;
    template <class F>
    void guarded(F&& f) {  // a failing rank releases the others instead of leaving them in a barrier
        try {
            f();
        } catch (...) {
            hub->abort();
            throw;
        }
    }
    void counts(const uint64_t* send, uint64_t* recv, cudaStream_t) override {
        LocalHub& H = *hub;
        guarded([&] {
            for (int p = 0; p < size; ++p) H.cnt[rank][p] = send[p];
            H.barrier(rank);
            for (int p = 0; p < size; ++p) recv[p] = H.cnt[p][rank];
            H.barrier(rank);
        });
    }
    void alltoallv(const uint8_t* send, const uint64_t* soff, const uint64_t* scnt, uint8_t* recv,
                   const uint64_t* roff, const uint64_t* rcnt, cudaStream_t s) override {
        LocalHub& H = *hub;
        guarded([&] {
            H.send[rank] = send;
            H.soff[rank] = soff;
            H.scnt[rank] = scnt;
            GX_CUDA(cudaEventRecord(H.ready[rank], s));
            H.barrier(rank);
            for (int p = 0; p < size; ++p) {
                if (!rcnt[p]) continue;
                if (H.scnt[p][rank] != rcnt[p]) fail(GX_LOGIC_ERROR, "exchange: peer byte counts disagree");
                GX_CUDA(cudaStreamWaitEvent(s, H.ready[p], 0));
                GX_CUDA(cudaMemcpyAsync(recv + roff[p], H.send[p] + H.soff[p][rank], rcnt[p], cudaMemcpyDefault, s));
            }
            GX_CUDA(cudaEventRecord(H.done[rank], s));
            H.barrier(rank);
            for (int p = 0; p < size; ++p) GX_CUDA(cudaStreamWaitEvent(s, H.done[p], 0));
            H.barrier(rank);  // every rank has queued its waits before the events are re-recorded
        });
    }
};

// Host-staged transport: the exchange itself is the caller's (a callback over
// host buffers -- MPI, gloo, sockets), for boxes or tests where NCCL cannot
// connect the ranks (e.g. several ranks sharing one GPU). Device bytes are
// staged through pinned buffers; the grouping, owner gathers and scatters are
// the same kernels the NCCL path runs.
struct HostTransport : Transport {
    gx_host_alltoallv_fn fn = nullptr;
    void* user = nullptr;
    PinBuf<uint8_t> hs, hr;
    void call(const void* send, const uint64_t* scnt, void* recv, const uint64_t* rcnt) {
        const int rc = fn(user, send, scnt, recv, rcnt);
        if (rc) fail(GX_RUNTIME_ERROR, "host exchange callback failed (" + std::to_string(rc) + ")");
    }
    void counts(const uint64_t* send, uint64_t* recv, cudaStream_t) override {
        std::vector<uint64_t> c8(size, 8);
        call(send, c8.data(), recv, c8.data());
    }
    void alltoallv(const uint8_t* send, const uint64_t* soff, const uint64_t* scnt, uint8_t* recv,
                   const uint64_t* roff, const uint64_t* rcnt, cudaStream_t s) override {
        uint64_t ts = 0, tr = 0;
        for (int p = 0; p < size; ++p) {
            ts += scnt[p];
            tr += rcnt[p];
        }
        hs.reserve(std::max<uint64_t>(ts, 1));
        hr.reserve(std::max<uint64_t>(tr, 1));
        uint64_t o = 0;  // pack the send pieces densely in rank order
        for (int p = 0; p < size; ++p) {
            if (scnt[p]) GX_CUDA(cudaMemcpyAsync(hs.p + o, send + soff[p], scnt[p], cudaMemcpyDeviceToHost, s));
            o += scnt[p];
        }
        GX_CUDA(cudaStreamSynchronize(s));
        call(hs.p, scnt, hr.p, rcnt);
        o = 0;
        for (int p = 0; p < size; ++p) {
            if (rcnt[p]) GX_CUDA(cudaMemcpyAsync(recv + roff[p], hr.p + o, rcnt[p], cudaMemcpyHostToDevice, s));
            o += rcnt[p];
        }
        GX_CUDA(cudaStreamSynchronize(s));  // the pinned staging is reused by the next call
    }
};

}  // namespace gx

struct gx_comm {
    gx_ctx* ctx = nullptr;
    std::unique_ptr<gx::Transport> t;
};

namespace gx {

struct Bounds {
    uint64_t lo[65];
    int P;
};

__device__ __forceinline__ int owner_of(const Bounds& b, uint64_t v) {
    int lo = 0, hi = b.P;  // lo[lo] <= v < lo[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (b.lo[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void k_owner_keys(const uint32_t* __restrict__ ids, uint64_t n, Bounds b, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals, unsigned long long* __restrict__ counts) {
    __shared__ unsigned int hist[64];
    for (int p = threadIdx.x; p < b.P; p += blockDim.x) hist[p] = 0;
    __syncthreads();
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
        const int o = owner_of(b, ids[j]);
        keys[j] = (uint32_t)o;
        vals[j] = (uint32_t)j;
        atomicAdd(&hist[o], 1u);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < b.P; p += blockDim.x)
        if (hist[p]) atomicAdd(&counts[p], (unsigned long long)hist[p]);
}

// send_ids[q] = local id (at its owner) of request perm[q]
__global__ void k_local_ids(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ owner, uint64_t n, Bounds b, uint32_t* __restrict__ out) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x)
        out[q] = (uint32_t)(ids[perm[q]] - b.lo[owner[q]]);
}

// out row perm[q] <- local row ids[q] (a rank's own requests), 16-byte
// vectors, R rows in flight per warp
template <int VEC>
__global__ void k_gather_scatter(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ perm, uint64_t n,
                                 const uint8_t* __restrict__ store, uint8_t* __restrict__ out, uint64_t rb,
                                 uint8_t* __restrict__ out2, const uint32_t* __restrict__ idx2) {
    using V = typename std::conditional<VEC == 16, uint4, uint32_t>::type;
    constexpr int R = 4;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31, nvec = (uint32_t)(rb / VEC);
    for (uint64_t q0 = warp * R; q0 < n; q0 += nwarps * R) {
        const V* src[R];
        V* dst[R];
        V* dst2[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const uint64_t q = q0 + k < n ? q0 + k : q0;
            const uint32_t j = __ldg(perm + q);
            src[k] = reinterpret_cast<const V*>(store + (uint64_t)__ldg(ids + q) * rb);
            dst[k] = reinterpret_cast<V*>(out + (uint64_t)j * rb);
            dst2[k] = out2 ? reinterpret_cast<V*>(out2 + (uint64_t)__ldg(idx2 + j) * rb) : nullptr;
        }
        for (uint32_t c = lane; c < nvec; c += 32) {
            V t[R];
#pragma unroll
            for (int k = 0; k < R; ++k) t[k] = src[k][c];
#pragma unroll
            for (int k = 0; k < R; ++k)
                if (q0 + k < n) {
                    dst[k][c] = t[k];
                    if (out2) dst2[k][c] = t[k];
                }
        }
    }
}

static void launch_gather_scatter(const uint32_t* ids, const uint32_t* perm, uint64_t n, const uint8_t* store,
                                  uint8_t* out, uint64_t rb, int num_sms, cudaStream_t s, uint8_t* out2,
                                  const uint32_t* idx2) {
    if (!n) return;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n * 8 + 255) / 256, (uint64_t)num_sms * 8);
    if (rb % 16 == 0) k_gather_scatter<16><<<blocks, 256, 0, s>>>(ids, perm, n, store, out, rb, out2, idx2);
    else k_gather_scatter<4><<<blocks, 256, 0, s>>>(ids, perm, n, store, out, rb, out2, idx2);
    GX_CHECK_LAUNCH();
}

static Bounds make_bounds(uint64_t N, int P) {
    Bounds b{};
    b.P = P;
    for (int r = 0; r <= P; ++r) b.lo[r] = (uint64_t)((unsigned __int128)N * r / P);
    return b;
}

double part_fetch(gx_features* f, const uint32_t* d_ids, uint64_t n, uint8_t* d_out, cudaStream_t s,
                  uint8_t* out2, const uint32_t* idx2) {
    const auto t0 = std::chrono::steady_clock::now();
    gx_ctx* ctx = f->ctx;
    Transport& T = *f->comm->t;
    const int P = T.size;
    if (P == 1 && n == 0) return 0.0;  // nothing to exchange with nobody
    const uint64_t rb = f->row_bytes;
    if (!f->part) f->part.reset(new PartScratch());
    PartScratch& x = *f->part;
    const Bounds b = make_bounds(f->n, P);
    // (1) owners, per-owner counts, stable grouping by owner
    x.counts.reserve(64);
    GX_CUDA(cudaMemsetAsync(x.counts.p, 0, 64 * 8, s));
    x.keys.reserve(n + 1);
    x.keys_alt.reserve(n + 1);
    x.vals.reserve(n + 1);
    x.vals_alt.reserve(n + 1);
    x.send_ids.reserve(n + 1);
    const uint32_t* perm = x.vals.p;
    const uint32_t* owner = x.keys.p;
    if (n) {
        k_owner_keys<<<ctx->num_sms * 2, 256, 0, s>>>(d_ids, n, b, x.keys.p, x.vals.p, x.counts.p);
        GX_CHECK_LAUNCH();
        if (P > 1) {
            int bits = 1;
            while ((1 << bits) < P) ++bits;
            cub::DoubleBuffer<uint32_t> dk(x.keys.p, x.keys_alt.p), dv(x.vals.p, x.vals_alt.p);
            size_t tb = 0;
            GX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, bits, s));
            x.cub_tmp.reserve(tb + 16);
            GX_CUDA(cub::DeviceRadixSort::SortPairs(x.cub_tmp.p, tb, dk, dv, (int)n, 0, bits, s));
            perm = dv.Current();
            owner = dk.Current();
        }
        k_local_ids<<<ctx->num_sms * 2, 256, 0, s>>>(d_ids, perm, owner, n, b, x.send_ids.p);
        GX_CHECK_LAUNCH();
    }
    std::vector<uint64_t> scnt(P), rcnt(P);
    {
        std::vector<unsigned long long> h(P);
        GX_CUDA(cudaMemcpyAsync(h.data(), x.counts.p, P * 8, cudaMemcpyDeviceToHost, s));
        GX_CUDA(cudaStreamSynchronize(s));
        for (int p = 0; p < P; ++p) scnt[p] = h[p];
    }
    // (2) counts, then ids. This rank's own requests never touch the network:
    // they are served straight from the local partition (step 3a).
    T.counts(scnt.data(), rcnt.data(), s);
    const int me = T.rank;
    std::vector<uint64_t> soff(P + 1, 0), roff(P + 1, 0);
    for (int p = 0; p < P; ++p) {
        soff[p + 1] = soff[p] + scnt[p];
        roff[p + 1] = roff[p] + (p == me ? 0 : rcnt[p]);
    }
    const uint64_t nrecv = roff[P];  // rows other ranks asked this rank for
    x.recv_ids.reserve(nrecv + 1);
    std::vector<uint64_t> sb(P), so(P), rbb(P), ro(P);
    for (int p = 0; p < P; ++p) {
        sb[p] = p == me ? 0 : scnt[p] * 4;
        so[p] = soff[p] * 4;
        rbb[p] = p == me ? 0 : rcnt[p] * 4;
        ro[p] = roff[p] * 4;
    }
    if (P > 1)
        T.alltoallv((const uint8_t*)x.send_ids.p, so.data(), sb.data(), (uint8_t*)x.recv_ids.p, ro.data(), rbb.data(),
                    s);
    // (3a) own requests: local row -> request position in one pass
    launch_gather_scatter(x.send_ids.p + soff[me], perm + soff[me], scnt[me], f->dev.p, d_out, rb, ctx->num_sms, s,
                          out2, idx2);
    // (3b) serve the other ranks' requests from this rank's partition (local ids)
    x.send_rows.reserve(std::max<uint64_t>(nrecv * rb, 16));
    x.dummy.reserve(8);
    if (nrecv) {
        cudaStream_t saved = ctx->launch_stream;
        ctx->launch_stream = s;
        try {
            launch_gather_resolved(ctx, x.recv_ids.p, nullptr, nrecv, nullptr, f->dev.p, rb, x.send_rows.p, x.dummy.p);
        } catch (...) {
            ctx->launch_stream = saved;
            throw;
        }
        ctx->launch_stream = saved;
    }
    // (4) rows back into their request-grouped slots; scatter to their requests
    const uint64_t n_remote = n - scnt[me];
    x.recv_rows.reserve(std::max<uint64_t>(n * rb, 16));
    for (int p = 0; p < P; ++p) {
        sb[p] = p == me ? 0 : rcnt[p] * rb;  // rows go back to whoever asked
        so[p] = roff[p] * rb;
        rbb[p] = p == me ? 0 : scnt[p] * rb;
        ro[p] = soff[p] * rb;
    }
    if (P > 1) {
        T.alltoallv(x.send_rows.p, so.data(), sb.data(), x.recv_rows.p, ro.data(), rbb.data(), s);
        launch_scatter_rows(x.recv_rows.p, perm, soff[me], d_out, rb, ctx->num_sms, s, out2, idx2);
        const uint64_t tail = soff[me] + scnt[me];
        launch_scatter_rows(x.recv_rows.p + tail * rb, perm + tail, n - tail, d_out, rb, ctx->num_sms, s, out2, idx2);
    }
    // counters
    f->xstats.calls += 1;
    f->xstats.rows_requested += n;
    f->xstats.rows_remote += n_remote;
    f->xstats.rows_served += nrecv + scnt[me];
    f->xstats.bytes_sent += n_remote * 4 + nrecv * rb;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    f->xstats.ms += ms;
    return ms;
}

}  // namespace gx

using namespace gx;

static gx_features* new_partition(gx_ctx* ctx, gx_comm* comm, uint64_t N, uint32_t dim, uint32_t sw) {
    if (!ctx || !comm) fail(GX_INVALID_ARGUMENT, "a partitioned table needs a context and a communicator");
    if (comm->ctx != ctx) fail(GX_INVALID_ARGUMENT, "communicator belongs to another context");
    if (sw != 4 && sw != 2) fail(GX_INVALID_ARGUMENT, "scalar_width must be 4 or 2");
    if (dim < 1) fail(GX_INVALID_ARGUMENT, "dim must be >= 1");
    if (N >= 0xFFFFFFFFull) fail(GX_OVERFLOW, "num_nodes exceeds the u32 device id range");
    auto f = new gx_features();
    f->ctx = ctx;
    f->n = N;
    f->dim = dim;
    f->scalar_width = sw;
    f->row_bytes = (uint64_t)dim * sw;
    f->backing = GX_BACKING_PARTITIONED;
    f->comm = comm;
    const Bounds b = make_bounds(N, comm->t->size);
    f->part_lo = b.lo[comm->t->rank];
    f->part_hi = b.lo[comm->t->rank + 1];
    try {
        f->dev.alloc(std::max<uint64_t>((f->part_hi - f->part_lo) * f->row_bytes, 16));
    } catch (...) {
        delete f;
        throw;
    }
    f->rows_dev_view = nullptr;  // rows are reached only through part_fetch
    return f;
}

extern "C" {

gx_status gx_comm_unique_id(void* id_out) {
    return guard([&] {
        ncclUniqueId id;
        GX_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

gx_status gx_comm_init_nccl(gx_ctx* ctx, const void* id, int nranks, int rank, gx_comm** out) {
    return guard([&] {
        if (!ctx) fail(GX_INVALID_ARGUMENT, "null context");
        if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) fail(GX_INVALID_ARGUMENT, "bad rank / size");
        auto t = std::make_unique<NcclTransport>();
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        GX_CUDA(cudaSetDevice(ctx->device));
        GX_NCCL(nccl().CommInitRank(&t->comm, nranks, uid, rank));
        t->rank = rank;
        t->size = nranks;
        auto c = new gx_comm();
        c->ctx = ctx;
        c->t = std::move(t);
        *out = c;
    });
}

gx_status gx_comm_init_local(gx_ctx* const* ctxs, int nranks, gx_comm** outs) {
    return guard([&] {
        if (nranks < 1 || nranks > 64) fail(GX_INVALID_ARGUMENT, "bad size");
        auto hub = std::make_shared<LocalHub>(nranks);
        for (int r = 0; r < nranks; ++r) {
            if (!ctxs[r]) fail(GX_INVALID_ARGUMENT, "null context");
            auto t = std::make_unique<LocalTransport>();
            t->hub = hub;
            t->rank = r;
            t->size = nranks;
            auto c = new gx_comm();
            c->ctx = ctxs[r];
            c->t = std::move(t);
            outs[r] = c;
        }
    });
}

gx_status gx_comm_init_host(gx_ctx* ctx, int nranks, int rank, gx_host_alltoallv_fn fn, void* user,
                            gx_comm** out) {
    return guard([&] {
        if (!ctx || !fn) fail(GX_INVALID_ARGUMENT, "null context or callback");
        if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) fail(GX_INVALID_ARGUMENT, "bad rank / size");
        auto t = std::make_unique<HostTransport>();
        t->fn = fn;
        t->user = user;
        t->rank = rank;
        t->size = nranks;
        auto c = new gx_comm();
        c->ctx = ctx;
        c->t = std::move(t);
        *out = c;
    });
}

void gx_comm_destroy(gx_comm* c) { delete c; }
int gx_comm_rank(const gx_comm* c) { return c ? c->t->rank : -1; }
int gx_comm_size(const gx_comm* c) { return c ? c->t->size : 0; }

gx_status gx_partition_bounds(uint64_t N, int P, int r, uint64_t* lo, uint64_t* hi) {
    return guard([&] {
        if (P < 1 || P > 64 || r < 0 || r >= P) fail(GX_INVALID_ARGUMENT, "bad rank / size");
        const Bounds b = make_bounds(N, P);
        *lo = b.lo[r];
        *hi = b.lo[r + 1];
    });
}

gx_status gx_features_partitioned_from_host(gx_ctx* ctx, gx_comm* comm, uint64_t N, uint32_t dim, uint32_t sw,
                                            const void* rows, gx_features** out) {
    return guard([&] {
        gx_features* f = new_partition(ctx, comm, N, dim, sw);
        const uint64_t bytes = (f->part_hi - f->part_lo) * f->row_bytes;
        if (bytes) {
            const cudaError_t e = cudaMemcpy(f->dev.p, rows, bytes, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                delete f;
                fail(GX_CUDA_ERROR, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
            }
        }
        *out = f;
    });
}

gx_status gx_features_partitioned_generate(gx_ctx* ctx, gx_comm* comm, uint64_t N, uint32_t dim, uint32_t sw,
                                           uint64_t vseed, gx_features** out) {
    return guard([&] {
        gx_features* f = new_partition(ctx, comm, N, dim, sw);
        try {
            launch_features(f->dev.p, f->part_hi - f->part_lo, dim, sw, vseed, f->part_lo, ctx->num_sms, ctx->stream);
            GX_CUDA(cudaStreamSynchronize(ctx->stream));
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

gx_status gx_features_partitioned_open(gx_ctx* ctx, gx_comm* comm, const char* path, gx_features** out) {
    return guard([&] {
        // header checks as FeatureFile::open, through a host-only file handle
        gx_features* hf = nullptr;
        const gx_status st = gx_features_open(nullptr, path, GX_BACKING_FILE, &hf);
        if (st != GX_OK) fail(st, gx_last_error());
        std::unique_ptr<gx_features> keep(hf);
        gx_features* f = new_partition(ctx, comm, hf->n, hf->dim, hf->scalar_width);
        try {
            // this rank's rows are one contiguous byte range: sequential reads
            RowReader& rd = *hf->file;
            const uint64_t rb = f->row_bytes, CH = 64ull << 20;
            const uint64_t lo = rd.poff + f->part_lo * rb, hi = rd.poff + f->part_hi * rb;
            PinBuf<uint8_t> pin;
            pin.alloc(std::min<uint64_t>(hi - lo, CH) + 2 * kPage);
            const int bfd = ::open(path, O_RDONLY);
            if (bfd < 0) fail(GX_RUNTIME_ERROR, std::string("cannot open: ") + path);
            for (uint64_t o = lo; o < hi; o += CH) {
                const uint64_t c = std::min(CH, hi - o);
                uint64_t done = 0;
                while (done < c) {
                    const ssize_t r = ::pread(bfd, pin.p + done, c - done, (off_t)(o + done));
                    if (r <= 0) {
                        ::close(bfd);
                        fail(GX_RUNTIME_ERROR, std::string("truncated feature file: ") + path);
                    }
                    done += (uint64_t)r;
                }
                GX_CUDA(cudaMemcpy(f->dev.p + (o - lo), pin.p, c, cudaMemcpyHostToDevice));
            }
            ::close(bfd);
        } catch (...) {
            delete f;
            throw;
        }
        *out = f;
    });
}

gx_status gx_features_exchange_stats(const gx_features* f, gx_exchange_stats* out) {
    return guard([&] {
        if (!f || !out) fail(GX_INVALID_ARGUMENT, "null handle");
        *out = f->xstats;
    });
}

}  // extern "C"
