// gx_common.cuh -- shared device/host plumbing for the B200 hot path.
//
// Error model: internal code throws gx::Error(status, msg); every extern "C"
// entry point runs inside gx::guard(), which maps it to gx_status and stores
// the message for gx_last_error() (include/gx_b200.h).
#pragma once
#include <cstdlib>
#include <atomic>

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gx_b200.h"

namespace gx {

// Global nanosecond timer (phase tracing: GX_SAMPLER_TRACE, GX_INSPECT_TRACE).
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Tuning knob from the environment (read once per call site); def when unset.
inline int env_int(const char* name, int def) {
    const char* e = std::getenv(name);
    return (e && *e) ? std::atoi(e) : def;
}

// Kernel attributes (cudaFuncSetAttribute) and occupancy results are per
// device: launch-configuration caches are kept per device ordinal so a second
// context on another GPU of the same process sets them up again.
template <class T>
struct PerDevice {
    std::mutex mu;
    std::map<int, T> m;
    // the entry of `dev`, value-initialised on first use; callers that fill it
    // lazily hold lock() while they do
    T& at(int dev) { return m[dev]; }
    std::unique_lock<std::mutex> lock() { return std::unique_lock<std::mutex>(mu); }
};
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Persistent grid-barrier kernels (sampler, inspector) are sized to be fully
// co-resident (occupancy query x SMs). GX_COOP=1 launches them with
// cudaLaunchCooperativeKernel; 0 uses an ordinary launch, which lets them share
// SMs with the executor stream's gathers -- safe because nothing those kernels
// wait on depends on this grid, so CTAs not yet resident are scheduled as
// the gather CTAs retire.
inline bool coop_launch() {
    static const bool v = env_int("GX_COOP", 1) != 0;
    return v;
}


struct Error : std::exception {
    gx_status status;
    std::string msg;
    Error(gx_status s, std::string m) : status(s), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] inline void fail(gx_status s, const std::string& m) { throw Error(s, m); }

void set_last_error(const std::string& m);

template <class F>
gx_status guard(F&& f) {
    try {
        f();
        return GX_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return GX_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return GX_RUNTIME_ERROR;
    }
}

#define GX_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess)                                                              \
            ::gx::fail(GX_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// Every launch of one of this library's kernels is followed by GX_CHECK_LAUNCH(),
// which also counts it (gx_pipeline_stats.kernel_launches).
inline std::atomic<uint64_t> g_kernel_launches{0};
#define GX_CHECK_LAUNCH()                                                  \
    do {                                                                   \
        ::gx::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
        GX_CUDA(cudaGetLastError());                                       \
    } while (0)

constexpr uint32_t kNever = 0xFFFFFFFFu;     // "no further access" / empty key
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kPage = 4096;

// ---------------------------------------------------------------------------
// Device RNG: SplitMix64 as a counter-based generator (common.hpp:68-101).
// Draw t (0-based) of SplitMix64(seed) == mix64(seed + t*gamma); bounded(n)
// == umulhi(draw, n). Verified bit-exact against the sequential stream.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += kGamma;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t index) {
    return mix64(base ^ mix64(index));
}
__device__ __forceinline__ uint64_t draw_bounded(uint64_t seed, uint64_t t, uint64_t n) {
    return __umul64hi(mix64(seed + t * kGamma), n);
}
__host__ __device__ __forceinline__ uint64_t pages_touched(uint64_t lo, uint64_t hi) {
    return hi <= lo ? 0 : (hi - 1) / kPage - lo / kPage + 1;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// ---------------------------------------------------------------------------
// Grid-wide barrier for persistent kernels launched cooperatively (all CTAs
// co-resident). Default: one monotonically increasing 64-bit arrival count
// (zeroed by the host before each launch, `barrier_reset`): barrier k of a
// launch completes when the count reaches k x gridDim, so a CTA's arrival is
// one atomic and the waiters poll the same word -- no second hop through a
// generation flag written by the last arriver. GX_BARRIER=0 (host knob,
// `count64` left at ~0): the previous count + generation barrier.
// ---------------------------------------------------------------------------
struct GridBarrier {
    unsigned int count;
    unsigned int gen;
    unsigned long long count64;
};

__device__ __forceinline__ unsigned cluster_ctas() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void grid_sync(GridBarrier* b) {
    __syncthreads();
    if (gridDim.x == 1) return;  // one-CTA launches (narrow inspector traces): the CTA barrier suffices
    if (gridDim.x == cluster_ctas()) {
        // the whole grid is one thread-block cluster (narrow inspector traces):
        // the hardware cluster barrier, release/acquire at cluster scope, which
        // orders the CTAs' global-memory writes before the other CTAs' reads
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    if (threadIdx.x == 0) {
        volatile unsigned long long* vc = &b->count64;
        if (*vc != ~0ull) {  // monotonic arrival count (host-zeroed per launch)
#ifndef GX_BARRIER_FENCES
            // release on the arrival (cumulative over the CTA's writes ordered
            // before it by the __syncthreads above), acquire on the polls
            unsigned long long old;
            asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(&b->count64) : "memory");
            const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
            unsigned long long cur;
            do {
                asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(cur) : "l"(&b->count64) : "memory");
            } while (cur < target);
#else
            __threadfence();
            const unsigned long long old = atomicAdd(&b->count64, 1ull);
            const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
            while (*vc < target) {
            }
            __threadfence();
#endif
        } else {
            volatile unsigned int* vgen = &b->gen;
            unsigned int g = *vgen;
            __threadfence();
            unsigned int arrived = atomicAdd(&b->count, 1u);
            if (arrived == gridDim.x - 1) {
                b->count = 0;
                __threadfence();
                atomicAdd(&b->gen, 1u);
            } else {
                unsigned ns = 32;
                while (*vgen == g) {
                    __nanosleep(ns);
                    if (ns < 256) ns <<= 1;
                }
            }
            __threadfence();
        }
    }
    __syncthreads();
}

// host: before every launch that synchronises through `b` on stream `st`
inline void barrier_reset(GridBarrier* b, cudaStream_t st) {
    static const bool mono = [] {
        const char* e = std::getenv("GX_BARRIER");
        return !e || std::atoi(e) != 0;
    }();
    // count64 = 0 selects the monotonic barrier, ~0 the generation barrier
    GX_CUDA(cudaMemsetAsync(&b->count64, mono ? 0 : 0xff, sizeof(unsigned long long), st));
}

// ---------------------------------------------------------------------------
// Warp / block scans
// ---------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive block scan; `total` gets the block sum. smem needs 33 T.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    T inc = warp_incl_scan(v);
    if (lane == 31) smem[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T s = lane < nw ? smem[lane] : T(0);
        T si = warp_incl_scan(s);
        if (lane < nw) smem[lane] = si - s;
        if (lane == nw - 1) smem[32] = si;
    }
    __syncthreads();
    T r = inc - v + smem[wid];
    total = smem[32];
    __syncthreads();
    return r;
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
    T tot;
    block_excl_scan(v, smem, tot);
    return tot;
}

// ---------------------------------------------------------------------------
// RAII device / pinned buffers
// ---------------------------------------------------------------------------
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    void alloc(size_t count) {
        release();
        static const bool trace = std::getenv("GX_ALLOC_TRACE") != nullptr;  // growth diagnostics
        if (trace && count) std::fprintf(stderr, "[gx alloc] %zu bytes\n", count * sizeof(T));
        if (count) {
            cudaError_t e = cudaMalloc(&p, count * sizeof(T));
            if (e != cudaSuccess) {
                p = nullptr;
                fail(GX_CUDA_ERROR, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                        " bytes failed: " + cudaGetErrorString(e));
            }
        }
        n = count;
    }
    // grow-only, with 25% headroom so per-superbatch size jitter does not
    // re-allocate (cudaMalloc/cudaFree stall the stream); buffers of 4 GiB and
    // more get 1/32 (a resident S = 500 superbatch is 46 GB of rows: 25 % would
    // be 11 GB of HBM for jitter of about 1 %)
    static size_t grow_to(size_t count, size_t cur) {
        const size_t big = (size_t(4) << 30) / sizeof(T);
        const size_t c = count + (count >= big ? count / 32 : count / 4);
        const size_t g = cur + (cur >= big ? cur / 32 : cur / 4);
        return std::max(c, g) + 64;
    }
    // elements reserve(count) would hold afterwards
    size_t reserved_after(size_t count) const { return count > n ? grow_to(count, n) : n; }
    void reserve(size_t count) {
        if (count > n) alloc(grow_to(count, n));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

template <class T>
struct PinBuf {
    T* p = nullptr;
    size_t n = 0;
    PinBuf() = default;
    ~PinBuf() { release(); }
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    void alloc(size_t count, unsigned flags = cudaHostAllocDefault) {
        release();
        if (count) GX_CUDA(cudaHostAlloc(&p, count * sizeof(T), flags));
        n = count;
    }
    void reserve(size_t count) {
        if (count > n) alloc(count);
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
    }
};

inline unsigned ceil_div(uint64_t a, uint64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace gx
