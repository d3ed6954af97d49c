// Random-access ceiling for the sampler's draw loop (phase E of k_sample), one B200.
// The phase is bound by scattered 4- and 8-byte accesses, not by bytes.
// This measures the rates the memory system sustains for the access mixes one
// draw makes, with as many accesses in flight as the GPU holds:
//   idx4     random 4-byte loads from a 6.4 GB array (the CSC indices)
//   idx4_l2  the same from a 64 MB array (L2-resident)
//   probe8   random 8-byte load, then a CAS on the same word, 0.4 GB table
//            (the last layer's dedup tables at papers shape)
//   draw     idx4 -> hash of the loaded id -> probe8, dependent (one draw)
// Addresses come from a counter hash, so no index array adds traffic.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o random_sectors random_sectors.cu
// Output of one run: r02z_random_sectors.txt.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int U>
__global__ void __launch_bounds__(256, 4) k_idx(const uint32_t* __restrict__ a, uint64_t n, uint32_t per, uint32_t* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t i = 0; i < per; i += U) {
        uint32_t v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) v[j] = __ldg(a + mix(t * 1000003ull + i + j) % n);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += v[j];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256, 4) k_probe(unsigned long long* tab, uint64_t n, uint32_t per, uint32_t* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t i = 0; i < per; i += U) {
        uint64_t s[U];
        unsigned long long g[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            s[j] = mix(t * 7919ull + i + j) % n;
            g[j] = __ldcg(tab + s[j]);
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (g[j] == ~0ull) g[j] = atomicCAS(tab + s[j], ~0ull, t << 32 | i);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += (uint32_t)g[j];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256, 4) k_draw(const uint32_t* __restrict__ a, uint64_t n, unsigned long long* tab,
                                                 uint64_t m, uint32_t per, uint32_t* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (uint32_t i = 0; i < per; i += U) {
        uint32_t c[U];
        unsigned long long g[U];
        uint64_t s[U];
#pragma unroll
        for (int j = 0; j < U; ++j) c[j] = __ldg(a + mix(t * 1000003ull + i + j) % n);
#pragma unroll
        for (int j = 0; j < U; ++j) {
            s[j] = mix(c[j] ^ (t << 20)) % m;
            g[j] = __ldcg(tab + s[j]);
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (g[j] == ~0ull) g[j] = atomicCAS(tab + s[j], ~0ull, (unsigned long long)c[j] << 32 | i);
#pragma unroll
        for (int j = 0; j < U; ++j) acc += (uint32_t)g[j];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

template <class F>
static float timeit(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t nidx = 1614950152ull, nsmall = 16ull << 20, ntab = 50ull << 20;  // 6.46 GB, 64 MB, 0.4 GB
    uint32_t *a, *out;
    unsigned long long* tab;
    cudaMalloc(&a, nidx * 4);
    cudaMalloc(&tab, ntab * 8);
    cudaMalloc(&out, 64);
    cudaMemset(a, 1, nidx * 4);
    const dim3 grid(sms * 4), block(256);
    const uint32_t per = 64;
    const double ops = (double)grid.x * block.x * per;
    auto rate = [&](float ms) { return ops / (ms * 1e-3) / 1e9; };
    float ms;
    ms = timeit([&] { k_idx<4><<<grid, block>>>(a, nidx, per, out); });
    printf("idx4     (6.4 GB, 4 in flight)        %7.3f ms  %6.1f G accesses/s\n", ms, rate(ms));
    ms = timeit([&] { k_idx<8><<<grid, block>>>(a, nidx, per, out); });
    printf("idx4     (6.4 GB, 8 in flight)        %7.3f ms  %6.1f G accesses/s\n", ms, rate(ms));
    ms = timeit([&] { k_idx<4><<<grid, block>>>(a, nsmall, per, out); });
    printf("idx4_l2  (64 MB, 4 in flight)         %7.3f ms  %6.1f G accesses/s\n", ms, rate(ms));
    auto clear = [&] { cudaMemset(tab, 0xff, ntab * 8); };
    for (int U : {2, 4}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            clear();
            cudaEventRecord(e0);
            if (U == 2) k_probe<2><<<grid, block>>>(tab, ntab, per, out);
            else k_probe<4><<<grid, block>>>(tab, ntab, per, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("probe8   (0.4 GB, load+CAS, %d in flt) %7.3f ms  %6.1f G accesses/s\n", U, best, rate(best));
        best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            clear();
            cudaEventRecord(e0);
            if (U == 2) k_draw<2><<<grid, block>>>(a, nidx, tab, ntab, per, out);
            else k_draw<4><<<grid, block>>>(a, nidx, tab, ntab, per, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("draw     (idx4 -> probe8, %d in flight) %7.3f ms  %6.1f G draws/s\n", U, best, rate(best));
    }
    printf("(%u threads x %u accesses = %.1fM per launch; err %s)\n", grid.x * block.x, per, ops / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
