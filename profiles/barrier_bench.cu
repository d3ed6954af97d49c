// Grid-barrier latency on one B200: N back-to-back grid_sync() calls in a
// cooperative kernel (gx_common.cuh's barrier, both forms), for the grid
// shapes the inspector (148 x 1024) and the sampler (592 x 256) use.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../include \
//        -I../paper_2208_09151_b200/csrc barrier_bench.cu -o barrier_bench
#include <cstdio>

#include "gx_common.cuh"

namespace gx {
void set_last_error(const std::string&) {}
}  // namespace gx
using namespace gx;

__global__ void k_barriers(GridBarrier* b, int n, unsigned long long* sink) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
        grid_sync(b);
        acc += i;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = acc;
}

int main() {
    GridBarrier* b;
    unsigned long long* sink;
    cudaMalloc(&b, sizeof(GridBarrier));
    cudaMalloc(&sink, 8);
    cudaStream_t st;
    cudaStreamCreate(&st);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int shapes[3][2] = {{sms, 1024}, {sms * 4, 256}, {sms * 2, 512}};
    for (int mono = 1; mono >= 0; --mono) {
        for (auto& sh : shapes) {
            const int n = 2000;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e9f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemsetAsync(b, 0, sizeof(GridBarrier), st);
                if (!mono) cudaMemsetAsync(&b->count64, 0xff, 8, st);
                int nn = n;
                void* args[] = {&b, &nn, &sink};
                cudaEventRecord(e0, st);
                cudaLaunchCooperativeKernel((void*)k_barriers, dim3(sh[0]), dim3(sh[1]), args, 0, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("{\"barrier\": \"%s\", \"ctas\": %d, \"threads\": %d, \"us_per_barrier\": %.3f}\n",
                   mono ? "monotonic" : "generation", sh[0], sh[1], best * 1e3 / n);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
