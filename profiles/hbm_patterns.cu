// HBM access-pattern microbenchmark (512-byte rows, one B200): the realistic ceilings
// for the executor kernels. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// -o hbm_patterns hbm_patterns.cu; output of one run: r01s6_hbm_patterns.txt.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
__device__ __forceinline__ uint4 ldnc(const uint4* p){uint4 r;asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];":"=r"(r.x),"=r"(r.y),"=r"(r.z),"=r"(r.w):"l"(p));return r;}
__device__ __forceinline__ void stna(uint4* p,const uint4&v){asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"::"l"(p),"r"(v.x),"r"(v.y),"r"(v.z),"r"(v.w));}
// warp moves R rows of 512B: src row sidx[k] -> dst row didx[k]
template<int R> __global__ void __launch_bounds__(256,3) k_move(const uint32_t* sidx,const uint32_t* didx,uint32_t n,const uint8_t* src,uint8_t* dst){
  uint32_t lane=threadIdx.x&31, warp=(blockIdx.x*blockDim.x+threadIdx.x)>>5, nw=(gridDim.x*blockDim.x)>>5;
  for(uint32_t r0=warp*R;r0<n;r0+=nw*R){
    uint32_t nr=min(n-r0,(uint32_t)R);
    const uint8_t* s=nullptr; uint8_t* d=nullptr;
    if(lane<nr){ s=src+(uint64_t)(sidx?sidx[r0+lane]:r0+lane)*512; d=dst+(uint64_t)(didx?didx[r0+lane]:r0+lane)*512; }
    uint4 t[R];
#pragma unroll
    for(int q=0;q<R;++q){ const uint4* sq=(const uint4*)__shfl_sync(~0u,(unsigned long long)s,q); if(q<(int)nr) t[q]=ldnc(sq+lane);}
#pragma unroll
    for(int q=0;q<R;++q){ uint4* dq=(uint4*)__shfl_sync(~0u,(unsigned long long)d,q); if(q<(int)nr) stna(dq+lane,t[q]);}
  }
}
// write-only: fill dst rows didx with a constant
__global__ void __launch_bounds__(256) k_write(const uint32_t* didx,uint32_t n,uint8_t* dst){
  uint32_t lane=threadIdx.x&31, warp=(blockIdx.x*blockDim.x+threadIdx.x)>>5, nw=(gridDim.x*blockDim.x)>>5;
  uint4 v=make_uint4(1,2,3,4);
  for(uint32_t r=warp;r<n;r+=nw){ uint8_t* d=dst+(uint64_t)(didx?didx[r]:r)*512; stna((uint4*)d+lane,v);}
}
int main(){
  const uint32_t N=18000000, M=6000000; // dst rows (batch), src rows
  uint8_t *src,*dst; uint32_t *perm,*rs;
  cudaMalloc(&src,(size_t)M*512*2); cudaMalloc(&dst,(size_t)N*512); cudaMalloc(&perm,N*4); cudaMalloc(&rs,N*4);
  std::vector<uint32_t> h(N); for(uint32_t i=0;i<N;++i)h[i]=i; std::mt19937 g(1); std::shuffle(h.begin(),h.end(),g);
  cudaMemcpy(perm,h.data(),N*4,cudaMemcpyHostToDevice);
  for(uint32_t i=0;i<N;++i)h[i]=g()%(2*M); cudaMemcpy(rs,h.data(),N*4,cudaMemcpyHostToDevice);
  cudaMemset(dst,0,(size_t)N*512); cudaMemset(src,1,(size_t)M*512*2);
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run=[&](const char* name,auto f,double bytes){ for(int w=0;w<3;++w)f(); cudaEventRecord(a); for(int i=0;i<10;++i)f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); ms/=10; printf("%-40s %.3f ms  %.0f GB/s\n",name,ms,bytes/ms/1e6);};
  uint32_t n=12000000;
  run("seq copy (read seq, write seq)",[&]{k_move<8><<<sms*3,256>>>(nullptr,nullptr,n,src,dst);},2.0*n*512);
  run("gather (read rand, write seq)",[&]{k_move<8><<<sms*3,256>>>(rs,nullptr,n,src,dst);},2.0*n*512);
  run("scatter (read seq, write rand)",[&]{k_move<8><<<sms*3,256>>>(nullptr,perm,n,src,dst);},2.0*n*512);
  run("rand-rand",[&]{k_move<8><<<sms*3,256>>>(rs,perm,n,src,dst);},2.0*n*512);
  run("write seq",[&]{k_write<<<sms*8,256>>>(nullptr,N,dst);},1.0*N*512);
  run("write rand",[&]{k_write<<<sms*8,256>>>(perm,N,dst);},1.0*N*512);
  cudaError_t e=cudaGetLastError(); printf("err %s\n",cudaGetErrorString(e));
}
