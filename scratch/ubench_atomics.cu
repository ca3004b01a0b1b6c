// Microbenchmark: smem / global atomic throughput on B200 (design input for bucketing + spreading)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x>>16; x*=0x7feb352d; x^=x>>15; x*=0x846ca68b; x^=x>>16; return x; }
template<int NB, int MODE>
__global__ void k_smem(int iters, uint32_t* out){
  extern __shared__ uint32_t sh[];
  for(int i=threadIdx.x;i<NB;i+=blockDim.x) sh[i]=0;
  __syncthreads();
  uint32_t s = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  uint32_t acc=0;
  for(int it=0; it<iters; ++it){
    s = hsh(s+it);
    uint32_t b = s & (NB-1);
    if (MODE==0) atomicAdd(&sh[b], 1u);              // RED-style (no return used)
    else if (MODE==1) acc += atomicAdd(&sh[b], 1u);  // with return (rank)
    else if (MODE==2) atomicAdd(reinterpret_cast<float*>(&sh[b]), 1.0f);
  }
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=sh[0]+acc;
}
// per-lane private grid: [W][32] layout, RMW without atomics
__global__ void k_private(int iters, float* out){
  extern __shared__ float shf[];
  const int W=32; int lane=threadIdx.x&31, warp=threadIdx.x>>5;
  float* g = shf + warp*W*32;
  for(int i=lane;i<W*32;i+=32) g[i]=0.f;
  __syncwarp();
  uint32_t s = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){
    s = hsh(s+it);
    int c = s % (W-6);
    #pragma unroll
    for(int t=0;t<6;++t) g[(c+t)*32+lane] += 1.0f;
  }
  __syncwarp();
  if(lane==0) out[blockIdx.x*32+warp]=g[0];
}
template<int MODE>
__global__ void k_glob(int iters, uint32_t* arr, uint32_t mask, uint32_t* out){
  uint32_t s = hsh(blockIdx.x*blockDim.x+threadIdx.x); uint32_t acc=0;
  for(int it=0; it<iters; ++it){ s=hsh(s+it); uint32_t b=s&mask;
    if(MODE==0) atomicAdd(&arr[b],1u); else acc+=atomicAdd(&arr[b],1u); }
  if(acc==0xFFFFFFFF) out[0]=acc;
}
int main(){
  uint32_t* out; CK(cudaMalloc(&out, 1<<24));
  uint32_t* arr; CK(cudaMalloc(&arr, (size_t)4<<24)); CK(cudaMemset(arr,0,(size_t)4<<24));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks=148*4, threads=512, iters=256; double nops=(double)blocks*threads*iters; float ms;
  auto run=[&](const char* name, auto launch){ launch(); cudaDeviceSynchronize(); cudaEventRecord(a); for(int r=0;r<5;++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); ms/=5; printf("%-40s %8.3f ms  %8.2f Gop/s  (%.3f cyc/lane/SM @1.9GHz)\n", name, ms, nops/ms/1e6, (ms*1e-3*1.9e9*148)/nops); };
  cudaFuncSetAttribute(k_smem<16384,0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_smem<16384,1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_smem<16384,2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  run("smem atomicAdd u32 16K bins (no ret)", [&]{ k_smem<16384,0><<<blocks,threads,65536>>>(iters,out); });
  run("smem atomicAdd u32 16K bins (ret)", [&]{ k_smem<16384,1><<<blocks,threads,65536>>>(iters,out); });
  run("smem atomicAdd f32 16K bins", [&]{ k_smem<16384,2><<<blocks,threads,65536>>>(iters,out); });
  run("smem atomicAdd u32 64 bins (no ret)", [&]{ k_smem<64,0><<<blocks,threads,256>>>(iters,out); });
  run("smem atomicAdd f32 64 bins", [&]{ k_smem<64,2><<<blocks,threads,256>>>(iters,out); });
  cudaFuncSetAttribute(k_private, cudaFuncAttributeMaxDynamicSharedMemorySize, 16*32*32*4);
  { double save=nops; nops*=6; run("private lane grid RMW (per tap)", [&]{ k_private<<<blocks,threads,16*32*32*4>>>(iters,(float*)out); }); nops=save; }
  run("global atomicAdd u32 16M addr (no ret)", [&]{ k_glob<0><<<blocks,threads>>>(iters,arr,(1u<<24)-1,out); });
  run("global atomicAdd u32 16M addr (ret)", [&]{ k_glob<1><<<blocks,threads>>>(iters,arr,(1u<<24)-1,out); });
  run("global atomicAdd u32 4M addr (ret)", [&]{ k_glob<1><<<blocks,threads>>>(iters,arr,(1u<<22)-1,out); });
  CK(cudaGetLastError());
  return 0;
}
