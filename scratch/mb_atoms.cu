// microbenchmark: conflict-free shared-memory read-modify-write (LDS + STS) vs RED.shared.add (u32, no return)
// 6 taps per step into a [32 cells][128 slots] column (bank = lane), random cell per lane and step
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned* out) {
  __shared__ float fcol[2][32 * 128];
  int (*icol)[32 * 128] = reinterpret_cast<int (*)[32 * 128]>(fcol);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = (warp & 3) * 32 + lane, cp = warp >> 2;   // 16 warps: 4 quadrants x 4 copies... use cp & 1
  for (int i = threadIdx.x; i < 2 * 32 * 128; i += blockDim.x) { (&fcol[0][0])[i] = 0.f; (&icol[0][0])[i] = 0; }
  __syncthreads();
  float* fc = fcol[cp & 1] + slot;
  int* ic = icol[cp & 1] + slot;
  uint32_t st = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u;
    const int c = (st >> 27);   // 0..31
    const int c0 = c > 26 ? 26 : c;
    if (MODE == 0) {
      float g[6];
#pragma unroll
      for (int m = 0; m < 6; ++m) g[m] = fc[(c0 + m) * 128];
#pragma unroll
      for (int m = 0; m < 6; ++m) fc[(c0 + m) * 128] = g[m] + 1.0f;
    } else if (MODE == 1) {
#pragma unroll
      for (int m = 0; m < 6; ++m) atomicAdd(ic + (c0 + m) * 128, (int)st >> (m + 8));
    } else {
#pragma unroll
      for (int m = 0; m < 6; ++m) atomicAdd(fc + (c0 + m) * 128, 1.0f + m);
    }
  }
  __syncthreads();
  float s = 0; int si = 0;
  for (int i = threadIdx.x; i < 2 * 32 * 128; i += blockDim.x) { s += (&fcol[0][0])[i]; si += (&icol[0][0])[i]; }
  if (s == 12345.f || si == 12345) out[0] = 1;
}
int main() {
  unsigned* o; cudaMalloc(&o, 4);
  int iters = 20000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148, 512>>>(iters, o); else if (mode == 1) k<1><<<148, 512>>>(iters, o); else k<2><<<148, 512>>>(iters, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double taps = 148.0 * 512 * iters * 6;
      printf("mode %d (%s): %.3f ms, %.3f SM-cycles per warp-tap at 1.965 GHz\n", mode, mode == 2 ? "atomicAdd f32" : mode ? "RED.add.u32" : "LDS+STS f32", ms,
             ms * 1e-3 * 1.965e9 / (taps / 32 / 148));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
