// Microbenchmark: write bandwidth of the projection's Z layout on B200 (Z [P][L] fp32 slice-major).
//  (a) epilogue pattern: CTA tile = 128 points x 256 slices, warp = 32 points x 128 slices, STG.32 per (slice)
//  (b) same tile, each lane writes 4 consecutive points of one slice (STG.128)
//  (c) contiguous memset-like stream (STG.128), same bytes
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void __launch_bounds__(256) k_tile32(float* Z, int64_t L, int P, int64_t ld) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = warp & 3, h = warp >> 2;
  const int64_t ntm = (L + 127) / 128;
  for (int64_t t = blockIdx.x; t < ntm; t += gridDim.x) {
    const int64_t i = t * 128 + 32 * q + lane;
    if (i >= L) continue;
    for (int s = h * 128; s < h * 128 + 128; ++s) Z[s * ld + i] = (float)s;
  }
}
__global__ void __launch_bounds__(256) k_tile128(float* Z, int64_t L, int P, int64_t ld) {
  // warp w: slices [32 w, 32 w + 32) of the tile; lane: 4 consecutive points (lane*4 .. +3) of 128
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntm = (L + 127) / 128;
  for (int64_t t = blockIdx.x; t < ntm; t += gridDim.x) {
    const int64_t i = t * 128 + 4 * lane;
    if (i + 3 >= L) continue;
    for (int s = warp * 32; s < warp * 32 + 32; ++s)
      *reinterpret_cast<float4*>(Z + s * ld + i) = make_float4(s, s, s, s);
  }
}
__global__ void k_stream(float4* Z, int64_t n4) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += (int64_t)gridDim.x * blockDim.x)
    Z[k] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
  const int64_t L = 200000;   // cfg2
  const int P = 256;
  const int64_t ld = L;
  float* Z;
  CK(cudaMalloc(&Z, sizeof(float) * L * P));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 4.0 * L * P;
  auto run = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 10;
    printf("%-50s %8.1f us  %7.2f TB/s\n", name, ms * 1e3, bytes / ms / 1e9);
    return 0;
  };
  run("tile 128x256, STG.32 per slice (epilogue)", [&] { k_tile32<<<148, 256>>>(Z, L, P, ld); });
  run("tile 128x256, STG.32 per slice, 296 CTAs", [&] { k_tile32<<<296, 256>>>(Z, L, P, ld); });
  run("tile 128x256, STG.128 (4 points / lane)", [&] { k_tile128<<<148, 256>>>(Z, L, P, ld); });
  run("tile 128x256, STG.128, 592 CTAs", [&] { k_tile128<<<592, 256>>>(Z, L, P, ld); });
  run("contiguous stream STG.128", [&] { k_stream<<<148 * 8, 256>>>(reinterpret_cast<float4*>(Z), L * P / 4); });
  CK(cudaGetLastError());
  return 0;
}
