#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstring>
__device__ __forceinline__ unsigned f2key_tc(float f) { const unsigned u = __float_as_uint(f); return (u & 0x80000000u) ? ~u : (u | 0x80000000u); }
#include "colrange_snip.h"
__global__ void k(const float* in, unsigned* out) {
  const int lane = threadIdx.x;
  const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1, b1 = (lane >> 1) & 1;
  uint32_t kmn[16], kmx[16];
  for (int j = 0; j < 16; ++j) { const float z = in[lane * 16 + j] * 1.0f; const uint32_t key = f2key_tc(z); kmn[j] = key; kmx[j] = key; }
  uint32_t amn, amx;
  colrange16(kmn, kmx, b4, b3, b2, b1, &amn, &amx);
  out[lane * 2] = amn; out[lane * 2 + 1] = amx;
}
int main() {
  float h[512]; for (int i = 0; i < 512; ++i) h[i] = sinf(i * 0.37f) * 3;
  for (int j = 0; j < 16; ++j) { unsigned u = 0x7fffffffu; memcpy(&h[5 * 16 + j], &u, 4); }
  float* d; unsigned* o; cudaMalloc(&d, 2048); cudaMalloc(&o, 256);
  cudaMemcpy(d, h, 2048, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(d, o);
  unsigned r[64]; cudaMemcpy(r, o, 256, cudaMemcpyDeviceToHost);
  for (int l = 0; l < 32; l += 2) printf("lane %d mn %08x mx %08x\n", l, r[2 * l], r[2 * l + 1]);
}
