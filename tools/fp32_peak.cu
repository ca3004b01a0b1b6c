// FP32 FMA throughput of one B200 (the "alu" roofline peak of bench.py): every SM runs 8 independent FMA chains
// per thread in three forms -- scalar FFMA with register operands (3-reg form), packed FFMA2 (fp32x2), and FFMA
// with an immediate operand -- and reports TFLOP/s (2 flop per FMA lane).  JSON on stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu && tools/fp32_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int FORM>
__global__ void __launch_bounds__(512) k_fma(int iters, float a, float b, float* out) {
  if (FORM == 0) {   // per-thread operands: the 3-vector-register form (not a uniform-register operand)
    a += threadIdx.x * 1e-12f;
    b += threadIdx.x * 1e-12f;
  }
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-7f + j;
  if (FORM == 1) {
    float2 y[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = make_float2(x[j], x[j] + 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = __ffma2_rn(y[j], a2, b2);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = y[j].x + y[j].y;
  } else {
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = FORM == 0 ? fmaf(x[j], a, b) : fmaf(x[j], 0.999999f, 1e-7f);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 16, blocks = sms * 4, threads = 512;
  const char* names[3] = {"ffma_reg", "ffma2", "ffma_imm"};
  printf("{\"sms\": %d, \"max_clock_mhz\": %d", sms, clk / 1000);
  for (int f = 0; f < 3; ++f) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (f == 0) k_fma<0><<<blocks, threads>>>(iters, 0.999999f, 1e-7f, out);
      if (f == 1) k_fma<1><<<blocks, threads>>>(iters, 0.999999f, 1e-7f, out);
      if (f == 2) k_fma<2><<<blocks, threads>>>(iters, 0.999999f, 1e-7f, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double lanes = static_cast<double>(blocks) * threads * 8 * iters * (f == 1 ? 2 : 1);
    printf(", \"%s_tflops\": %.2f", names[f], 2.0 * lanes / (best * 1e-3) / 1e12);
  }
  printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
