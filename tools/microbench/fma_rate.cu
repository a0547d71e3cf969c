// Microbenchmark: FP32 FMA issue/throughput on B200 for FFMA vs packed FFMA2
// (fma.rn.f32x2), the engine choice for the direct 45->13 controller
// (SURVEY.md §7 hard part #1).  Prints FMA/clk/SM for each variant.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int MODE>
__global__ void bench(float* out, const float* w, int iters) {
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = out[threadIdx.x & 31];
  unsigned long long a2[8];
  for (int i = 0; i < 8; ++i) a2[i] = pk(acc[2 * i], acc[2 * i + 1]);
  const unsigned long long xx = pk(x, x + 1.0f);
  for (int it = 0; it < iters; ++it) {
    const float wv = w[it & 63];
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(x, wv, acc[i]);
    } else if (MODE == 1) {
      const unsigned long long ww = pk(wv, wv);
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = ffma2(xx, ww, a2[i]);
    } else {
      const unsigned long long ww = *reinterpret_cast<const unsigned long long*>(w + ((2 * it) & 63));
#pragma unroll
      for (int i = 0; i < 8; ++i) a2[i] = ffma2(xx, ww, a2[i]);
    }
  }
  float s = 0.f;
  if (MODE == 0)
    for (int i = 0; i < 16; ++i) s += acc[i];
  else
    for (int i = 0; i < 8; ++i) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a2[i]));
      s += lo + hi;
    }
  if (s == 12345.f) out[blockIdx.x] = s;
}

int main() {
  float *out, *w;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&w, 1024);
  cudaMemset(out, 0, 1 << 20);
  cudaMemset(w, 0, 1024);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 1 << 14;
  for (int threads : {256, 512, 1024}) {
    for (int mode = 0; mode < 3; ++mode) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int blocks = sms * (2048 / threads);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) bench<0><<<blocks, threads>>>(out, w, iters);
        if (mode == 1) bench<1><<<blocks, threads>>>(out, w, iters);
        if (mode == 2) bench<2><<<blocks, threads>>>(out, w, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double fmas = (double)blocks * threads * iters * 16;
      const double per_s = fmas / (ms * 1e-3);
      printf("threads %4d mode %d (%s): %.1f TFMA/s = %.1f FMA/clk/SM at %d MHz max clock\n", threads, mode,
             mode == 0 ? "FFMA" : (mode == 1 ? "FFMA2 bcast-mov" : "FFMA2 pair-load"), per_s / 1e12,
             per_s / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
