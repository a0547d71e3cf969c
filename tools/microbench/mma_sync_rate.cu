// Microbenchmark: warp-level mma.sync throughput on B200 (legacy HMMA path)
// for TF32 m16n8k8 and BF16 m16n8k16, versus FFMA.  Question it answers:
// can the direct 45->13 controller (16-cell genome groups per tile, K=48,
// N=16) run as 3xTF32 mma.sync faster than the FP32 FMA chain?
// Prints MAC/clk/SM per variant for several warps-per-SM counts.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bench(float* out, int iters, long long* cyc) {
  float d[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) d[i][j] = 0.f;
  unsigned a[4], b[2];
  for (int j = 0; j < 4; ++j) a[j] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + j);
  for (int j = 0; j < 2; ++j) b[j] = __float_as_uint(0.5f + j);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (MODE == 1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          d[i][j] = fmaf(__uint_as_float(a[j]), __uint_as_float(b[j & 1]), d[i][j]);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += d[i][j];
  if (s == 12345.f) out[blockIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps, double mac_per_inst) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  const int iters = 4096;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  bench<MODE><<<sms, warps * 32>>>(out, 16, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE><<<sms, warps * 32>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double inst_per_warp = 8.0 * iters;
  const double mac_per_sm = inst_per_warp * warps * mac_per_inst;
  printf("%-10s warps/SM %2d: %8.1f MAC/clk/SM (clock64 %lld cyc), %.3f ms, %.1f TMAC/s\n", name, warps,
         mac_per_sm / (double)c, c, ms, mac_per_sm * sms / (ms * 1e-3) / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16, 32}) run<0>("tf32 1688", w, 16 * 8 * 8);
  for (int w : {4, 8, 16, 32}) run<1>("bf16 16816", w, 16 * 8 * 16);
  for (int w : {4, 8, 16, 32}) run<2>("ffma", w, 32 * 4);
  return 0;
}
