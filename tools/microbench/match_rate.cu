// Microbenchmark: cost of warp-aggregated shared-memory ranking with
// __match_any_sync vs a plain shared-memory atomicAdd (census / bucketing).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void bench(int* out, int iters, int nbins) {
  __shared__ int bins[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    const int key = (s >> 16) % nbins;
    if (MODE == 0) {
      const unsigned mask = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(mask) - 1;
      int base = 0;
      if ((threadIdx.x & 31) == leader) base = atomicAdd(&bins[key], __popc(mask));
      base = __shfl_sync(0xffffffffu, base, leader);
      acc += base + __popc(mask & ((1u << (threadIdx.x & 31)) - 1u));
    } else {
      acc += atomicAdd(&bins[key], 1);
    }
  }
  if (acc == 123456789) out[0] = acc;
}

int main() {
  int* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nbins : {64, 8, 1}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) bench<0><<<sms * 4, 256>>>(out, iters, nbins);
        else bench<1><<<sms * 4, 256>>>(out, iters, nbins);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * 4 * 256 * iters;
      printf("bins %3d %-22s %.2f ns/op-per-SM (%.1f Gop/s)\n", nbins, mode == 0 ? "match_any aggregated" : "plain atomicAdd",
             ms * 1e6 / (ops / sms), ops / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
