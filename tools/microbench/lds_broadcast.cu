// Microbenchmark: shared-memory cost of LDS.128 / LDS.32 when a warp reads D
// distinct addresses (broadcast groups of 32/D lanes), the distinct addresses
// either in distinct 16-byte bank groups (stride 36 floats) or the same one
// (stride 32).  Decides how per-genome weight tables of pass 1 are shared.
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC>
__global__ void bench(float* out, int iters, int distinct, int stride_f) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 1e-3f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int grp = lane % distinct;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(s);
  float acc = 0.f;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    const unsigned off = ((grp * stride_f + (it * 44) % 4000) & ~3u) * 4u;
    if (VEC == 4) {
      float a, b, c, d;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "r"(sbase + off));
      acc += a + b + c + d;
    } else {
      float a;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(a) : "r"(sbase + off));
      acc += a;
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1 << 14;
  for (int vec : {4, 1}) {
    for (int distinct : {1, 2, 4, 8, 32}) {
      for (int stride : {36, 32}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a);
          if (vec == 4) bench<4><<<sms * 4, 256>>>(out, iters, distinct, stride);
          else bench<1><<<sms * 4, 256>>>(out, iters, distinct, stride);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double warp_ops = (double)sms * 4 * 8 * iters;
        printf("LDS.%-3d distinct %2d stride %2d: %.3f cycles per warp-LDS per SM (at 1.9 GHz)\n", vec * 32,
               distinct, stride, ms * 1e-3 * 1.9e9 / (warp_ops / sms));
      }
    }
  }
  return 0;
}
