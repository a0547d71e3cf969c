// Replays the weight-load address pattern of k_pass1_direct's first warp
// (slots per lane as bucketed in tile 0, W12 base 63680 B, genome stride
// 2160 B) with LDS.64 / LDS.128 and counts wavefronts (read under ncu).
#include <cstdio>
#include <cuda_runtime.h>

__constant__ int c_slot[32] = {0,0,0,0,0,0,0,0,0,0,0,1,1,1,1,1,2,2,2,2,2,2,2,2,3,3,3,3,3,3,3,3};

template <int VEC, bool VOL>
__global__ void k(float* out, unsigned base_b) {
  extern __shared__ __align__(16) float s[];
  for (int i = threadIdx.x; i < 50000; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(s) + base_b + c_slot[lane] * 2160;
  float acc = 0.f;
#pragma unroll
  for (int st = 0; st < 9; ++st)
#pragma unroll
    for (int ch = 0; ch < 5; ++ch)
#pragma unroll
      for (int p = 0; p < 12 / VEC; ++p) {
        const unsigned a = base + (st * 60 + ch * 12 + p * VEC) * 4;
        if (VEC == 2) {
          float x, y;
          if (VOL) asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
          else asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
          acc += x * y;
        } else {
          float x, y, z, w;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
          acc += x * y + z * w;
        }
      }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<2, true><<<1, 32, smem>>>(out, 63680);
  k<2, false><<<1, 32, smem>>>(out, 63680);
  k<4, false><<<1, 32, smem>>>(out, 63680);
  k<2, true><<<1, 32, smem>>>(out, 0);
  k<4, false><<<1, 32, smem>>>(out, 0);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
