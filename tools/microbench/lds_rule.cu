// Shared-memory wavefronts per LDS.64 / LDS.128 as a function of how many
// distinct (conflict-free) addresses each quarter-/half-warp touches.
// Read under ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int group_of(int pat, int lane) {
  switch (pat) {
    case 0: return 0;                  // uniform
    case 1: return lane / 16;          // one address per half-warp
    case 2: return lane / 8;           // one per quarter
    case 3: return lane / 4;           // two per quarter
    case 4: return (lane / 8) * 2 + (lane & 1);  // two per quarter, interleaved
    case 5: return lane / 2;           // four per quarter
    case 6: return lane;               // eight per quarter (all distinct)
    case 7: return (lane + 4) / 8;     // quarters straddle groups (2 per quarter)
    default: return 0;
  }
}

template <int VEC>
__global__ void k(float* out, int iters, int pat, int stride, int off = 0) {
  extern __shared__ __align__(16) float s[];
  const int lane = threadIdx.x & 31;
  const int grp = group_of(pat, lane);
  // group g at word offset g*36 (+4 banks per group: conflict-free for <= 8 groups of float4)
  const unsigned base = (unsigned)__cvta_generic_to_shared(s) + off * 4 + grp * stride * 4;
  float acc = 0.f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const unsigned a = base + ((it * 64) & 4095) * 4;
    if (VEC == 4) {
      float x, y, z, w;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
      acc += x + y + z + w;
    } else {
      float x, y;
      asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
      acc += x + y;
    }
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int strides[] = {36, 68, 132, 260, 516, 540, 1028, 2052, 4100, 548, 556, 572, 604};
  const int offs[] = {0, 4, 8, 12, 16, 20, 24, 28, 15680, 15684, 15688, 15692, 20000, 30000, 40000};
  for (int o : offs) k<2><<<1, 32, smem>>>(out, 100, 7, 540, o);
  for (int o : offs) k<4><<<1, 32, smem>>>(out, 100, 7, 540, o);
  for (int o : offs) k<2><<<1, 32, smem>>>(out, 100, 3, 540, o);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
