// Wavefronts per LDS.128 when lanes read per-group float4 rows (stride 540
// floats between groups), group sizes 8 lanes, in various block shapes.
// Read under ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  extern __shared__ __align__(16) float s[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int grp;
  if (MODE == 0) grp = warp * 4 + lane / 8;          // 4 groups of 8, consecutive
  else if (MODE == 1) grp = (warp * 32 + lane) / 7;  // groups of 7 spanning warps
  else if (MODE == 2) grp = lane / 8;                // same in every warp
  else grp = 0;
  grp %= 64;
  const unsigned base = (unsigned)__cvta_generic_to_shared(s) + 4096 * 4 + grp * 540 * 4;
  float acc = 0.f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int sidx = it % 9, ch = (it / 9) % 5, j = (it / 45) % 3;
    const unsigned a = base + (sidx * 60 + ch * 12 + j * 4) * 4;
    float x, y, z, w;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
    acc += x + y + z + w;
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<0><<<1, 32, smem>>>(out, 135);
  k<0><<<1, 576, smem>>>(out, 135);
  k<1><<<1, 576, smem>>>(out, 135);
  k<2><<<1, 576, smem>>>(out, 135);
  k<3><<<1, 576, smem>>>(out, 135);
  k<0><<<148, 576, smem>>>(out, 135);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
