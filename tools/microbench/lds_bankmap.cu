// Wavefronts of one LDS.64 per iteration for the bucketed lane->slot pattern
// {11,5,8,8} (genome stride 2160 B) as a function of the uniform word offset,
// to map shared-memory bank behaviour (read under ncu).
#include <cstdio>
#include <cuda_runtime.h>

__constant__ int c_slot[32] = {0,0,0,0,0,0,0,0,0,0,0,1,1,1,1,1,2,2,2,2,2,2,2,2,3,3,3,3,3,3,3,3};

__global__ void k(float* out, int off_words, int stride_b) {
  extern __shared__ __align__(16) float s[];
  const int lane = threadIdx.x & 31;
  const unsigned a = (unsigned)__cvta_generic_to_shared(s) + off_words * 4 + c_slot[lane] * stride_b;
  float acc = 0.f;
#pragma unroll 1
  for (int it = 0; it < 100; ++it) {
    float x, y;
    asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
    acc += x * y;
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int o = 0; o < 64; o += 2) k<<<1, 32, smem>>>(out, o, 2160);
  for (int o = 0; o < 64; o += 2) k<<<1, 32, smem>>>(out, o, 2176);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
