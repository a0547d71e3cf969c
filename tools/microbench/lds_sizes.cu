// Wavefronts of one LDS.64 per iteration when consecutive lane groups of the
// given sizes read different genome rows (stride 2160 B): which group
// layouts a warp can be served in one wavefront (read under ncu).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int VEC>
__global__ void k(float* out, const int* slot_of_lane) {
  extern __shared__ __align__(16) float s[];
  const int lane = threadIdx.x & 31;
  const unsigned a = (unsigned)__cvta_generic_to_shared(s) + slot_of_lane[lane] * 2160;
  float acc = 0.f;
#pragma unroll 1
  for (int it = 0; it < 100; ++it) {
    if (VEC == 2) {
      float x, y;
      asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
      acc += x * y;
    } else {
      float x, y, z, w;
      asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
      acc += x * y + z * w;
    }
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  int* d;
  cudaMalloc(&out, 4);
  cudaMalloc(&d, 32 * 4);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<std::vector<int>> pats = {
      {32}, {16, 16}, {8, 8, 8, 8}, {4, 8, 8, 8, 4}, {11, 5, 8, 8}, {9, 7, 8, 8}, {12, 4, 8, 8},
      {8, 24}, {11, 21}, {3, 13, 16}, {2, 8, 9, 8, 5}, {7, 7, 7, 7, 4}, {1, 31}, {31, 1}, {15, 17},
      {17, 15}, {4, 4, 4, 4, 4, 4, 4, 4}, {6, 10, 16}, {10, 6, 16}, {16, 10, 6}, {16, 6, 10}};
  for (auto& p : pats) {
    int h[32], lane = 0;
    for (size_t g = 0; g < p.size(); ++g)
      for (int i = 0; i < p[g]; ++i) h[lane++] = (int)g;
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    k<2><<<1, 32, 64 * 1024>>>(out, d);
    k<4><<<1, 32, 64 * 1024>>>(out, d);
    cudaDeviceSynchronize();
    printf("pattern");
    for (int v : p) printf(" %d", v);
    printf("\n");
  }
  return 0;
}
