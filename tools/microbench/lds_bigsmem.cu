// Wavefronts of a warp-uniform LDS.128 broadcast as a function of the
// shared-memory address and carveout (read under ncu).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(float* out, int iters, int off_floats) {
  extern __shared__ __align__(16) float s[];
  const unsigned base = (unsigned)__cvta_generic_to_shared(s) + off_floats * 4;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const unsigned a = base + ((it * 16) & 1023);
    float x, y, z, w;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
    acc += x + y + z + w;
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  const int smem = 210 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int off : {0, 16 * 1024, 40 * 1024, 50 * 1024}) {  // floats: 0, 64 KB, 160 KB, 200 KB
    k<<<1, 640, smem>>>(out, 64, off);
    k<<<1, 32, smem>>>(out, 64, off);
  }
  k<<<1, 32, 1024>>>(out, 64, 0);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
