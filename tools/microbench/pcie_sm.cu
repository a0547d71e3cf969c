// SM-driven host<->device copies over PCIe (mapped page-locked host memory):
// a grid of G CTAs streams int4 loads from host memory into device memory
// (pull) or device memory into host memory (push); bandwidth per direction
// alone and both at once, for several G.  Compare with DMA in pcie_pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_sm pcie_sm.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void copy16(int4* __restrict__ dst, const int4* __restrict__ src, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  const size_t bytes = 26u << 20;
  const size_t n = bytes / 16;
  void *h_in = aligned_alloc(4096, bytes), *h_out = aligned_alloc(4096, bytes);
  memset(h_in, 1, bytes);
  memset(h_out, 1, bytes);
  cudaHostRegister(h_in, bytes, cudaHostRegisterMapped);
  cudaHostRegister(h_out, bytes, cudaHostRegisterMapped);
  void *dh_in, *dh_out;
  cudaHostGetDevicePointer(&dh_in, h_in, 0);
  cudaHostGetDevicePointer(&dh_out, h_out, 0);
  printf("mapped pointers equal host pointers: %d %d\n", dh_in == h_in, dh_out == h_out);
  void *d_in, *d_out;
  cudaMalloc(&d_in, bytes);
  cudaMalloc(&d_out, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, z, e2;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
  for (int threads : {512})
    for (int G : {16, 32, 64})
      for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
          cudaDeviceSynchronize();
          cudaEventRecord(a, s1);
          cudaStreamWaitEvent(s2, a, 0);
          if (mode != 1) copy16<<<G, threads, 0, s1>>>((int4*)d_in, (const int4*)dh_in, n);
          if (mode != 0) copy16<<<G, threads, 0, s2>>>((int4*)dh_out, (const int4*)d_out, n);
          cudaEventRecord(e2, s2);
          cudaStreamWaitEvent(s1, e2, 0);
          cudaEventRecord(z, s1);
          cudaEventSynchronize(z);
          float ms;
          cudaEventElapsedTime(&ms, a, z);
          if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("threads=%4d G=%3d %-4s %.3f ms  %.1f GB/s per direction %s\n", threads, G,
               mode == 0 ? "pull" : (mode == 1 ? "push" : "both"), best, bytes / 1e6 / best,
               e ? cudaGetErrorString(e) : "");
      }
  // mixed: SM pull + DMA D2H (in `chunks` pieces), DMA H2D + SM push
  for (int chunks : {1, 4, 8, 20})
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 6; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, s1);
        cudaStreamWaitEvent(s2, a, 0);
        const size_t cb = bytes / chunks;
        if (mode == 0) {
          copy16<<<32, 512, 0, s1>>>((int4*)d_in, (const int4*)dh_in, n);
          for (int k = 0; k < chunks; ++k)
            cudaMemcpyAsync((char*)h_out + k * cb, (char*)d_out + k * cb, cb, cudaMemcpyDeviceToHost, s2);
        } else {
          for (int k = 0; k < chunks; ++k)
            cudaMemcpyAsync((char*)d_in + k * cb, (char*)h_in + k * cb, cb, cudaMemcpyHostToDevice, s1);
          copy16<<<32, 512, 0, s2>>>((int4*)dh_out, (const int4*)d_out, n);
        }
        cudaEventRecord(e2, s2);
        cudaStreamWaitEvent(s1, e2, 0);
        cudaEventRecord(z, s1);
        cudaEventSynchronize(z);
        float ms;
        cudaEventElapsedTime(&ms, a, z);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("mixed %s chunks=%2d both %.3f ms  %.1f GB/s per direction\n",
             mode == 0 ? "SM-pull + DMA-d2h" : "DMA-h2d + SM-push", chunks, best, bytes / 1e6 / best);
    }
  return 0;
}
