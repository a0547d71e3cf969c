// Does a concurrent cudaMemcpy2DAsync (host<->device, 6 rows with a plane
// pitch, the evo_step_host band copy) slow kernels more than a 1-D copy of
// the same bytes?  A short HBM-streaming kernel is timed back to back alone
// and under each kind of concurrent copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copy2d_interference copy2d_interference.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void stream_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = a[i];
    v.x += 1.f;
    b[i] = v;
  }
}

int main() {
  const size_t plane = 4u << 20, rows = 6;  // 6 planes of 4 MB, copy the first 3.3 MB of each
  const size_t w = 3400000;
  unsigned char *h, *d;
  h = (unsigned char*)aligned_alloc(4096, plane * rows * 4);
  memset(h, 1, plane * rows * 4);
  cudaHostRegister(h, plane * rows * 4, cudaHostRegisterMapped | cudaHostRegisterPortable);
  cudaMalloc(&d, plane * rows * 4);
  const size_t nk = 8u << 20;  // 8M float4 = 128 MB each way
  float4 *ka, *kb;
  cudaMalloc(&ka, nk * 16);
  cudaMalloc(&kb, nk * 16);
  cudaStream_t ks, cs;
  cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  const char* names[] = {"alone", "1D d2h", "2D d2h", "1D h2d", "2D h2d"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaDeviceSynchronize();
      for (int k = 0; k < 8 && mode; ++k) {  // enough copy work to cover the kernel loop
        if (mode == 1) cudaMemcpyAsync(h, d, w * rows, cudaMemcpyDeviceToHost, cs);
        if (mode == 2) cudaMemcpy2DAsync(h, plane, d, plane, w, rows, cudaMemcpyDeviceToHost, cs);
        if (mode == 3) cudaMemcpyAsync(d, h, w * rows, cudaMemcpyHostToDevice, cs);
        if (mode == 4) cudaMemcpy2DAsync(d, plane, h, plane, w, rows, cudaMemcpyHostToDevice, cs);
      }
      cudaEventRecord(a, ks);
      for (int k = 0; k < 20; ++k) stream_kernel<<<148 * 4, 512, 0, ks>>>(ka, kb, nk);
      cudaEventRecord(z, ks);
      cudaEventSynchronize(z);
      float ms;
      cudaEventElapsedTime(&ms, a, z);
      if (ms < best) best = ms;
    }
    printf("%-7s kernel %.1f us\n", names[mode], best / 20 * 1e3);
  }
  return 0;
}
