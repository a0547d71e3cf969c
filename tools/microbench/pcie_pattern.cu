// Host<->device copy patterns of the host-pipelined step (evo_step_host):
// one big copy vs B bands x 5 plane copies (4+4+12+4+1 bytes per cell), per
// direction and both directions at once, cudaHostAlloc vs malloc +
// cudaHostRegister host memory, with and without a small kernel after each
// band on the copy stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_pattern pcie_pattern.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void touch(int* p) {
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

static const size_t kCells = 1 << 20;
#ifndef NSEG
#define NSEG 5
#endif
#if NSEG == 5
static const int kBytes[5] = {4, 4, 12, 4, 1};
#elif NSEG == 3
static const int kBytes[3] = {20, 4, 1};
#else
static const int kBytes[1] = {25};
#endif

struct Buf {
  unsigned char* h[NSEG];
  unsigned char* d[NSEG];
};

static void alloc(Buf& b, bool reg) {
  for (int i = 0; i < NSEG; ++i) {
    const size_t n = kCells * kBytes[i];
    if (reg) {
      b.h[i] = (unsigned char*)aligned_alloc(4096, n);
      memset(b.h[i], 1, n);
      cudaHostRegister(b.h[i], n, cudaHostRegisterDefault);
    } else {
      cudaHostAlloc((void**)&b.h[i], n, cudaHostAllocDefault);
      memset(b.h[i], 1, n);
    }
    cudaMalloc(&b.d[i], n);
  }
}

static void issue(const Buf& b, int bands, bool h2d, cudaStream_t s, bool kern, int* flag) {
  for (int k = 0; k < bands; ++k) {
    const size_t c0 = kCells * k / bands, c1 = kCells * (k + 1) / bands;
    for (int i = 0; i < NSEG; ++i) {
      const size_t o = c0 * kBytes[i], n = (c1 - c0) * kBytes[i];
      if (h2d)
        cudaMemcpyAsync(b.d[i] + o, b.h[i] + o, n, cudaMemcpyHostToDevice, s);
      else
        cudaMemcpyAsync(b.h[i] + o, b.d[i] + o, n, cudaMemcpyDeviceToHost, s);
    }
    if (kern) touch<<<1, 32, 0, s>>>(flag);
  }
}

int main() {
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  int* flag;
  cudaMalloc(&flag, 4);
  for (int reg = 1; reg < 2; ++reg) {
    Buf in, out;
    alloc(in, reg);
    alloc(out, reg);
    for (int bands : {1, 2, 3, 4, 6, 8})
      for (int kern = 0; kern < 1; ++kern)
        for (int mode = 0; mode < 3; ++mode) {  // 0 h2d, 1 d2h, 2 both
          float best = 1e9;
          for (int rep = 0; rep < 6; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, s1);
            cudaStreamWaitEvent(s2, a, 0);
            if (mode != 1) issue(in, bands, true, s1, kern, flag);
            if (mode != 0) issue(out, bands, false, s2, kern, flag);
            cudaEvent_t e2;
            cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
            cudaEventRecord(e2, s2);
            cudaStreamWaitEvent(s1, e2, 0);
            cudaEventRecord(z, s1);
            cudaEventSynchronize(z);
            cudaEventDestroy(e2);
            float ms;
            cudaEventElapsedTime(&ms, a, z);
            if (rep > 0 && ms < best) best = ms;
          }
          const double mb = kCells * 25 / 1e6;
          printf("%s bands=%2d kern=%d %-4s %.3f ms  %.1f GB/s per direction\n", reg ? "registered" : "hostalloc ",
                 bands, kern, mode == 0 ? "h2d" : (mode == 1 ? "d2h" : "both"), best, mb / best);
        }
  }
  return 0;
}
