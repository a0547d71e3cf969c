// Validation of the tcgen05 kind::tf32 building blocks used by the hidden-
// layer controller: canonical K-major no-swizzle smem layout + descriptors,
// instruction descriptor, TMEM alloc / 32x32b loads, mbarrier commit, and
// 3xTF32 split accuracy (D = Ahi*Bhi + Ahi*Blo + Alo*Bhi) against float64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_tf32 tc_tf32.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128, K = 48;

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// canonical K-major, no swizzle: 16-byte core rows; chunk (kc, row/8) at
// (kc * (R/8) + row/8) * 128 B, row % 8 at 16 B stride.
__device__ __forceinline__ uint32_t canon_off(int row, int k, int R) {
  return ((k >> 2) * (R >> 3) + (row >> 3)) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__global__ void k(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* Ahi = reinterpret_cast<float*>(sm);
  float* Alo = Ahi + M * K;
  float* Bhi = Alo + M * K;
  float* Blo = Bhi + N * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    const float a = A[i], ah = tf32_rna(a), al = tf32_rna(a - ah);
    *reinterpret_cast<float*>(reinterpret_cast<char*>(Ahi) + canon_off(r, kk, M)) = ah;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(Alo) + canon_off(r, kk, M)) = mode ? al : 0.f;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    const float b = B[i], bh = tf32_rna(b), bl = tf32_rna(b - bh);
    *reinterpret_cast<float*>(reinterpret_cast<char*>(Bhi) + canon_off(r, kk, N)) = bh;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(Blo) + canon_off(r, kk, N)) = mode ? bl : 0.f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a_hi = (uint32_t)__cvta_generic_to_shared(Ahi), a_lo = (uint32_t)__cvta_generic_to_shared(Alo);
    const uint32_t b_hi = (uint32_t)__cvta_generic_to_shared(Bhi), b_lo = (uint32_t)__cvta_generic_to_shared(Blo);
    const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
    int acc = 0;
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t offA = 2 * ks * lboA, offB = 2 * ks * lboB;
      const uint64_t dAh = make_desc(a_hi + offA, lboA, 128), dAl = make_desc(a_lo + offA, lboA, 128);
      const uint64_t dBh = make_desc(b_hi + offB, lboB, 128), dBl = make_desc(b_lo + offB, lboB, 128);
      const uint64_t as[3] = {dAl, dAh, dAh}, bs[3] = {dBh, dBl, dBh};
      for (int t = 0; t < 3; ++t) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(as[t]), "l"(bs[t]), "r"(idesc), "r"(acc));
        acc = 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  // wait for the MMAs
  {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(b), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() / (double)RAND_MAX * 4 - 2);
  for (auto& x : B) x = (float)((rand() / (double)RAND_MAX * 2 - 1) * 0.6);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 4 * M * K * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    k<<<1, 128, smem>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0, worst_abs = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0, mag = 0;
        for (int kk = 0; kk < K; ++kk) {
          ref += (double)A[i * K + kk] * B[j * K + kk];
          mag += fabs((double)A[i * K + kk] * B[j * K + kk]);
        }
        const double err = fabs(D[i * N + j] - ref);
        worst = fmax(worst, err / mag);
        worst_abs = fmax(worst_abs, err);
      }
    printf("mode %s: max |err| / sum|a*b| = %.3e, max abs err %.3e  (D[0]=%f)\n", mode ? "3xTF32" : "1xTF32", worst,
           worst_abs, D[0]);
  }
  return 0;
}
