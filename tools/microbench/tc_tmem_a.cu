// tcgen05.mma kind::tf32 with the A operand in TMEM (written by tcgen05.st,
// thread = lane = row, one 32-bit column per K element) and B in shared
// memory; checks the layout against float64 (M=128, N=16, K=64, 3xTF32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_tmem_a tc_tmem_a.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, K = 64;

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t canon_off(int row, int k, int R) {
  return ((k >> 2) * (R >> 3) + (row >> 3)) * 128 + (row & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__global__ void k(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) unsigned char Bs[2][N * K * 4];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, kk = i % K;
    const float b = B[i], bh = tf32_rna(b), bl = tf32_rna(b - bh);
    *reinterpret_cast<float*>(Bs[0] + canon_off(r, kk, N)) = bh;
    *reinterpret_cast<float*>(Bs[1] + canon_off(r, kk, N)) = bl;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // A hi at columns [64, 128), A lo at [128, 192); D at [0, 16)
  const int row = warp * 32 + lane;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < K; c += 8) {
    uint32_t h[8], l[8];
    for (int j = 0; j < 8; ++j) {
      const float a = A[row * K + c + j], ah = tf32_rna(a), al = tf32_rna(a - ah);
      h[j] = __float_as_uint(ah);
      l[j] = __float_as_uint(al);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_addr + 64 + c),
                 "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_addr + 128 + c),
                 "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t lB = (N / 8) * 128;
    const uint32_t bh = (uint32_t)__cvta_generic_to_shared(Bs[0]), bl = (uint32_t)__cvta_generic_to_shared(Bs[1]);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t ah = tmem + 64 + ks * 8, al = tmem + 128 + ks * 8;
      const uint64_t dbh = make_desc(bh + 2 * ks * lB, lB, 128), dbl = make_desc(bl + 2 * ks * lB, lB, 128);
      const uint32_t ta[3] = {al, ah, ah};
      const uint64_t tb[3] = {dbh, dbl, dbh};
      for (int t = 0; t < 3; ++t) {
        const uint32_t acc = (ks > 0 || t > 0);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "r"(ta[t]), "l"(tb[t]), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(lane_addr + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(5);
  for (auto& x : A) x = (float)tanh(rand() / (double)RAND_MAX * 6 - 3);
  for (auto& x : B) x = (float)((rand() / (double)RAND_MAX * 2 - 1) * 0.6);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0, wabs = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double ref = 0, mag = 0;
      for (int kk = 0; kk < K; ++kk) {
        ref += (double)A[i * K + kk] * B[j * K + kk];
        mag += fabs((double)A[i * K + kk] * B[j * K + kk]);
      }
      worst = fmax(worst, fabs(D[i * N + j] - ref) / mag);
      wabs = fmax(wabs, fabs(D[i * N + j] - ref));
    }
  printf("A in TMEM: max|err|/sum|ab| %.3e  max abs %.3e  D[0]=%f\n", worst, wabs, D[0]);
  return 0;
}
