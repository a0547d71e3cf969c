// Issue-to-completion time of back-to-back tcgen05.mma kind::tf32 chains
// (M=128, K=8 per MMA, operands in shared memory, canonical K-major
// no-swizzle layout) for several N, accumulating into one or several TMEM
// accumulators; prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_rate tc_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n" : "=r"(pred));
  return pred;
}

__global__ void k(int n_mma, int N, int nacc, long long* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 * 48 + 256 * 48); i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base)));
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
  if (warp == 0) {  // warp-uniform issue path; one elected lane executes the MMA
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm), b = a + 128 * 48 * 4;
    const uint32_t lA = 128 * 16, lB = N * 16;
    const uint32_t leader = mode == 0 ? (tid == 0) : elect_one();
    (void)lA;
    (void)lB;
    const long long c0 = clock64();
    if (mode == 0) {
      if (leader) {
        for (int i = 0; i < n_mma; ++i) {
          const int ks = i % 6;
          const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
          const uint64_t da = make_desc(a + 2 * ks * lA, lA, 128), db = make_desc(b + 2 * ks * lB, lB, 128);
          const uint32_t acc = i >= nacc;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                       "l"(da), "l"(db), "r"(id), "r"(acc));
        }
      }
    } else if (mode == 3) {  // fully unrolled, constant offsets, 2 accumulators
      const uint64_t da0 = make_desc(a, lA, 128), db0 = make_desc(b, lB, 128);
#pragma unroll
      for (int i = 0; i < 18; ++i) {
        const int ks = i % 6;
        const uint32_t d = tmem + (uint32_t)((i & 1) * N);
        const uint64_t da = da0 + (uint64_t)((2 * ks * 128 * 16) >> 4), db = db0 + (uint64_t)((2 * ks * lB) >> 4);
        asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                     "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                     "l"(da), "l"(db), "r"(id), "r"(i >= 2 ? 1u : 0u), "r"(leader));
      }
    } else if (mode == 2) {  // K-major SWIZZLE_128B: 8-row x 128 B atoms (SBO 1024), +32 B per K=8 step
      const uint64_t sw = (uint64_t)2 << 61;
      const uint64_t da0 = make_desc(a, 16, 1024) | sw, db0 = make_desc(b, 16, 1024) | sw;
      for (int i = 0; i < n_mma; ++i) {
        const int ks = i % 4;
        const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
        const uint64_t da = da0 + (uint64_t)((ks * 32) >> 4), db = db0 + (uint64_t)((ks * 32) >> 4);
        const uint32_t acc = i >= nacc;
        asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                     "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                     "l"(da), "l"(db), "r"(id), "r"(acc), "r"(leader));
      }
    } else {
      const uint64_t da0 = make_desc(a, lA, 128), db0 = make_desc(b, lB, 128);
      for (int i = 0; i < n_mma; ++i) {
        const int ks = i % 6;
        const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
        const uint64_t da = da0 + (uint64_t)((2 * ks * lA) >> 4), db = db0 + (uint64_t)((2 * ks * lB) >> 4);
        const uint32_t acc = i >= nacc;
        asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
                     "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                     "l"(da), "l"(db), "r"(id), "r"(acc), "r"(leader));
      }
    }
    const long long c1 = clock64();
    if (leader) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&bar)));
    }
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
    const long long c2 = clock64();
    if (tid == 0) {
      out[0] = c1 - c0;
      out[1] = c2 - c0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const int smem = (128 * 48 + 256 * 48) * 4 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int Ns[] = {16, 32, 64, 128, 256};
  for (int mode = 0; mode < 4; ++mode)
    for (int N : Ns)
      for (int n : {18, 180}) {
        if (mode == 3 && n != 18) continue;
        k<<<1, 128, smem>>>(n, N, 2, d, mode);
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s N=%3d mmas=%3d: issue %6lld cyc, complete %6lld cyc, %.1f cyc/MMA, %.0f MAC/clk\n",
               mode == 3 ? "unrolled  " : mode == 2 ? "sw128     " : (mode ? "warp+elect" : "tid==0   "), N, n, h[0], h[1], (double)h[1] / n, (double)n * 128 * N * 8 / h[1]);
      }
  return 0;
}
