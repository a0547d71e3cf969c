// Issue cost of tcgen05.mma kind::tf32 (M=128, K=8, N=16..64) by how the
// operands reach the instruction:
//   0 "waterfall":  descriptors built per MMA in ordinary registers inside
//                   `if (tid == 0)` - ptxas wraps every UTCHMMA in an
//                   ELECT / BRA.U.ANY loop over the distinct operand values;
//   1 "uniform":    whole warp 0 runs the loop (warp-uniform control flow),
//                   descriptors derived from uniform values only (shared
//                   window base, loop counter, constant TMEM column), the
//                   MMA predicated on elect.sync inside the same asm block;
//   2 "uniform+ur": as 1, descriptors advanced by adding constants to one
//                   64-bit base (no per-MMA shifts/masks).
// Prints cycles per MMA for a chain of 96 MMAs into 2 accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_issue tc_issue.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

template <int MODE, int N>
__global__ void k(int n_mma, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 * 48 + 256 * 48); i += blockDim.x) reinterpret_cast<float*>(sm_raw)[i] = 0.001f * (i & 7);
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
  constexpr uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  constexpr uint32_t lA = 128 * 16, lB = N * 16;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm_raw), b = a + 128 * 48 * 4;
  long long c0 = 0, c1 = 0;
  if (MODE == 0) {
    const uint32_t tmem = tmem_base;
    c0 = clock64();
    if (tid == 0) {
      for (int i = 0; i < n_mma; ++i) {
        const int ks = i % 6;
        const uint32_t d = tmem + (uint32_t)((i & 1) * N);
        const uint64_t da = make_desc(a + 2 * ks * lA, lA, 128), db = make_desc(b + 2 * ks * lB, lB, 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                     "l"(da), "l"(db), "n"(id), "r"((uint32_t)(i >= 2)));
      }
    }
    c1 = clock64();
  } else if (warp == 0) {
    c0 = clock64();
    const uint64_t da0 = make_desc(a, lA, 128), db0 = make_desc(b, lB, 128);
#pragma unroll 1
    for (int i0 = 0; i0 < n_mma; i0 += 12) {
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const int ks = j % 6;
        uint64_t da, db;
        if (MODE == 1) {
          da = make_desc(a + 2 * ks * lA, lA, 128);
          db = make_desc(b + 2 * ks * lB, lB, 128);
        } else {
          da = da0 + (uint64_t)((2 * ks * lA) >> 4);
          db = db0 + (uint64_t)((2 * ks * lB) >> 4);
        }
        const uint32_t acc = (i0 + j) >= 2;
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %3, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}\n" ::"r"((uint32_t)((j & 1) * N)),
            "l"(da), "l"(db), "r"(acc), "n"(id));
      }
    }
    c1 = clock64();
  }
  if (warp == 0) {
    if (tid == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&bar)));
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

template <int MODE, int N>
void run(long long* d) {
  const int smem = (128 * 48 + 256 * 48) * 4;
  cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int n : {12, 96, 960}) {
    k<MODE, N><<<1, 128, smem>>>(n, d);
    long long h[2] = {0, 0};
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d N=%3d mmas=%4d: issue %7lld cyc, complete %7lld cyc, %6.1f cyc/MMA (floor %d) %s\n", MODE, N, n,
           h[0], h[1], (double)h[1] / n, 128 * N / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  // mode 1/2 use a TMEM column offset from column 0 (the only CTA on the SM)
  run<0, 16>(d);
  run<1, 16>(d);
  run<2, 16>(d);
  run<0, 32>(d);
  run<2, 32>(d);
  run<0, 64>(d);
  run<2, 64>(d);
  run<2, 128>(d);
  return 0;
}
