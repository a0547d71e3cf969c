// Shared-memory wavefronts per LDS.128 / LDS.32 for broadcast patterns
// (read under ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum /
// executed LDS).  pattern: 0 all lanes one address; 1 one address per
// quarter-warp; 2 two addresses by half-warp; 3 two addresses interleaved
// (even/odd lanes); 4 four addresses interleaved (lane % 4); 5 32 distinct.
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC, int PAT, int STRIDE = 36>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float s[11000];
  for (int i = threadIdx.x; i < 11000; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int grp;
  switch (PAT) {
    case 0: grp = 0; break;
    case 1: grp = lane / 8; break;
    case 2: grp = lane / 16; break;
    case 3: grp = lane & 1; break;
    case 4: grp = lane & 3; break;
    case 6: grp = lane / 7; break;  // 5 groups of 7,7,7,7,4 lanes
    case 7: grp = ((blockIdx.x * blockDim.x + threadIdx.x) * 2) / 17; break;  // pairs of a sorted tile, 8.5 pairs/genome
    case 8: grp = ((threadIdx.x) * 2) / 17 + (threadIdx.x & 32 ? 1 : 0); break;
    default: grp = lane; break;
  }
  if (PAT >= 7) grp = grp % 18;
  const unsigned base = (unsigned)__cvta_generic_to_shared(s) + grp * STRIDE * 4;  // distinct bank groups
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const unsigned a = base + ((it * 48) % 2040) * 4;
    if (VEC == 4) {
      float x, y, z, w;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
      acc += x + y + z + w;
    } else {
      float x;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
      acc += x;
    }
  }
  if (acc == -1.f) out[0] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  k<4, 0><<<1, 32>>>(out, 64);
  k<4, 1><<<1, 32>>>(out, 64);
  k<4, 2><<<1, 32>>>(out, 64);
  k<4, 3><<<1, 32>>>(out, 64);
  k<4, 4><<<1, 32>>>(out, 64);
  k<4, 5><<<1, 32>>>(out, 64);
  k<4, 1, 540><<<1, 32>>>(out, 64);
  k<4, 6, 540><<<1, 32>>>(out, 64);
  k<4, 1, 544><<<1, 32>>>(out, 64);
  k<4, 6, 548><<<1, 32>>>(out, 64);
  k<4, 7, 540><<<1, 640>>>(out, 64);
  k<4, 7, 540><<<1, 32>>>(out, 64);
  k<1, 0><<<1, 32>>>(out, 64);
  k<1, 4><<<1, 32>>>(out, 64);
  k<1, 5><<<1, 32>>>(out, 64);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
