// Field radiation selection (BASELINE config 3 extension):
// every occupied cell of the front genome plane draws one uniform from the
// host's Philox stream rng.stream(seed, t, "field_radiation")
// (/root/reference/pkg/src/evoca/rng.py:19-33) in ascending cell order - the
// r-th occupied cell takes the r-th double of the stream, exactly as
// ``stream(...).random(n_occupied)`` on the host - and is selected when
// u < p.  Selected cells are kept on the device with per-slot parent counts
// for the host; after the host admits one child per parent, evo_remap_selected
// moves the selected cells to their child slots.
//
// NumPy's Philox is Philox4x64-10 (key = 128-bit stream key as two 64-bit
// words, low first); the counter is incremented before each block, so draw r
// is word r % 4 of the block with counter r / 4 + 1; a double is
// (u64 >> 11) * 2^-53.

#include <algorithm>

#include "evoca_internal.h"

namespace evo {

namespace {

constexpr int kSelThreads = 256;
constexpr int kSelPerThread = 16;
constexpr int kSelChunk = kSelThreads * kSelPerThread;

__device__ __forceinline__ void philox4x64(unsigned long long c[4], unsigned long long k0, unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ double stream_double(unsigned long long r, unsigned long long k0, unsigned long long k1) {
  unsigned long long c[4] = {r / 4 + 1, 0, 0, 0};
  philox4x64(c, k0, k1);
  const unsigned long long w = c[r & 3];
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_occ_count(const int32_t* gi, long long n, int32_t* chunk_cnt) {
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSelChunk;
  int c = 0;
#pragma unroll
  for (int j = 0; j < kSelPerThread; ++j) {
    const long long i = base + j * kSelThreads + threadIdx.x;
    c += (i < n && gi[i] >= 0) ? 1 : 0;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = s;
}

// exclusive scan of the chunk counts (one CTA; chunk counts are few)
// (offsets start at `first`: a row strip's cells draw after those of the
// strips above it; off[nchunks] receives first + the strip's total)
__global__ void k_chunk_scan(const int32_t* cnt, long long* off, int nchunks, long long first) {
  __shared__ long long carry;
  __shared__ long long warp_tot[32];
  if (threadIdx.x == 0) carry = first;
  __syncthreads();
  for (int b0 = 0; b0 < nchunks; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    long long v = i < nchunks ? cnt[i] : 0, x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      long long t = warp_tot[lane], tx = t;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, tx, d);
        if (lane >= d) tx += y;
      }
      warp_tot[lane] = tx - t;
    }
    __syncthreads();
    if (i < nchunks) off[i] = carry + warp_tot[w] + x - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += warp_tot[w] + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[nchunks] = carry;
}

__global__ void k_select(const int32_t* gi, long long n, const long long* chunk_off, unsigned long long k0,
                         unsigned long long k1, double p, int32_t* list, unsigned long long* n_sel,
                         int32_t* parent_cnt) {
  __shared__ int warp_cnt[kSelThreads / 32];
  __shared__ long long base_s;
  const long long base = (long long)blockIdx.x * kSelChunk;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base_s = chunk_off[blockIdx.x];
  __syncthreads();
  long long rank0 = base_s;
  for (int j = 0; j < kSelPerThread; ++j) {
    const long long i = base + (long long)j * kSelThreads + threadIdx.x;
    const int g = i < n ? gi[i] : -1;
    const bool occ = g >= 0;
    const unsigned m = __ballot_sync(0xffffffffu, occ);
    if (lane == 0) warp_cnt[w] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kSelThreads / 32; ++k) {
      before += k < w ? warp_cnt[k] : 0;
      total += warp_cnt[k];
    }
    if (occ) {
      const long long r = rank0 + before + __popc(m & ((1u << lane) - 1u));
      if (stream_double((unsigned long long)r, k0, k1) < p) {
        const unsigned long long at = atomicAdd(n_sel, 1ull);
        list[at] = (int32_t)i;
        atomicAdd(&parent_cnt[g], 1);
      }
    }
    rank0 += total;
    __syncthreads();
  }
}

__global__ void k_remap(int32_t* gi, const int32_t* list, const unsigned long long* n_sel, const int32_t* map) {
  const unsigned long long n = *n_sel;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const int32_t c = list[k];
    const int32_t g = gi[c];
    if (g >= 0) {
      const int32_t to = map[g];
      if (to >= 0) gi[c] = to;
    }
  }
}

}  // namespace

int select_chunks(long long n) { return (int)((n + kSelChunk - 1) / kSelChunk); }

cudaError_t launch_count_occupied(const int32_t* gi, long long n, int32_t* chunk_cnt, long long* chunk_off,
                                  cudaStream_t st) {
  const int nch = select_chunks(n);
  if (nch == 0) return cudaMemsetAsync(chunk_off, 0, sizeof(long long), st);
  k_occ_count<<<nch, kSelThreads, 0, st>>>(gi, n, chunk_cnt);
  k_chunk_scan<<<1, 1024, 0, st>>>(chunk_cnt, chunk_off, nch, 0);
  return cudaGetLastError();
}

cudaError_t launch_select_cells(const int32_t* gi, long long n, unsigned long long k0, unsigned long long k1, double p,
                                int32_t* chunk_cnt, long long* chunk_off, int32_t* list, unsigned long long* n_sel,
                                int32_t* parent_cnt, int capacity, long long first_draw, cudaStream_t st) {
  const int nch = select_chunks(n);
  cudaError_t e = cudaMemsetAsync(n_sel, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(parent_cnt, 0, (size_t)capacity * sizeof(int32_t), st);
  if (e != cudaSuccess || nch == 0) return e;
  k_occ_count<<<nch, kSelThreads, 0, st>>>(gi, n, chunk_cnt);
  k_chunk_scan<<<1, 1024, 0, st>>>(chunk_cnt, chunk_off, nch, first_draw);
  k_select<<<nch, kSelThreads, 0, st>>>(gi, n, chunk_off, k0, k1, p, list, n_sel, parent_cnt);
  return cudaGetLastError();
}

cudaError_t launch_remap_selected(int32_t* gi, const int32_t* list, const unsigned long long* n_sel,
                                  const int32_t* map, long long max_n, cudaStream_t st) {
  if (max_n <= 0) return cudaSuccess;
  const int grid = (int)std::min<long long>((max_n + 255) / 256, 4096);
  k_remap<<<grid, 256, 0, st>>>(gi, list, n_sel, map);
  return cudaGetLastError();
}

}  // namespace evo
