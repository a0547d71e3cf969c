// Hidden-layer controller on the 5th-generation tensor cores (SURVEY.md §8a
// A5; BASELINE config 5: 45 -> 128 (tanh) -> 13, reference
// hypernet.forward_batched, hypernet.py:233-252).
//
// A hidden-layer net is a dense contraction (45 x H + H x 13 MACs per cell),
// so cells are grouped by genome across the WHOLE strip (not per tile: with
// thousands of genomes a 32x32 tile holds ~1 cell per genome) and each
// genome's cells are pushed through tcgen05 MMAs in 128-row tiles:
//   k_hid_count  per-slot occupancy (smem histograms)
//   k_hid_scan   cell offsets and 128-row tile offsets per slot
//   k_hid_sense  sensor vectors (engine.py:164-177 order, 45 + 3 zero pad)
//                written to the slot's row range, one 192-byte row per cell
//   k_hid_net    persistent CTA per SM: per tile, A (128 x 48 sensors) and the
//                slot's W1 / W2 staged in shared memory in the UMMA canonical
//                K-major layout, z1 = A.W1^T by tcgen05.mma kind::tf32 into
//                TMEM, epilogue z1 + b1 -> tanh -> shared memory, z2 = h.W2^T
//                by a second MMA chain, epilogue z2 + b2 -> the reference
//                sigmoid sequence -> the cell's actuator row.
// FP32 accuracy from TF32 units: every operand is split x = hi + lo (both
// TF32) and each product accumulates lo.hi + hi.lo + hi.hi in the FP32 TMEM
// accumulator ("3xTF32"; measured max |err| / sum|a.b| = 3.6e-7,
// tools/microbench/tc_tf32.cu).  The physics then runs as pass 1 with these
// actions injected (bit-exact physics given the actions).

#include <algorithm>

#include "evoca_device.cuh"
#include "evoca_tc.cuh"

namespace evo {

namespace {

constexpr int kRows = 128;   // MMA M: cells per tile
constexpr int kK1 = 48;      // 45 sensors padded to the TF32 K granularity (8)
constexpr int kNetThreads = 256;
constexpr int kTmemCols = 512;
// The TF32 MMA accumulates in TMEM with less than FP32 rounding accuracy
// (tools/microbench/tc_split.cu: rms error 3x an FP32 FMA chain, whatever the
// operand split).  Partial sums therefore go to separate accumulators - one
// per two K=8 steps in layer 1 (3 x nh columns), one per K step in layer 2
// (nh/8 x 16 columns, reusing layer 1's columns once its epilogue has read
// them) - and are added in FP32 on the CUDA cores in k order: accuracy then
// matches (layer 1) or beats (layer 2) a sequential FP32 FMA chain.
constexpr int kL1StepsPerAcc = 2;

__global__ void k_hid_count(const int32_t* gi, long long n, int cap, int32_t* counts) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < cap; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int g = gi[i];
    if (g >= 0) atomicAdd(&hist[g], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < cap; b += blockDim.x)
    if (hist[b]) atomicAdd(&counts[b], hist[b]);
}

// exclusive scans of counts (cells) and ceil(counts / 128) (tiles); one CTA
__global__ void k_hid_scan(const int32_t* counts, int cap, int32_t* offs, int32_t* tiles, int32_t* cursor,
                           int32_t* n_tiles) {
  __shared__ int carry_c, carry_t;
  __shared__ int wc[32], wt[32];
  if (threadIdx.x == 0) carry_c = carry_t = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int b0 = 0; b0 < cap; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int c = i < cap ? counts[i] : 0, t = (c + kRows - 1) / kRows;
    int xc = c, xt = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int yc = __shfl_up_sync(0xffffffffu, xc, d), yt = __shfl_up_sync(0xffffffffu, xt, d);
      if (lane >= d) xc += yc, xt += yt;
    }
    if (lane == 31) wc[w] = xc, wt[w] = xt;
    __syncthreads();
    if (w == 0) {
      int ac = wc[lane], at = wt[lane], sc = ac, st = at;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int yc = __shfl_up_sync(0xffffffffu, sc, d), yt = __shfl_up_sync(0xffffffffu, st, d);
        if (lane >= d) sc += yc, st += yt;
      }
      wc[lane] = sc - ac;
      wt[lane] = st - at;
    }
    __syncthreads();
    if (i < cap) {
      offs[i] = carry_c + wc[w] + xc - c;
      tiles[i] = carry_t + wt[w] + xt - t;
      cursor[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry_c += wc[w] + xc, carry_t += wt[w] + xt;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offs[cap] = carry_c;
    tiles[cap] = carry_t;
    *n_tiles = carry_t;
  }
}

__global__ void k_hid_sense(const StepGeom g, const Planes f, const int32_t* offs, int32_t* cursor, float* sens,
                            int32_t* rowcell, uint8_t* flag) {
  const long long n = (long long)g.W * g.H;
  const long long st = g.stride;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(c / g.W), x = (int)(c - (long long)y * g.W);
    const long long self = (long long)(y + 1) * g.W + x;
    const int slot = f.gi[self];
    if (slot < 0) {
      flag[c] = 0;
      continue;
    }
    const int rank = offs[slot] + atomicAdd(&cursor[slot], 1);
    rowcell[rank] = (int32_t)c;
    const int rot = f.rot[self];
    float v[kK1];
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      long long o = self;
      if (s > 0) {
        const int d = perm_dir(rot, s - 1);
        int xx = x + dir_dx(d);
        xx = xx < 0 ? xx + g.W : (xx >= g.W ? xx - g.W : xx);
        o = (long long)(y + dir_dy(d) + 1) * g.W + xx;  // ghost rows -1 / H exist
      }
      v[s * 5 + 0] = __ldg(f.E + o);
      v[s * 5 + 1] = __ldg(f.I + o);
      v[s * 5 + 2] = __ldg(f.C + o);
      v[s * 5 + 3] = __ldg(f.C + st + o);
      v[s * 5 + 4] = __ldg(f.C + 2 * st + o);
    }
    v[45] = v[46] = v[47] = 0.0f;
    float4* dst = reinterpret_cast<float4*>(sens + (size_t)rank * kK1);
#pragma unroll
    for (int q = 0; q < kK1 / 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

struct NetArgs {
  Params net;
  int nh;  // hidden padded to 16: layer-1 N, layer-2 K
  const int32_t* offs;
  const int32_t* tiles;
  const int32_t* n_tiles;
  int cap;
  const float* sens;
  const int32_t* rowcell;
  float* act;
  uint8_t* flag;
};

__device__ __forceinline__ void put_split(unsigned char* hi, unsigned char* lo, uint32_t off, float x) {
  float h, l;
  tc::split_tf32(x, h, l);
  *reinterpret_cast<float*>(hi + off) = h;
  *reinterpret_cast<float*>(lo + off) = l;
}

__global__ void __launch_bounds__(kNetThreads, 1) k_hid_net(const NetArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int nh = a.nh;
  const int H = a.net.hidden, hp = a.net.hpad;
  unsigned char* B1hi = smem;
  unsigned char* B1lo = B1hi + nh * kK1 * 4;
  unsigned char* B2hi = B1lo + nh * kK1 * 4;
  unsigned char* B2lo = B2hi + 16 * nh * 4;
  float* b1 = reinterpret_cast<float*>(B2lo + 16 * nh * 4);
  float* b2 = b1 + nh;
  unsigned char* Ahi = reinterpret_cast<unsigned char*>(b2 + 16);
  Ahi = reinterpret_cast<unsigned char*>(((uintptr_t)Ahi + 1023) & ~(uintptr_t)1023);
  const int a_bytes = kRows * (nh > kK1 ? nh : kK1) * 4;
  unsigned char* Alo = Ahi + a_bytes;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int T = *a.n_tiles;
  const int per = (T + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(T, t0 + per);
  if (t0 >= t1) return;
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tmem_base);
  if (tid == 0) tc::mbar_init(&bar, 1);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  uint32_t phase = 0;
  int cur = -1;
  const uint32_t id1 = tc::idesc_tf32(kRows, nh), id2 = tc::idesc_tf32(kRows, 16);

  for (int t = t0; t < t1; ++t) {
    // slot of tile t: last s with tiles[s] <= t
    int lo = 0, hi = a.cap;  // tiles[cap] = T > t
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.tiles + mid) <= t) lo = mid; else hi = mid;
    }
    const int slot = lo;
    const int row0 = __ldg(a.offs + slot) + (t - __ldg(a.tiles + slot)) * kRows;
    const int nrows = min(kRows, __ldg(a.offs + slot + 1) - row0);
    if (slot != cur) {  // stage the slot's weights (canonical K-major, split)
      cur = slot;
      const float* W1 = a.net.wA + (size_t)slot * kSensors * hp;
      for (int i = tid; i < nh * kK1; i += kNetThreads) {
        const int h = i % nh, k = i / nh;
        const float w = (h < H && k < kSensors) ? __ldg(W1 + (size_t)k * hp + h) : 0.0f;
        put_split(B1hi, B1lo, tc::canon_off(h, k, nh), w);
      }
      const float* W2 = a.net.wB + (size_t)slot * hp * kOutPad;
      for (int i = tid; i < 16 * nh; i += kNetThreads) {
        const int j = i & 15, h = i >> 4;
        const float w = (h < H && j < kActuators) ? __ldg(W2 + (size_t)h * kOutPad + j) : 0.0f;
        put_split(B2hi, B2lo, tc::canon_off(j, h, 16), w);
      }
      for (int h = tid; h < nh; h += kNetThreads) b1[h] = h < H ? __ldg(a.net.bA + (size_t)slot * hp + h) : 0.0f;
      if (tid < 16) b2[tid] = tid < kActuators ? __ldg(a.net.bB + (size_t)slot * kOutPad + tid) : 0.0f;
    }
    // A1: 128 sensor rows, each thread half a row (24 floats)
    {
      const int r = tid >> 1, half = tid & 1;
      const float4* src = reinterpret_cast<const float4*>(a.sens + (size_t)(row0 + r) * kK1) + half * 6;
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const float4 v = r < nrows ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        const int k = (half * 6 + q) * 4;
        float4 h4, l4;
        tc::split_tf32(v.x, h4.x, l4.x);
        tc::split_tf32(v.y, h4.y, l4.y);
        tc::split_tf32(v.z, h4.z, l4.z);
        tc::split_tf32(v.w, h4.w, l4.w);
        const uint32_t off = tc::canon_off(r, k, kRows);
        *reinterpret_cast<float4*>(Ahi + off) = h4;
        *reinterpret_cast<float4*>(Alo + off) = l4;
      }
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      const uint32_t lA = kRows * 16, lB = nh * 16;
      const uint32_t ah = tc::smem_u32(Ahi), al = tc::smem_u32(Alo), bh = tc::smem_u32(B1hi), bl = tc::smem_u32(B1lo);
#pragma unroll
      for (int ks = 0; ks < kK1 / 8; ++ks) {
        const uint32_t oa = 2 * ks * lA, ob = 2 * ks * lB;
        const uint32_t d = tmem + (uint32_t)((ks / kL1StepsPerAcc) * nh);
        tc::mma_tf32(d, tc::smem_desc(al + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id1, ks % kL1StepsPerAcc);
        tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bl + ob, lB, 128), id1, 1);
        tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id1, 1);
      }
      tc::commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    // epilogue 1: z1 + b1 -> tanh -> A2 (K = hidden), warps share lane quadrants
    {
      const int q = warp & 3, r = q * 32 + lane;
      const int c_begin = (warp >> 2) * (nh / 2), c_end = c_begin + nh / 2;
      const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
      for (int c0 = c_begin; c0 < c_end; c0 += 8) {
        float v[8], p[8];
        tc::tmem_ld8(lane_base + c0, v);
#pragma unroll
        for (int g = 1; g < kK1 / 8 / kL1StepsPerAcc; ++g) {
          tc::tmem_ld8(lane_base + g * nh + c0, p);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = __fadd_rn(v[j], p[j]);
        }
        float4 h4[2], l4[2];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float th = tanhf(__fadd_rn(v[j], b1[c0 + j]));
          float hh, ll;
          tc::split_tf32(th, hh, ll);
          reinterpret_cast<float*>(h4)[j] = hh;
          reinterpret_cast<float*>(l4)[j] = ll;
        }
        *reinterpret_cast<float4*>(Ahi + tc::canon_off(r, c0, kRows)) = h4[0];
        *reinterpret_cast<float4*>(Ahi + tc::canon_off(r, c0 + 4, kRows)) = h4[1];
        *reinterpret_cast<float4*>(Alo + tc::canon_off(r, c0, kRows)) = l4[0];
        *reinterpret_cast<float4*>(Alo + tc::canon_off(r, c0 + 4, kRows)) = l4[1];
      }
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      const uint32_t lA = kRows * 16, lB = 16 * 16;
      const uint32_t ah = tc::smem_u32(Ahi), al = tc::smem_u32(Alo), bh = tc::smem_u32(B2hi), bl = tc::smem_u32(B2lo);
      for (int ks = 0; ks < nh / 8; ++ks) {
        const uint32_t oa = 2 * ks * lA, ob = 2 * ks * lB, d = tmem + (uint32_t)(ks * 16);
        tc::mma_tf32(d, tc::smem_desc(al + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id2, 0);
        tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bl + ob, lB, 128), id2, 1);
        tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id2, 1);
      }
      tc::commit(&bar);
    }
    tc::mbar_wait(&bar, phase);
    phase ^= 1;
    tc::fence_after();
    // epilogue 2: z2 + b2 -> sigmoid (hypernet.py:246-251) -> actuator row
    if (warp < 4) {
      const int r = warp * 32 + lane;
      float z[16], p[16];
      const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
      tc::tmem_ld8(lane_base, z);
      tc::tmem_ld8(lane_base + 8, z + 8);
      for (int ks = 1; ks < nh / 8; ++ks) {
        tc::tmem_ld8(lane_base + ks * 16, p);
        tc::tmem_ld8(lane_base + ks * 16 + 8, p + 8);
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = __fadd_rn(z[j], p[j]);
      }
      if (r < nrows) {
        const int cell = __ldg(a.rowcell + row0 + r);
        float* dst = a.act + (size_t)cell * kActuators;
#pragma unroll
        for (int j = 0; j < kActuators; ++j) dst[j] = squash(__fadd_rn(z[j], b2[j]));
        a.flag[cell] = 1;
      }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

int hidden_tc_nh(int hidden) { return ((hidden + 15) / 16) * 16; }

bool hidden_tc_supported(int hidden) { return hidden >= 1 && hidden_tc_nh(hidden) <= 128; }

size_t hidden_tc_smem(int hidden) {
  const int nh = hidden_tc_nh(hidden);
  const size_t fixed = (size_t)2 * nh * kK1 * 4 + (size_t)2 * 16 * nh * 4 + (size_t)(nh + 16) * 4;
  const size_t a_bytes = (size_t)kRows * (nh > kK1 ? nh : kK1) * 4;
  return ((fixed + 1023) & ~(size_t)1023) + 2 * a_bytes + 1024;  // + alignment slack
}

cudaError_t launch_hidden_tc(const HidBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                             int capacity, int num_sms, cudaStream_t st) {
  const long long n = (long long)g.W * g.H;
  cudaError_t e = cudaMemsetAsync(b.counts, 0, (size_t)capacity * 4, st);
  if (e != cudaSuccess) return e;
  const int cgrid = (int)std::min<long long>((n + 255) / 256, (long long)num_sms * 4);
  k_hid_count<<<cgrid, 256, (size_t)capacity * 4, st>>>(front.gi + g.W, n, capacity, b.counts);
  k_hid_scan<<<1, 1024, 0, st>>>(b.counts, capacity, b.offs, b.tiles, b.cursor, b.n_tiles);
  const int sgrid = (int)std::min<long long>((n + 255) / 256, (long long)num_sms * 16);
  k_hid_sense<<<sgrid, 256, 0, st>>>(g, front, b.offs, b.cursor, b.sens, b.rowcell, b.flag);
  NetArgs a;
  a.net = net;
  a.nh = hidden_tc_nh(net.hidden);
  a.offs = b.offs;
  a.tiles = b.tiles;
  a.n_tiles = b.n_tiles;
  a.cap = capacity;
  a.sens = b.sens;
  a.rowcell = b.rowcell;
  a.act = b.act;
  a.flag = b.flag;
  const size_t smem = hidden_tc_smem(net.hidden);
  e = cudaFuncSetAttribute(k_hid_net, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_hid_net<<<num_sms, kNetThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace evo
