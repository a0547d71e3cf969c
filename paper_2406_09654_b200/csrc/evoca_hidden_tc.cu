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
//   k_hid_net    persistent CTA per SM: per 128-row tile (one genome), A
//                (128 x 48 sensors) and the slot's W1 staged in shared
//                memory in the UMMA canonical K-major layout, z1 = A.W1^T by
//                tcgen05.mma kind::tf32 into one of two TMEM accumulator
//                buffers (the next tile's layer 1 runs during this tile's
//                epilogue); epilogue z1 + b1 -> tanh -> z2 = h.W2^T in FP32
//                FMAs -> + b2 -> the reference sigmoid sequence -> the
//                cell's actuator row.
// FP32 accuracy from TF32 units (layer 1): every operand is split x = hi +
// lo (both TF32) and each product accumulates lo.hi + hi.lo + hi.hi in the
// FP32 TMEM accumulator ("3xTF32"; measured max |err| / sum|a.b| = 3.6e-7,
// tools/microbench/tc_tf32.cu).  Layer 2 is fmaf-chained FP32 in hidden-unit
// order per quarter, the four quarter sums added in order.  The physics then runs as pass 1 with these
// actions injected (bit-exact physics given the actions).

#include <algorithm>
#include <cstdlib>

#include "evoca_gather.cuh"
#include "evoca_net.cuh"
#include "evoca_tc.cuh"

namespace evo {

// Diagnostics build (-DEVO_PHASE_TIMING): per-phase cycle sums of k_hid_net
// (thread 0 of each CTA), read with evo_debug_hidden_cycles.
__device__ unsigned long long g_hid_cycles[8];
#ifdef EVO_PHASE_TIMING
#define HID_MARK(k)                                                  \
  if (threadIdx.x == 0) {                                            \
    const long long now = clock64();                                 \
    atomicAdd(&g_hid_cycles[k], (unsigned long long)(now - t_mark)); \
    t_mark = now;                                                    \
  }
#else
#define HID_MARK(k)
#endif

namespace {

constexpr int kRows = 128;   // MMA M: cells per tile
constexpr int kK1 = 48;      // 45 sensors padded to the TF32 K granularity (8)
constexpr int kNetThreads = 512;  // 16 warps: four per TMEM lane quadrant
constexpr int kTmemCols = 512;
// The TF32 MMA accumulates in TMEM with less than FP32 rounding accuracy
// (tools/microbench/tc_split.cu: rms error 3x an FP32 FMA chain, whatever the
// operand split).  Layer-1 partial sums therefore go to two accumulators
// (three K=8 steps each, see the TMEM map at k_hid_net) added in FP32 on the
// CUDA cores in k order; actions stay within the 1e-5 relative tier-B
// tolerance of the float64 oracle (test_tensor_core_net_vs_oracle_and_cuda_core).

// Deterministic counting sort of the occupied cells by slot, without hot
// global atomics: each CTA owns kSortTiles consecutive 32x32 tiles (tile
// row-major order), histograms them in shared memory and writes the histogram
// out; a column scan turns the per-CTA histograms into per-CTA row bases; the
// sense pass then ranks cells inside the CTA with shared-memory atomics.
constexpr int kSortTiles = 16;
constexpr int kSortThreads = 256;
constexpr int kST = 32;  // sort / sense tile edge

__global__ void k_hid_count(const StepGeom g, const int32_t* gi, int cap, int32_t* cta_hist) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < cap; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int tiles_x = (g.W + kST - 1) / kST, ntiles = tiles_x * ((g.H + kST - 1) / kST);
  const int t0 = blockIdx.x * kSortTiles, t1 = min(ntiles, t0 + kSortTiles);
  for (int t = t0; t < t1; ++t) {
    const int x0 = (t % tiles_x) * kST, y0 = (t / tiles_x) * kST;
    for (int i = threadIdx.x; i < kST * kST; i += blockDim.x) {
      const int y = y0 + i / kST, x = x0 + i % kST;
      if (y >= g.H || x >= g.W) continue;
      const int s = gi[(y + 1) * g.W + x];
      if (s >= 0) atomicAdd(&hist[s], 1);
    }
  }
  __syncthreads();
  int32_t* out = cta_hist + (size_t)blockIdx.x * cap;
  for (int b = threadIdx.x; b < cap; b += blockDim.x) out[b] = hist[b];
}

// per slot: exclusive scan of the per-CTA counts over CTAs (in place) and the
// slot total.  One CTA per 32 slots: lane = slot (coalesced), warp w owns a
// contiguous chunk of the sort CTAs; chunk sums are scanned across warps in
// shared memory.
__global__ void __launch_bounds__(1024) k_hid_colscan(int32_t* cta_hist, int nctas, int cap, int32_t* counts) {
  __shared__ int part[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = blockIdx.x * 32 + lane;
  const int per = (nctas + 31) / 32, c0 = w * per, c1 = min(nctas, c0 + per);
  int sum = 0;
  if (g < cap)
    for (int c = c0; c < c1; ++c) sum += cta_hist[(size_t)c * cap + g];
  part[w][lane] = sum;
  __syncthreads();
  if (w == 0) {
    int run = 0;
    for (int k = 0; k < 32; ++k) {
      const int v = part[k][lane];
      part[k][lane] = run;
      run += v;
    }
    if (g < cap) counts[g] = run;
  }
  __syncthreads();
  int run = part[w][lane];
  if (g < cap)
    for (int c = c0; c < c1; ++c) {
      int32_t* p = cta_hist + (size_t)c * cap + g;
      const int v = *p;
      *p = run;
      run += v;
    }
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

// Sensor rows.  Element 45 of a row carries the cell index (its bit
// pattern; rows' pad columns meet zero weights, and index bits below
// 0x7F800000 are finite floats, evo_create bounds the strip), so the net
// kernel needs no separate row -> cell map.  Per 32x32 tile the five sensed
// planes' halo (34 x 34) is staged in shared memory with coalesced loads;
// each warp assembles 32 rows from it and writes them out cooperatively (12
// lanes per 192-byte row, whole sectors per store instruction).
constexpr int kRowPitch = 52;  // floats per staged row: 16-byte rows, 13 x 16 B apart (conflict-free STS/LDS.128)
constexpr int kSH = kST + 2;   // halo edge

struct SenseSmem {
  float4 eic[kSH * kSH];  // {E, I, C0, C1} interleaved: one LDS.128 per Moore slot
  float c2[kSH * kSH];
  int gi[kST * kST];
  uint8_t rot[kST * kST];
  float stage[kSortThreads / 32][32 * kRowPitch];
};

size_t sense_smem_bytes(int cap) { return sizeof(SenseSmem) + (size_t)((cap + 3) & ~3) * 4; }

__global__ void __launch_bounds__(kSortThreads, 2) k_hid_sense(const StepGeom g, const Planes f, const int32_t* offs,
                                                            const int32_t* cta_base, int cap, float* sens,
                                                            int32_t* rank_of_cell, int identity_rank) {
  extern __shared__ __align__(16) unsigned char sraw[];
  SenseSmem& sm = *reinterpret_cast<SenseSmem*>(sraw);
  int* cursor = reinterpret_cast<int*>(sraw + sizeof(SenseSmem));
  const int32_t* base = cta_base + (size_t)blockIdx.x * cap;
  for (int b = threadIdx.x; b < cap; b += blockDim.x) cursor[b] = __ldg(offs + b) + __ldg(base + b);
  const int tiles_x = (g.W + kST - 1) / kST, ntiles = tiles_x * ((g.H + kST - 1) / kST);
  const int t0 = blockIdx.x * kSortTiles, t1 = min(ntiles, t0 + kSortTiles);
  const int st = (int)g.stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* stage = sm.stage[warp];
  // the next tile's halo planes, genome and rotation are loaded into
  // registers while the current tile's rows are assembled and stored
  constexpr int kPH = (kSH * kSH + kSortThreads - 1) / kSortThreads;
  constexpr int kPC = (kST * kST) / kSortThreads;
  float pv[kPH][5];
  int pg[kPC], pr[kPC];
  auto load_tile = [&](int t) {
    const int x0 = (t % tiles_x) * kST, y0 = (t / tiles_x) * kST;
#pragma unroll
    for (int j = 0; j < kPH; ++j) {
      const int i = threadIdx.x + j * kSortThreads;
      if (i < kSH * kSH) {
        const int hy = i / kSH, hx = i - hy * kSH;
        int y = y0 + hy - 1;
        y = y > g.H ? g.H : y;  // beyond a partial tile: never read
        int x = x0 + hx - 1;
        x = x < 0 ? x + g.W : (x >= g.W ? x - g.W : x);
        x = x >= g.W ? g.W - 1 : x;
        const int o = (y + 1) * g.W + x;
        pv[j][0] = __ldg(f.E + o);
        pv[j][1] = __ldg(f.I + o);
        pv[j][2] = __ldg(f.C + o);
        pv[j][3] = __ldg(f.C + st + o);
        pv[j][4] = __ldg(f.C + 2 * st + o);
      }
    }
#pragma unroll
    for (int j = 0; j < kPC; ++j) {
      const int i = threadIdx.x + j * kSortThreads;
      const int y = y0 + i / kST, x = x0 + i % kST;
      const bool in = y < g.H && x < g.W;
      const int o = (y + 1) * g.W + x;
      pg[j] = in ? __ldg(f.gi + o) : -1;
      pr[j] = in ? (int)__ldg(f.rot + o) : 0;
    }
  };
  if (t0 < t1) load_tile(t0);
  for (int t = t0; t < t1; ++t) {
    const int x0 = (t % tiles_x) * kST, y0 = (t / tiles_x) * kST;
    __syncthreads();  // previous tile's readers are done (and cursor init on the first pass)
#pragma unroll
    for (int j = 0; j < kPH; ++j) {
      const int i = threadIdx.x + j * kSortThreads;
      if (i < kSH * kSH)
#pragma unroll
      {
        sm.eic[i] = make_float4(pv[j][0], pv[j][1], pv[j][2], pv[j][3]);
        sm.c2[i] = pv[j][4];
      }
    }
#pragma unroll
    for (int j = 0; j < kPC; ++j) {
      const int i = threadIdx.x + j * kSortThreads;
      sm.gi[i] = pg[j];
      sm.rot[i] = (uint8_t)pr[j];
    }
    __syncthreads();
    if (t + 1 < t1) load_tile(t + 1);
    for (int cb = warp * 32; cb < kST * kST; cb += blockDim.x) {
      const int i = cb + lane, ty = i / kST, tx = i - ty * kST;
      const int y = y0 + ty, x = x0 + tx;
      const int slot = sm.gi[i];
      int rank = -1;
      if (y < g.H && x < g.W) {
        const int c = y * g.W + x;
        if (slot >= 0) {
          rank = atomicAdd(&cursor[slot], 1);
          const int rot = sm.rot[i];
          const int hb = (ty + 1) * kSH + tx + 1;
          float v[kK1];
#pragma unroll
          for (int s = 0; s < 9; ++s) {
            const int hp = s == 0 ? hb : hb + dir_dy(perm_dir(rot, s - 1)) * kSH + dir_dx(perm_dir(rot, s - 1));
            const float4 q = sm.eic[hp];
            v[s * 5 + 0] = q.x;
            v[s * 5 + 1] = q.y;
            v[s * 5 + 2] = q.z;
            v[s * 5 + 3] = q.w;
            v[s * 5 + 4] = sm.c2[hp];
          }
          v[45] = __int_as_float(c);
          v[46] = v[47] = 0.0f;
          float4* row = reinterpret_cast<float4*>(stage + lane * kRowPitch);
#pragma unroll
          for (int part = 0; part < 12; ++part)
            row[part] = make_float4(v[4 * part], v[4 * part + 1], v[4 * part + 2], v[4 * part + 3]);
        }
        // (identity_rank: the net writes each actuator row at its cell index)
        if (rank_of_cell) rank_of_cell[c] = identity_rank ? (rank >= 0 ? c : -1) : rank;
      }
      __syncwarp();
      for (int k = lane; k < 32 * 12; k += 32) {  // 12 lanes per 192-byte row
        const int r = k / 12, part = k - r * 12;
        const int rk = __shfl_sync(0xffffffffu, rank, r);
        if (rk >= 0) {
          reinterpret_cast<float4*>(sens + (size_t)rk * kK1)[part] =
              *reinterpret_cast<const float4*>(stage + r * kRowPitch + part * 4);
        }
      }
      __syncwarp();
    }
  }
}

// x = hi + lo with hi = x truncated to TF32 (low 13 mantissa bits cleared)
// and lo = x - hi exact in FP32 (the tensor core reads lo's top 11 bits:
// error <= 2^-22 |x|, below the accumulation error, tools/microbench/
// tc_split.cu); 2 instructions instead of two TF32 round-to-nearest cvts.
__device__ __forceinline__ void split_fast(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// tanh(x) = 1 - 2 / (1 + 2^(2x log2 e)) with the SFU exp2 / reciprocal:
// absolute error ~2e-7 (the hidden activations only enter the next dot
// product, where absolute error is what counts), 2 MUFU + 3 FMA-pipe ops
// instead of the libdevice tanhf sequence.
__device__ __forceinline__ float tanh_sfu(float x) {
  float t, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(x * 2.8853900817779268f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + t));
  return fmaf(-2.0f, r, 1.0f);
}

// per 128-row tile: {slot, first row, rows, 0} - one 16-byte load per tile
// tile -> {slot, first row, rows}: one thread per tile, slot found by binary
// search over the per-slot tile offsets (a per-slot loop serialised ~500
// tiles per thread on config 3)
__global__ void k_hid_tilemap(const int32_t* offs, const int32_t* tiles, int cap, const int32_t* n_tiles,
                              int4* tile_info) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= *n_tiles) return;
  int lo = 0, hi = cap;  // largest g with tiles[g] <= t (tiles[cap] = n_tiles > t)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(tiles + mid) <= t) lo = mid; else hi = mid;
  }
  const int row0 = __ldg(offs + lo) + (t - __ldg(tiles + lo)) * kRows;
  tile_info[t] = make_int4(lo, row0, min(kRows, __ldg(offs + lo + 1) - row0), 0);
}

struct NetArgs {
  Params net;
  int nh;  // hidden padded to 16: layer-1 N, layer-2 K
  const int32_t* offs;
  const int32_t* tiles;
  const int32_t* n_tiles;
  const int4* tile_info;
  int cap;
  const float* sens;
  float* act;  // [rows][16], or [rows][8] decided rows (direct nets, no export)
  int decided;
  // gather form (k_hid_net2<true>): sorted cell list and sense texture
  // instead of sensor rows; actuator rows land at the cell index
  const uint32_t* sorted;
  const float* tex;
  int W;
  int contig;  // gather form: contiguous tile range per CTA instead of claimed runs
  const unsigned char* htab;  // gather form: per-slot pre-split tables (hid_table_bytes each)
};

__device__ __forceinline__ void put_split(unsigned char* hi, unsigned char* lo, uint32_t off, float x) {
  float h, l;
  tc::split_tf32(x, h, l);
  *reinterpret_cast<float*>(hi + off) = h;
  *reinterpret_cast<float*>(lo + off) = l;
}

// TMEM map (512 columns, lanes = the tile's 128 rows): two layer-1
// accumulator buffers, one per tile in flight; buffer b at columns
// [256 b, 256 b + 2 nh): accumulator 0 (K steps 0-2) in the first nh columns,
// accumulator 1 (K steps 3-5) in the next nh.  Layer 2 (45->H->13: H x 13
// MACs per cell, N = 13) runs on the CUDA cores inside the tanh epilogue:
// as 13-column tensor-core MMAs it was issue-bound (32 tcgen05.mma of
// ~60 issue cycles each per tile, tools/microbench/tc_rate.cu), and keeping
// it off the tensor core frees the TMEM that lets the next tile's layer 1 run
// during this tile's epilogue.
constexpr int kAccBuf = 256;  // TMEM columns per layer-1 accumulator buffer
constexpr int kXPitch = 4 * kActuators + 1;  // exchange row: 4 quarter sums x 13, odd pitch

__global__ void __launch_bounds__(kNetThreads, 1) k_hid_net(const NetArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int nh = a.nh;
  const int H = a.net.hidden, hp = a.net.hpad;
  unsigned char* B1hi = smem;
  unsigned char* B1lo = B1hi + nh * kK1 * 4;
  float* W2s = reinterpret_cast<float*>(B1lo + nh * kK1 * 4);  // [nh][16]: W2^T rows
  float* b1 = W2s + nh * 16;
  float* b2 = b1 + nh;
  float* xbuf = b2 + 16;  // [kRows][kXPitch] quarter-sum exchange (odd pitch: conflict-free)
  unsigned char* A1 = reinterpret_cast<unsigned char*>(((uintptr_t)(xbuf + kRows * kXPitch) + 1023) & ~(uintptr_t)1023);
  constexpr int kA1Bytes = kRows * kK1 * 4;  // one of hi / lo
  // A1 double buffer: buffer i at A1 + i * 2 * kA1Bytes (hi) and + kA1Bytes (lo)
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int T = *a.n_tiles;
  const int per = (T + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(T, t0 + per);
  if (t0 >= t1) return;
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  uint32_t ph0 = 0u, ph1 = 0u;
  const uint32_t id1 = tc::idesc_tf32(kRows, nh);
  const bool issuer = tid == 4 * 32;

  const int ar = tid >> 2, aq = tid & 3;  // this thread's quarter sensor row (staging)
  float4 pf[3];
  auto fetch = [&](const int4 ti) {
    const float4* src = reinterpret_cast<const float4*>(a.sens + (size_t)(ti.y + ar) * kK1) + aq * 3;
#pragma unroll
    for (int q = 0; q < 3; ++q) pf[q] = ar < ti.z ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  // split the prefetched quarter row into A1 buffer `buf` (canonical
  // layout); element 45 of a row is its cell index
  auto stage_a1 = [&](int buf) {
    unsigned char* hi = A1 + buf * 2 * kA1Bytes;
    unsigned char* lo = hi + kA1Bytes;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float4 v = pf[q];
      // (never written back into pf: a modified component made the compiler
      // copy it right after its load, exposing the whole load latency)
      if (q == 2 && aq == 3) v.y = 0.0f;
      float4 h4, l4;
      split_fast(v.x, h4.x, l4.x);
      split_fast(v.y, h4.y, l4.y);
      split_fast(v.z, h4.z, l4.z);
      split_fast(v.w, h4.w, l4.w);
      const uint32_t off = tc::canon_off(ar, (aq * 3 + q) * 4, kRows);
      *reinterpret_cast<float4*>(hi + off) = h4;
      *reinterpret_cast<float4*>(lo + off) = l4;
    }
  };
  auto stage_weights = [&](int slot) {
    const float* W1 = a.net.wA + (size_t)slot * kSensors * hp;
    for (int i = tid; i < nh * kK1; i += kNetThreads) {
      const int h = i % nh, k = i / nh;
      const float w = (h < H && k < kSensors) ? __ldg(W1 + (size_t)k * hp + h) : 0.0f;
      put_split(B1hi, B1lo, tc::canon_off(h, k, nh), w);
    }
    const float* W2 = a.net.wB + (size_t)slot * hp * kOutPad;
    for (int i = tid; i < 16 * nh; i += kNetThreads) {
      const int j = i & 15, h = i >> 4;
      W2s[i] = (h < H && j < kActuators) ? __ldg(W2 + (size_t)h * kOutPad + j) : 0.0f;
    }
    for (int h = tid; h < nh; h += kNetThreads) b1[h] = h < H ? __ldg(a.net.bA + (size_t)slot * hp + h) : 0.0f;
    if (tid < 16) b2[tid] = tid < kActuators ? __ldg(a.net.bB + (size_t)slot * kOutPad + tid) : 0.0f;
  };
  // layer 1 of the tile in A1 buffer `buf` into TMEM buffer `buf`: 6 K steps x
  // (lo.hi, hi.lo, hi.hi), accumulator 0 for steps 0-2, accumulator 1 for 3-5
  auto issue_l1 = [&](int buf) {
    if (issuer) {
      const uint32_t lA = kRows * 16, lB = nh * 16;
      const uint32_t ah = tc::smem_u32(A1 + buf * 2 * kA1Bytes), al = ah + kA1Bytes;
      const uint32_t bh = tc::smem_u32(B1hi), bl = tc::smem_u32(B1lo);
      const uint32_t tb = tmem + (uint32_t)(buf * kAccBuf);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int acc = 0; acc < 2; ++acc) {
          const int ks = acc * 3 + j;
          const uint32_t oa = 2 * ks * lA, ob = 2 * ks * lB;
          const uint32_t d = tb + (acc ? (uint32_t)nh : 0u);
          tc::mma_tf32(d, tc::smem_desc(al + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id1, j > 0);
          tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bl + ob, lB, 128), id1, 1);
          tc::mma_tf32(d, tc::smem_desc(ah + oa, lA, 128), tc::smem_desc(bh + ob, lB, 128), id1, 1);
        }
      tc::commit(&bar[buf]);
    }
  };

  // tile infos t, t + 1, t + 2, t + 3 ride along in registers, so that no
  // row fetch waits on a dependent tile-info load
  const int4 z4 = make_int4(0, 0, 0, 0);
  int4 ti0 = __ldg(a.tile_info + t0);
  int4 ti1 = t0 + 1 < t1 ? __ldg(a.tile_info + t0 + 1) : z4;
  int4 ti2 = t0 + 2 < t1 ? __ldg(a.tile_info + t0 + 2) : z4;
  int4 ti3 = t0 + 3 < t1 ? __ldg(a.tile_info + t0 + 3) : z4;
  int cur = ti0.x;
  fetch(ti0);
  stage_weights(cur);
  stage_a1(0);
  if (t0 + 1 < t1) {
    fetch(ti1);
    stage_a1(1);
  }
  if (t0 + 2 < t1) fetch(ti2);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  issue_l1(0);
  long long t_mark = clock64();
  (void)t_mark;

  const int q = warp & 3, qt = warp >> 2;  // TMEM lane quadrant, hidden-unit quarter
  const int r = q * 32 + lane;               // this thread's tile row (TMEM lane)
  const int c_begin = qt * (nh / 4), c_end = c_begin + nh / 4;
  for (int t = t0; t < t1; ++t) {
    const int buf = (t - t0) & 1;
    const int4 ti = ti0;
    const bool has_next = t + 1 < t1;
    const int next_slot = has_next ? ti1.x : cur;
    ti0 = ti1;
    ti1 = ti2;
    ti2 = ti3;
    ti3 = t + 4 < t1 ? __ldg(a.tile_info + t + 4) : z4;
    // (a) the next tile's layer 1 (same genome: its weights are resident) runs
    //     on the tensor core during this tile's epilogue
    const bool early = has_next && next_slot == cur;
    if (early) issue_l1(buf ^ 1);
    HID_MARK(0);
    tc::mbar_wait(&bar[buf], buf ? ph1 : ph0);
    if (buf) ph1 ^= 1u; else ph0 ^= 1u;
    tc::fence_after();
    HID_MARK(1);
    // (b) rows of tile t + 2 into this tile's A1 buffer (its layer 1 is done),
    //     then the rows of tile t + 3 into registers
    if (t + 2 < t1) stage_a1(buf);
    if (t + 3 < t1) fetch(ti2);  // (shifted: ti2 now holds tile t + 3)
    HID_MARK(2);
    // (c) epilogue: z1 = acc0 + acc1 + b1 -> tanh -> z2 += h W2 (FP32, h
    //     ascending) over this thread's quarter of the hidden units
    {
      const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kAccBuf);
      u64 z2p[6];
      float z12 = 0.0f;
#pragma unroll
      for (int p = 0; p < 6; ++p) z2p[p] = 0ull;
      auto column = [&](int h, float s) {
        const float th = tanh_sfu(__fadd_rn(s, b1[h]));
        const float4* w4 = reinterpret_cast<const float4*>(W2s + h * 16);
        const float4 wa = w4[0], wb = w4[1], wc = w4[2], wd = w4[3];
        ffma2(z2p[0], th, pk2(wa.x, wa.y));
        ffma2(z2p[1], th, pk2(wa.z, wa.w));
        ffma2(z2p[2], th, pk2(wb.x, wb.y));
        ffma2(z2p[3], th, pk2(wb.z, wb.w));
        ffma2(z2p[4], th, pk2(wc.x, wc.y));
        ffma2(z2p[5], th, pk2(wc.z, wc.w));
        z12 = fmaf(th, wd.x, z12);
      };
      uint32_t v[16], pv[16];
      int c0 = c_begin;
      if (c0 + 16 <= c_end) {
        tc::tmem_ld16_nw(lb + c0, v);
        tc::tmem_ld16_nw(lb + nh + c0, pv);
      }
      for (; c0 + 16 <= c_end; c0 += 16) {  // 16-column chunks, the next chunk's loads in flight
        tc::tmem_wait_ld();
        tc::reg_fence(v);
        tc::reg_fence(pv);
        float sum[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) sum[j] = __fadd_rn(__uint_as_float(v[j]), __uint_as_float(pv[j]));
        if (c0 + 32 <= c_end) {
          tc::tmem_ld16_nw(lb + c0 + 16, v);
          tc::tmem_ld16_nw(lb + nh + c0 + 16, pv);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) column(c0 + j, sum[j]);
      }
      for (; c0 < c_end; c0 += 4) {  // 4-column tail (nh / 4 is a multiple of 4)
        uint32_t va[4], pa[4];
        tc::tmem_ld4_nw(lb + c0, va);
        tc::tmem_ld4_nw(lb + nh + c0, pa);
        tc::tmem_wait_ld();
        tc::reg_fence(va);
        tc::reg_fence(pa);
#pragma unroll
        for (int j = 0; j < 4; ++j) column(c0 + j, __fadd_rn(__uint_as_float(va[j]), __uint_as_float(pa[j])));
      }
      float z2[kActuators];
#pragma unroll
      for (int p = 0; p < 6; ++p) up2(z2p[p], z2[2 * p], z2[2 * p + 1]);
      z2[12] = z12;
      // (d) quarter sums through shared memory; thread quarter qt finishes
      //     outputs 4 qt .. 4 qt + 3 as ((q0 + q1) + q2) + q3 + b2
      float* xr = xbuf + r * kXPitch;
#pragma unroll
      for (int j = 0; j < kActuators; ++j) xr[qt * kActuators + j] = z2[j];
      HID_MARK(3);
      __syncthreads();
      HID_MARK(4);
      const int jh = qt * 4;
      if (r < ti.z) {  // actuator row at its sorted position: 16-byte quarters, coalesced
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int jj = jh + j;
          if (jj < kActuators) {
            float zz = __fadd_rn(xr[jj], xr[kActuators + jj]);
            zz = __fadd_rn(zz, xr[2 * kActuators + jj]);
            zz = __fadd_rn(zz, xr[3 * kActuators + jj]);
            o[j] = squash(__fadd_rn(zz, b2[jj]));
          } else {
            o[j] = 0.0f;
          }
        }
        reinterpret_cast<float4*>(a.act + (size_t)(ti.y + r) * 16)[qt] = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    HID_MARK(5);
    // (e) end of tile: TMEM buffer, exchange rows and staged A1 free / visible
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (has_next && !early) {  // genome change: restage the weights, then layer 1
      cur = next_slot;
      stage_weights(cur);
      tc::fence_async_smem();
      tc::fence_before();
      __syncthreads();
      tc::fence_after();
      issue_l1(buf ^ 1);
    }
    HID_MARK(6);
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

// Both layers on the tensor core (k_hid_net2, the default for hidden sizes
// the TMEM map below holds; EVO_F_L2_CUDA_CORE selects k_hid_net).  Per
// 128-row tile (one genome), 512 threads, one CTA per SM, TMEM:
//   [0, nh)        layer-1 accumulator 0 (K steps 0-2), then h_hi in place
//   [nh, 2 nh)     layer-1 accumulator 1 (K steps 3-5), then h_lo in place
//   [256 + 32 i, 288 + 32 i)  layer-2 accumulator i = 0..3 (a quarter of
//                  the hidden K steps each)
// (1) layer 1 as in k_hid_net (3xTF32: lo.hi + hi.lo + hi.hi, A and B in
//     shared memory); (2) epilogue 1: each thread (row r = TMEM lane, hidden
//     quarter qt) reads its 2 x nh/4 accumulator columns, z1 = acc0 + acc1 +
//     b1, h = tanh(z1), split h = hi + lo (hi = h with the low 13 mantissa
//     bits cleared) and writes h_hi / h_lo over the columns it read
//     (tcgen05.st; each thread owns those lane/column cells); (3) layer 2:
//     A = h_hi / h_lo from TMEM, B = [W2_hi | W2_lo] (N = 32, K = nh) in
//     shared memory, two MMAs per K step (lo.lo included) into the
//     accumulator of its half of the hidden units (kL2Acc = 2); (4) as soon
//     as layer 2 has read h, the next tile's layer 1 goes out and the
//     epilogue 2 (four warps: z2_j = the partial sums (W2_hi and W2_lo
//     columns added first) in order + b2_j, the reference sigmoid sequence,
//     the actuator row) overlaps it.
// Accuracy (test_tensor_core_net_vs_oracle_and_cuda_core, H = 128): actions
// 7.8e-6 from the float64 oracle against 2.9e-6 with layer 2 in FP32 FMAs;
// four accumulators gave 6.6e-6 (0.3 ms slower per config-5 step), lo
// rounded to nearest TF32 (cvt.rna, on the saturated conversion pipe) 6.8e-6
// (0.4 ms slower): the error is the tensor core's own rounding inside each
// K = 8 step, not the split or the accumulation length.  Layer 2 on the CUDA cores (k_hid_net)
//     was bound by the W2 broadcasts from shared memory (each lane receives
//     its own copy; 57 % of the tile in the epilogue, round-1 phase timing).
constexpr uint32_t kL2 = 256;  // layer-2 accumulators: kL2Acc x 32 columns
constexpr int kHgRun = 2;     // gather form: consecutive tiles per claim
constexpr int kL2Acc = 2;

__device__ __forceinline__ void tmem_st4(uint32_t addr, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a0), "r"(a1), "r"(a2),
               "r"(a3));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(tc::smem_u32(bar))
      : "memory");
}

size_t hidden_tc2_smem(int hidden) {
  const int nh = hidden_tc_nh(hidden);
  const size_t fixed = (size_t)2 * nh * kK1 * 4 + (size_t)32 * nh * 4 + (size_t)(nh + 16) * 4;
  return ((fixed + 1023) & ~(size_t)1023) + (size_t)4 * kRows * kK1 * 4 + 1024;
}

// Per-slot pre-split tables of k_hid_net2 in its shared-memory layout:
// B1hi | B1lo (canonical K-major, N = nh) | B2 = [W2_hi | W2_lo] (N = 32) |
// b1 (nh) | b2 (16), built once per weight change (k_hid_tables) and copied
// whole by cp.async.bulk when the gather form changes slot.
__host__ __device__ inline int hid_table_bytes(int nh) { return 2 * nh * kK1 * 4 + 32 * nh * 4 + (nh + 16) * 4; }

__global__ void k_hid_tables(const Params net, int nh, unsigned char* out) {
  const int slot = blockIdx.x;
  const int H = net.hidden, hp = net.hpad;
  unsigned char* B1hi = out + (size_t)slot * hid_table_bytes(nh);
  unsigned char* B1lo = B1hi + nh * kK1 * 4;
  unsigned char* B2 = B1lo + nh * kK1 * 4;
  float* b1 = reinterpret_cast<float*>(B2 + 32 * nh * 4);
  float* b2 = b1 + nh;
  const float* W1 = net.wA + (size_t)slot * kSensors * hp;
  for (int i = threadIdx.x; i < nh * kK1; i += blockDim.x) {
    const int h = i % nh, k = i / nh;
    const float w = (h < H && k < kSensors) ? __ldg(W1 + (size_t)k * hp + h) : 0.0f;
    put_split(B1hi, B1lo, tc::canon_off(h, k, nh), w);
  }
  const float* W2 = net.wB + (size_t)slot * hp * kOutPad;
  for (int i = threadIdx.x; i < 16 * nh; i += blockDim.x) {
    const int j = i & 15, h = i >> 4;
    const float w = (h < H && j < kActuators) ? __ldg(W2 + (size_t)h * kOutPad + j) : 0.0f;
    float wh, wl;
    split_fast(w, wh, wl);
    *reinterpret_cast<float*>(B2 + tc::canon_off(j, h, 32)) = wh;
    *reinterpret_cast<float*>(B2 + tc::canon_off(16 + j, h, 32)) = wl;
  }
  for (int h = threadIdx.x; h < nh; h += blockDim.x) b1[h] = h < H ? __ldg(net.bA + (size_t)slot * hp + h) : 0.0f;
  if (threadIdx.x < 16) b2[threadIdx.x] = threadIdx.x < kActuators ? __ldg(net.bB + (size_t)slot * kOutPad + threadIdx.x) : 0.0f;
}

template <bool GATHER>
__global__ void __launch_bounds__(kNetThreads, 1) k_hid_net2(const NetArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int nh = a.nh;
  const int H = a.net.hidden, hp = a.net.hpad;
  // the slot's tables: B1hi | B1lo | B2 = [W2_hi | W2_lo] (N = 32, K = nh,
  // canonical) | b1 | b2 (hid_table_bytes); the gather form keeps a second
  // copy after the A1 buffers, filled by a bulk copy of the next slot's
  // pre-split table while the current tile runs
  const int tab = hid_table_bytes(nh);
  unsigned char* wbase[2];
  wbase[0] = smem;
  unsigned char* A1 = smem + ((tab + 1023) & ~1023);
  constexpr int kA1Bytes = kRows * kK1 * 4;  // one of hi / lo; buffer i at A1 + i * 2 * kA1Bytes
  wbase[1] = A1 + 4 * kA1Bytes;
  int wb = 0;
  unsigned char* B1hi = wbase[0];
  unsigned char* B1lo = B1hi + nh * kK1 * 4;
  unsigned char* B2 = B1lo + nh * kK1 * 4;
  float* b1 = reinterpret_cast<float*>(B2 + 32 * nh * 4);
  float* b2 = b1 + nh;
  auto use_weights = [&](int w) {
    wb = w;
    B1hi = wbase[w];
    B1lo = B1hi + nh * kK1 * 4;
    B2 = B1lo + nh * kK1 * 4;
    b1 = reinterpret_cast<float*>(B2 + 32 * nh * 4);
    b2 = b1 + nh;
  };
  __shared__ __align__(8) uint64_t wbar;  // gather form: the bulk weight copy
  uint32_t wph = 0u;
  // thread 0: the slot's pre-split table into weight buffer w (async)
  auto fetch_weights = [&](int slot, int w) {
    const uint32_t mb = tc::smem_u32(&wbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(tab) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tc::smem_u32(wbase[w])),
        "l"(a.htab + (size_t)slot * tab), "r"(tab), "r"(mb)
        : "memory");
  };
  auto wait_weights = [&]() {
    tc::mbar_wait(&wbar, wph);
    wph ^= 1u;
  };
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];  // 0: layer 1 done, 1: layer 2 done
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // Tile sequence.  Rows form: one contiguous range per CTA (a genome's
  // tiles stay together, its tables staged once).  Gather form: runs of
  // kHgRun tiles claimed from one counter, so all CTAs sweep the row bands
  // together and the band's texture stays in L2 (a contiguous range per CTA
  // would gather from every band at once: 9.2 ms against 3.7 ms per
  // config-5 net); the run after next is claimed two runs ahead (ring).
  __shared__ int ring[4];
  const int T = a.n_tiles[0];
  int32_t* const counter = const_cast<int32_t*>(a.n_tiles) + 1;  // gather form: n_ht[1], zeroed by the sort
  int t = 0, tend = T, k = 0;
  const bool dyn = GATHER && !a.contig;
  if (dyn) {
    if (tid == 0) {
      ring[3] = atomicAdd(counter, 1) * kHgRun;
      ring[0] = atomicAdd(counter, 1) * kHgRun;
      ring[1] = atomicAdd(counter, 1) * kHgRun;
    }
    __syncthreads();
    t = ring[3];
  } else {
    const int per = (T + gridDim.x - 1) / gridDim.x;
    t = blockIdx.x * per;
    tend = min(T, t + per);
  }
  // the tile after u (T = none); thread 0 refills the ring slot two runs
  // ahead of the one consumed (read only after >= kHgRun barriers)
  auto next_tile = [&](int u) {
    if (u >= tend) return T;
    if (!dyn) return u + 1 < tend ? u + 1 : T;
    if ((u + 1) % kHgRun) return u + 1 < T ? u + 1 : T;
    const int nx = ring[k & 3];
    if (tid == 0) ring[(k + 2) & 3] = atomicAdd(counter, 1) * kHgRun;
    ++k;
    return nx < T ? nx : T;
  };
  if (t >= tend) return;
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tmem_base);
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::mbar_init(&wbar, 1);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  uint32_t ph0 = 0u, ph1 = 0u;
  const uint32_t id1 = tc::idesc_tf32(kRows, nh), id2 = tc::idesc_tf32(kRows, 32);

  const int ar = tid >> 2, aq = tid & 3;  // staging: this thread's quarter sensor row (k = 12 aq .. 12 aq + 11)
  float4 pf[3];
  // gather form: the Moore records this quarter row needs (Moore slots
  // sb .. sb + 3 of the cell's own order; k = 5 s + ch)
  gs::f8r rec[4];
  const int sb = aq == 0 ? 0 : aq == 1 ? 2 : aq == 2 ? 4 : 7;
  auto fetch = [&](const int4 ti) {
    if (GATHER) {
      const gs::GCell c = gs::gcell(__ldg(a.sorted + ti.y + (ar < ti.z ? ar : 0)), a.W);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (sb + j <= 8) rec[j] = gs::ld_rec(gs::rec_ptr(a.tex, c, a.W, c.rot, sb + j));
    } else {
      const float4* src = reinterpret_cast<const float4*>(a.sens + (size_t)(ti.y + ar) * kK1) + aq * 3;
#pragma unroll
      for (int q = 0; q < 3; ++q) pf[q] = ar < ti.z ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  // the quarter row from the records (selects, no divergence: the four
  // quarters of a row sit on neighbouring lanes)
  auto assemble = [&]() {
    float v[12];
#pragma unroll
    for (int kk = 0; kk < 12; ++kk) {
      float x0, x1, x2, x3;
      {  // aq = 0: k = kk
        const int k = kk, s = k / 5;
        x0 = rec[s - 0].v[gs::tex_ch(k % 5)];
      }
      {  // aq = 1: k = 12 + kk
        const int k = 12 + kk, s = k / 5;
        x1 = rec[s - 2].v[gs::tex_ch(k % 5)];
      }
      {  // aq = 2: k = 24 + kk
        const int k = 24 + kk, s = k / 5;
        x2 = rec[s - 4].v[gs::tex_ch(k % 5)];
      }
      {  // aq = 3: k = 36 + kk (45 .. 47 pad)
        const int k = 36 + kk, s = k / 5;
        x3 = k < kSensors ? rec[s - 7].v[gs::tex_ch(k % 5)] : 0.0f;
      }
      v[kk] = aq == 0 ? x0 : aq == 1 ? x1 : aq == 2 ? x2 : x3;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) pf[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  };
  auto stage_a1 = [&](int buf) {
    unsigned char* hi = A1 + buf * 2 * kA1Bytes;
    unsigned char* lo = hi + kA1Bytes;
    if (GATHER) assemble();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float4 v = pf[q];
      if (!GATHER && q == 2 && aq == 3) v.y = 0.0f;  // element 45 of a sensor row is the cell index
      float4 h4, l4;
      split_fast(v.x, h4.x, l4.x);
      split_fast(v.y, h4.y, l4.y);
      split_fast(v.z, h4.z, l4.z);
      split_fast(v.w, h4.w, l4.w);
      const uint32_t off = tc::canon_off(ar, (aq * 3 + q) * 4, kRows);
      *reinterpret_cast<float4*>(hi + off) = h4;
      *reinterpret_cast<float4*>(lo + off) = l4;
    }
  };
  auto stage_weights = [&](int slot) {
    const float* W1 = a.net.wA + (size_t)slot * kSensors * hp;
    for (int i = tid; i < nh * kK1; i += kNetThreads) {
      const int h = i % nh, k = i / nh;
      const float w = (h < H && k < kSensors) ? __ldg(W1 + (size_t)k * hp + h) : 0.0f;
      put_split(B1hi, B1lo, tc::canon_off(h, k, nh), w);
    }
    const float* W2 = a.net.wB + (size_t)slot * hp * kOutPad;  // W2^T [hp][16]
    for (int i = tid; i < 16 * nh; i += kNetThreads) {
      const int j = i & 15, h = i >> 4;
      const float w = (h < H && j < kActuators) ? __ldg(W2 + (size_t)h * kOutPad + j) : 0.0f;
      float wh, wl;
      split_fast(w, wh, wl);
      *reinterpret_cast<float*>(B2 + tc::canon_off(j, h, 32)) = wh;
      *reinterpret_cast<float*>(B2 + tc::canon_off(16 + j, h, 32)) = wl;
    }
    for (int h = tid; h < nh; h += kNetThreads) b1[h] = h < H ? __ldg(a.net.bA + (size_t)slot * hp + h) : 0.0f;
    if (tid < 16) b2[tid] = tid < kActuators ? __ldg(a.net.bB + (size_t)slot * kOutPad + tid) : 0.0f;
  };
  // warp 0 issues (uniform control flow, one elected lane per MMA)
  auto issue_l1 = [&](int buf) {
    if (warp == 0) {
      const uint32_t lA = kRows * 16, lB = nh * 16;
      const uint64_t ah = tc::smem_desc(tc::smem_u32(A1 + buf * 2 * kA1Bytes), lA, 128);
      const uint64_t al = tc::smem_desc(tc::smem_u32(A1 + buf * 2 * kA1Bytes + kA1Bytes), lA, 128);
      const uint64_t bh = tc::smem_desc(tc::smem_u32(B1hi), lB, 128);
      const uint64_t bl = tc::smem_desc(tc::smem_u32(B1lo), lB, 128);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int acc = 0; acc < 2; ++acc) {
          const int ks = acc * 3 + j;
          const uint64_t oa = (uint64_t)((2 * ks * lA) >> 4), ob = (uint64_t)((2 * ks * lB) >> 4);
          const uint32_t d = tmem + (acc ? (uint32_t)nh : 0u);
          mma_ss_e(d, al + oa, bh + ob, id1, j > 0);
          mma_ss_e(d, ah + oa, bl + ob, id1, 1u);
          mma_ss_e(d, ah + oa, bh + ob, id1, 1u);
        }
      commit_e(&bar[0]);
    }
  };
  auto issue_l2 = [&]() {
    if (warp == 0) {
      const uint32_t lB = 32 * 16;
      const uint64_t bd = tc::smem_desc(tc::smem_u32(B2), lB, 128);
      const int nks = nh / 8, quarter = nks / kL2Acc;  // nh is a multiple of 32 here
      for (int ks = 0; ks < nks; ++ks) {
        const uint32_t d = tmem + kL2 + 32u * (uint32_t)(ks / quarter);
        const uint64_t b = bd + (uint64_t)((2 * ks * lB) >> 4);
        mma_ts(d, tmem + (uint32_t)(8 * ks), b, id2, (uint32_t)(ks % quarter != 0));
        mma_ts(d, tmem + (uint32_t)(nh + 8 * ks), b, id2, 1u);
      }
      commit_e(&bar[1]);
    }
  };
  auto sync_tc = [&]() {
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  };

  const int4 z4 = make_int4(0, 0, 0, 0);
  int u1 = next_tile(t), u2 = next_tile(u1);
  int4 ti0 = __ldg(a.tile_info + t);
  int4 ti1 = u1 < T ? __ldg(a.tile_info + u1) : z4;
  int4 ti2 = u2 < T ? __ldg(a.tile_info + u2) : z4;
  int cur = ti0.x;
  fetch(ti0);
  if (GATHER) {
    if (tid == 0) fetch_weights(cur, 0);
    wait_weights();
  } else {
    stage_weights(cur);
  }
  stage_a1(0);
  if (u1 < T) fetch(ti1);
  tc::fence_async_smem();
  sync_tc();
  issue_l1(0);
  const int q = warp & 3, qt = warp >> 2;
  const int r = q * 32 + lane;  // this thread's tile row (TMEM lane)
  const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16);
  const int c_begin = qt * (nh / 4), c_end = c_begin + nh / 4;
  int buf = 0;
  while (t < T) {
    const int4 ti = ti0;
    const bool has_next = u1 < T;
    const int next_slot = has_next ? ti1.x : cur;
    // (a) the next tile's rows into the other A1 buffer (its layer 1 reads
    //     it after this tile's layer 2), the one after into registers
    if (has_next) stage_a1(buf ^ 1);
    if (u2 < T) fetch(ti2);
    const int u3 = next_tile(u2);
    ti0 = ti1;
    ti1 = ti2;
    ti2 = u3 < T ? __ldg(a.tile_info + u3) : z4;
    // (b) epilogue 1: h = tanh(acc0 + acc1 + b1) over this thread's quarter,
    //     written back split over the columns it read
    tc::mbar_wait(&bar[0], ph0);
    ph0 ^= 1u;
    tc::fence_after();
    for (int c0 = c_begin; c0 < c_end; c0 += 4) {
      uint32_t va[4], vb[4];
      tc::tmem_ld4_nw(lb + c0, va);
      tc::tmem_ld4_nw(lb + nh + c0, vb);
      tc::tmem_wait_ld();
      tc::reg_fence(va);
      tc::reg_fence(vb);
      uint32_t hh[4], hl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float h = tanh_sfu(__fadd_rn(__fadd_rn(__uint_as_float(va[j]), __uint_as_float(vb[j])), b1[c0 + j]));
        float x, y;
        split_fast(h, x, y);
        hh[j] = __float_as_uint(x);
        hl[j] = __float_as_uint(y);
      }
      tmem_st4(lb + c0, hh[0], hh[1], hh[2], hh[3]);
      tmem_st4(lb + nh + c0, hl[0], hl[1], hl[2], hl[3]);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc::fence_async_smem();  // the next A1 buffer staged in (a)
    sync_tc();
    // (c) layer 2 of this tile; gather form: the next slot's table into the
    //     other weight buffer (every reader of it has passed the barrier)
    issue_l2();
    if (GATHER && has_next && next_slot != cur && tid == 0) fetch_weights(next_slot, wb ^ 1);
    // (d) layer 2 has read h once it completes: the next tile's layer 1
    tc::mbar_wait(&bar[1], ph1);
    ph1 ^= 1u;
    tc::fence_after();
    float bias2[kActuators];  // this tile's b2, read before a restage replaces it
#pragma unroll
    for (int j = 0; j < kActuators; ++j) bias2[j] = b2[j];
    if (has_next && next_slot != cur) {  // genome change
      if (GATHER) {  // the bulk copy issued in (c)
        wait_weights();
        cur = next_slot;
        use_weights(wb ^ 1);
      } else {  // restage every table first
        sync_tc();
        cur = next_slot;
        stage_weights(cur);
        tc::fence_async_smem();
        sync_tc();
      }
    }
    if (has_next) issue_l1(buf ^ 1);
    // (e) epilogue 2 (one warp per lane quadrant) overlapping that layer 1
    if (qt == 0) {
      float zs[kActuators];
#pragma unroll
      for (int i = 0; i < kL2Acc; ++i) {
        uint32_t dh[16], dl[16];
        tc::tmem_ld16_nw(lb + kL2 + 32 * i, dh);
        tc::tmem_ld16_nw(lb + kL2 + 32 * i + 16, dl);
        tc::tmem_wait_ld();
        tc::reg_fence(dh);
        tc::reg_fence(dl);
#pragma unroll
        for (int j = 0; j < kActuators; ++j) {
          const float p = __fadd_rn(__uint_as_float(dh[j]), __uint_as_float(dl[j]));
          zs[j] = i ? __fadd_rn(zs[j], p) : p;
        }
      }
      if (r < ti.z) {
        // the row at the cell index (the physics then reads it coalesced):
        // the gather form's list entry, or element 45 of the sensor row (its
        // cell index, k_hid_sense)
        const size_t row = GATHER ? (size_t)gs::gcell(__ldg(a.sorted + ti.y + r), a.W).cell
                                  : (size_t)__float_as_int(__ldg(a.sens + (size_t)(ti.y + r) * kK1 + 45));
        if (a.decided) {
          // 32-byte decided record {inv, liq, m0..m2, xmax, kstar, 0}: five
          // sigmoids and explore_pick (exact) instead of thirteen sigmoids
          float z[kActuators];
#pragma unroll
          for (int j = 0; j < kActuators; ++j) z[j] = __fadd_rn(zs[j], bias2[j]);
          int ks;
          float xm;
          explore_pick(z + 5, ks, xm);
          asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a.act + row * 8),
                       "f"(squash(z[0])), "f"(squash(z[1])), "f"(squash(z[2])), "f"(squash(z[3])), "f"(squash(z[4])),
                       "f"(xm), "f"(__int_as_float(ks)), "f"(0.0f)
                       : "memory");
        } else {
          float o[16];
#pragma unroll
          for (int j = 0; j < kActuators; ++j) o[j] = squash(__fadd_rn(zs[j], bias2[j]));
          o[13] = o[14] = o[15] = 0.0f;
          float4* dst = reinterpret_cast<float4*>(a.act + row * 16);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        }
      }
      tc::fence_before();  // the layer-2 columns are read before the next layer 2 (after the next epilogue 1's barrier)
    }
    t = u1;
    u1 = u2;
    u2 = u3;
    buf ^= 1;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTmemCols>(tmem);
}

// Direct 45->13 controller over genome-sorted sensor rows (many-genome
// pools, e.g. BASELINE configs 3-4 with 256-1024 genomes, where a 32x32 tile
// holds ~1-4 cells per genome and per-tile weight fetches dominate).  Each
// WARP takes contiguous 64-row half-tiles (one genome each): the genome's
// 2.4 KB of weights are staged in a warp-private shared buffer once per run
// of half-tiles (every weight load a warp-uniform broadcast); each lane
// streams its two 192-byte rows straight from global memory into registers,
// kDrDepth whole 32-byte sectors per row in flight (LDG.256; no shared-memory staging, so
// 16 warps fit per SM instead of the 8 that double-buffered 53 KB row tiles
// allowed), and runs the same packed FFMA2 chains, pairing and k order as the
// tile kernel (net_direct_unit), so results are bit-identical to it.
constexpr int kDrWarps = 4;
constexpr int kDrThreads = kDrWarps * 32;
constexpr int kDrDepth = 3;     // 32-byte chunks (whole sectors) per row in flight
constexpr int kDrW = kSensors * 12 + 48 + kOutPad;  // W12 [45][12] | W1 [48] | bias [16]

struct f8 {
  float v[8];
};
// one whole 32-byte sector per lane (LDG.256)
__device__ __forceinline__ f8 ld_row32(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                 "=f"(r.v[7])
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(kDrThreads, 4) k_direct_rows(const NetArgs a) {
  __shared__ __align__(16) float wsm[kDrWarps][kDrW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* W12 = wsm[warp];
  float* W1 = W12 + kSensors * 12;
  float* Bs = W1 + 48;
  const int H = 2 * *a.n_tiles;  // 64-row half-tiles
  const int nw = gridDim.x * kDrWarps, gw = blockIdx.x * kDrWarps + warp;
  const int per = (H + nw - 1) / nw;
  const int h0 = gw * per, h1 = min(H, h0 + per);
  // next non-empty half-tile at or after h (empty second halves of short
  // tiles are skipped; warp-uniform)
  auto advance = [&](int h, int4& ti) {
    for (; h < h1; ++h) {
      ti = __ldg(a.tile_info + (h >> 1));
      if ((h & 1) * 64 < ti.z) break;
    }
    return h;
  };
  auto row_ptr = [&](const int4& ti, int h, int r) {
    const int rr = (h & 1) * 64 + r;
    return a.sens + (size_t)(ti.y + (rr < ti.z ? rr : 0)) * kK1;
  };
  int cur = -1;
  int4 ti = make_int4(0, 0, 0, 0);
  int h = advance(h0, ti);
  f8 q0[6], q1[6];
  if (h < h1) {  // the first half-tile's leading sectors; later ones are
                 // issued during the previous half-tile's last chunks
    const float* g0 = row_ptr(ti, h, lane);
    const float* g1 = row_ptr(ti, h, lane + 32);
#pragma unroll
    for (int c = 0; c < kDrDepth; ++c) {
      q0[c] = ld_row32(g0 + 8 * c);
      q1[c] = ld_row32(g1 + 8 * c);
    }
  }
  while (h < h1) {
    int4 tn = ti;
    const int hn = advance(h + 1, tn);
    if (ti.x != cur) {
      cur = ti.x;
      __syncwarp();
      const float4* w12 = reinterpret_cast<const float4*>(a.net.wA + (size_t)cur * kSensors * 12);
      for (int i = lane; i < kSensors * 3; i += 32) reinterpret_cast<float4*>(W12)[i] = __ldg(w12 + i);
      for (int i = lane; i < kSensors; i += 32) W1[i] = __ldg(a.net.wB + (size_t)cur * kSensors + i);
      if (lane < kOutPad) Bs[lane] = __ldg(a.net.bA + (size_t)cur * kOutPad + lane);
      __syncwarp();
    }
    const int rb = (h & 1) * 64;
    const int r0 = rb + lane, r1 = rb + lane + 32;
    const float* g0 = row_ptr(ti, h, lane);
    const float* g1 = row_ptr(ti, h, lane + 32);
    const bool more = hn < h1;
    const float* n0 = row_ptr(tn, hn, lane);
    const float* n1 = row_ptr(tn, hn, lane + 32);
    u64 acc[2][6];
    float acc12[2] = {0.0f, 0.0f};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int p = 0; p < 6; ++p) acc[c][p] = 0ull;
#pragma unroll
    for (int k = 0; k < kSensors; ++k) {
      const int ch = k >> 3, j = k & 7;
      if (j == 0 && ch + kDrDepth < 6) {  // refill the sector pipeline
        q0[ch + kDrDepth] = ld_row32(g0 + 8 * (ch + kDrDepth));
        q1[ch + kDrDepth] = ld_row32(g1 + 8 * (ch + kDrDepth));
      }
      if (j == 0 && ch >= 6 - kDrDepth && more) {  // the next half-tile's leading sectors
        q0[ch - (6 - kDrDepth)] = ld_row32(n0 + 8 * (ch - (6 - kDrDepth)));
        q1[ch - (6 - kDrDepth)] = ld_row32(n1 + 8 * (ch - (6 - kDrDepth)));
      }
      const float x0 = q0[ch].v[j];
      const float x1 = q1[ch].v[j];
      const float4* w4 = reinterpret_cast<const float4*>(W12 + k * 12);
      const float4 wa = w4[0], wb = w4[1], wc = w4[2];
      const u64 wp[6] = {pk2(wa.x, wa.y), pk2(wa.z, wa.w), pk2(wb.x, wb.y),
                         pk2(wb.z, wb.w), pk2(wc.x, wc.y), pk2(wc.z, wc.w)};
      const float w12 = W1[k];
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        ffma2(acc[0][p], x0, wp[p]);
        ffma2(acc[1][p], x1, wp[p]);
      }
      acc12[0] = fmaf(x0, w12, acc12[0]);
      acc12[1] = fmaf(x1, w12, acc12[1]);
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int r = c ? r1 : r0;
      if (r >= ti.z) continue;
      float z[13];
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        float lo, hi;
        up2(acc[c][p], lo, hi);
        z[2 * p] = __fadd_rn(lo, Bs[2 * p]);
        z[2 * p + 1] = __fadd_rn(hi, Bs[2 * p + 1]);
      }
      z[12] = __fadd_rn(acc12[c], Bs[12]);
      if (a.decided) {  // 32 bytes at the cell's index: the physics needs only these (explore_pick is exact)
        int ks;
        float xm;
        explore_pick(z + 5, ks, xm);
        const int cell = __float_as_int(c ? q1[5].v[5] : q0[5].v[5]);  // row element 45
        // one whole-sector store per record (STG.256): scattered cells, so
        // every store instruction is 32 sectors and their count is the cost
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a.act + (size_t)cell * 8),
                     "f"(squash(z[0])), "f"(squash(z[1])), "f"(squash(z[2])), "f"(squash(z[3])), "f"(squash(z[4])),
                     "f"(xm), "f"(__int_as_float(ks)), "f"(0.0f)
                     : "memory");
      } else {
        float v[16];
#pragma unroll
        for (int j = 0; j < 13; ++j) v[j] = squash(z[j]);
        v[13] = v[14] = v[15] = 0.0f;
        float4* dst = reinterpret_cast<float4*>(a.act + (size_t)(ti.y + r) * 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
    h = hn;
    ti = tn;
  }
}



}  // namespace

cudaError_t debug_hidden_cycles(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_hid_cycles, sizeof(unsigned long long) * 8);
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_hid_cycles, z, sizeof(z));
  }
  return e;
}

int hidden_sort_ctas(int W, int H) {
  const int ntiles = ((W + kST - 1) / kST) * ((H + kST - 1) / kST);
  return (ntiles + kSortTiles - 1) / kSortTiles;
}

int hidden_tc_nh(int hidden) { return ((hidden + 15) / 16) * 16; }

bool hidden_tc_supported(int hidden) { return hidden >= 1 && hidden_tc_nh(hidden) <= 128; }

size_t hidden_tc_smem(int hidden) {
  const int nh = hidden_tc_nh(hidden);
  const size_t fixed = (size_t)2 * nh * kK1 * 4 + (size_t)16 * nh * 4 + (size_t)(nh + 16) * 4 + (size_t)kRows * kXPitch * 4;
  return ((fixed + 1023) & ~(size_t)1023) + (size_t)4 * kRows * kK1 * 4 + 1024;  // + alignment slack
}

bool hidden_gather_supported(int hidden) {
  const int nh = hidden_tc_nh(hidden);
  return hidden >= 1 && nh <= 128 && nh % 32 == 0;
}

size_t hidden_table_bytes(int hidden) { return (size_t)hid_table_bytes(hidden_tc_nh(hidden)); }

cudaError_t launch_hidden_tables(const Params& net, int cap, unsigned char* out, cudaStream_t st) {
  k_hid_tables<<<cap, 256, 0, st>>>(net, hidden_tc_nh(net.hidden), out);
  return cudaGetLastError();
}

cudaError_t launch_hidden_gather(const GatherBuffers& b, const StepGeom& g, const Params& net, int cap, int num_sms,
                                 const unsigned char* htab, float* act, cudaStream_t st) {
  NetArgs a{};
  a.net = net;
  a.nh = hidden_tc_nh(net.hidden);
  a.n_tiles = b.n_ht;
  a.tile_info = b.info;
  a.cap = cap;
  a.act = act;
  a.sorted = b.sorted;
  a.tex = b.tex;
  a.W = g.W;
  a.contig = 0;
  a.htab = htab;
  // weights | A1 x 4 | second weights (the static 1 KB holds the barriers:
  // 230,976 + 1,024 of the 232,448 bytes a CTA may have at nh = 128)
  const int nh = hidden_tc_nh(net.hidden), tb = hid_table_bytes(nh);
  const size_t smem = (size_t)((tb + 1023) & ~1023) + (size_t)4 * kRows * kK1 * 4 + (size_t)tb;
  cudaError_t e = cudaFuncSetAttribute(k_hid_net2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_hid_net2<true><<<num_sms, kNetThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// k_hid_net2 (both layers on the tensor core) serves this width; with
// `decided` it leaves 32-byte decided records at the cell index
bool hidden_net2_used(int hidden, bool l2_cuda_core) {
  return hidden > 0 && !l2_cuda_core && hidden_tc_nh(hidden) <= 128 && hidden_tc_nh(hidden) % 32 == 0;
}

cudaError_t launch_hidden_tc(const HidBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                             int capacity, int num_sms, bool decided, bool l2_cuda_core, cudaStream_t st) {
  const int nctas = hidden_sort_ctas(g.W, g.H);
  const size_t hsmem = (size_t)capacity * 4;
  const size_t ssmem = sense_smem_bytes(capacity);
  cudaError_t e = cudaSuccess;
  if (hsmem > 48 * 1024) {
    e = cudaFuncSetAttribute(k_hid_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    if (e != cudaSuccess) return e;
  }
  if (ssmem > 48 * 1024) {
    e = cudaFuncSetAttribute(k_hid_sense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem);
    if (e != cudaSuccess) return e;
  }
  k_hid_count<<<nctas, kSortThreads, hsmem, st>>>(g, front.gi, capacity, b.cta_hist);
  k_hid_colscan<<<(capacity + 31) / 32, 1024, 0, st>>>(b.cta_hist, nctas, capacity, b.counts);
  k_hid_scan<<<1, 1024, 0, st>>>(b.counts, capacity, b.offs, b.tiles, b.cursor, b.n_tiles);
  {
    const long long max_tiles = ((long long)g.W * g.H + kRows - 1) / kRows + capacity;
    k_hid_tilemap<<<(unsigned)((max_tiles + 255) / 256), 256, 0, st>>>(b.offs, b.tiles, capacity, b.n_tiles,
                                                                       b.tile_info);
  }
  // decided records of direct nets land at the cell index: no cell -> row map
  int32_t* rank = decided && net.hidden == 0 ? nullptr : b.rank;
  const bool net2 = hidden_net2_used(net.hidden, l2_cuda_core);
  k_hid_sense<<<nctas, kSortThreads, ssmem, st>>>(g, front, b.offs, b.cta_hist, capacity, b.sens, rank, net2 ? 1 : 0);
  NetArgs a;
  a.net = net;
  a.nh = net.hidden > 0 ? hidden_tc_nh(net.hidden) : 0;
  a.offs = b.offs;
  a.tiles = b.tiles;
  a.n_tiles = b.n_tiles;
  a.cap = capacity;
  a.sens = b.sens;
  a.tile_info = b.tile_info;
  a.act = b.act;
  a.decided = decided && (net.hidden == 0 || net2) ? 1 : 0;
  if (net.hidden == 0) {
    k_direct_rows<<<num_sms * 4, kDrThreads, 0, st>>>(a);  // 16 warps per SM, one wave
    return cudaGetLastError();
  }
  if (net2) {
    const size_t smem = hidden_tc2_smem(net.hidden);
    e = cudaFuncSetAttribute(k_hid_net2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_hid_net2<false><<<num_sms, kNetThreads, smem, st>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = hidden_tc_smem(net.hidden);
  e = cudaFuncSetAttribute(k_hid_net, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_hid_net<<<num_sms, kNetThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace evo
