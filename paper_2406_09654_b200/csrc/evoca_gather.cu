// Direct 45 -> 13 controller for large pools without sensor rows (BASELINE
// configs 3-4: 256-1024 genomes drawn uniformly per cell, so a 32x32 tile
// holds 1-4 cells per genome and no genome's 2.4 KB of weights is reused
// inside a tile).  Reference: sense engine.py:164-190, forward
// hypernet.py:233-252 with the hidden layer removed (BASELINE direct net).
//
// The round-1/2 rows path (evoca_hidden_tc.cu: k_hid_sense -> k_direct_rows)
// wrote a 192-byte sensor row per cell to HBM and read it back (9.5 GB per
// config-3 step).  Here nothing per-cell but a 4-byte sorted cell list leaves
// the chip between sense and net:
//   k_gs_count    per count CTA (a run of rows): the 32-byte sense texture
//                 record of every cell {E, I, C0, C1, C2, 0, 0, 0} (one
//                 sector), the CTA's histogram of occupied cells by slot and
//                 each cell's rank in it (one shared-memory atomic per cell)
//   k_gs_colscan / k_gs_scan_band / k_gs_scan_bands  per row band (~1 M
//                 cells, so the band's texture stays in the 126 MB L2):
//                 CTA bases inside each (band, slot) group, group offsets,
//                 band bases
//   k_gs_scatter  cell list sorted by (band, slot): positions from the
//                 scans and ranks, no atomics
//   k_gs_tilemap  64-cell half-tiles of one (band, slot) group
//   k_direct_gather  one warp per half-tile: the slot is uniform, so every
//                 weight load is a warp-uniform broadcast; each lane gathers
//                 its two cells' nine texture records in their own Moore
//                 order (PERM_TABLE[rot], physics.py:48-62; whole 32-byte
//                 sectors, L2 hits: half-tiles are handed out band by band)
//                 and runs the tile kernel's FFMA2 chains in the same k
//                 order, so the actions are bit-identical to the tile and
//                 rows paths.  Output: the 32-byte decided record at the
//                 cell index (k_physics_rows), or 16-float actuator rows at
//                 the cell index (export).

#include <algorithm>
#include <cstdlib>

#include "evoca_gather.cuh"
#include "evoca_net.cuh"
#include "evoca_tc.cuh"

namespace evo {

namespace {

using namespace gs;

constexpr int kGsThreads = 512;  // count / scatter CTA
// GsPlan.rb: bins per slot (8 = one per rotation for the FFMA warp kernel,
// whose Moore order must be warp-uniform; 1 for the tensor-core kernel,
// which gathers each row in its own order); GsPlan.tile: cells per tile
// (64 = one warp, 128 = one MMA M).
constexpr int kGsBandCells = 1 << 20;
// EVO_BAND_CELLS overrides the band size (tuning runs)
static long long band_cells_default() {
  static const long long v = [] {
    const char* e = std::getenv("EVO_BAND_CELLS");
    const long long x = e ? std::atoll(e) : 0;
    return x >= 4096 ? x : (long long)kGsBandCells;
  }();
  return v;
}

struct GsPlan {
  int rows_per_cta, ctas_per_band, nctas, nbands, bins, rb, tile;
};
__device__ __forceinline__ int gs_bin(const GsPlan& p, int s, int r) { return s * p.rb + (r & (p.rb - 1)); }

__device__ __forceinline__ void st_rec(float* p, float e, float i, float c0, float c1, float c2) {
  // (no "memory" clobber: nothing in the writing kernel reads the texture,
  //  and the clobber would pin every later load behind the store)
  asm volatile("st.global.v8.f32 [%0], {%1,%3,%4,%5,%2,%6,%6,%6};" ::"l"(p), "f"(e), "f"(i), "f"(c0), "f"(c1),
               "f"(c2), "f"(0.0f));  // {E, C0, C1, C2 | I, 0, 0, 0}: tex_ch()
}

// Pass-1 record of the fused step (FusedPhysics, evoca_internal.h):
// {E', C0', C1', C2' | I', q, genome, proposal byte}, one sector at the cell index.
__device__ __forceinline__ void st_mid(float* p, const CellOut& o) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(o.e), "f"(o.c0), "f"(o.c1),
               "f"(o.c2), "f"(o.inf), "f"(o.q), "f"(__int_as_float(o.slot)), "f"(__int_as_float((int)o.rp))
               : "memory");
}

// Texture records of the CTA's rows (plus ghost row -1 / H on the first /
// last CTA) and the band histogram by (slot, rotation).  Slots outside
// [0, cap) are left out (no out-of-bounds shared-memory write); the step's
// range check reports them.  Widths divisible by 4 move four cells per
// thread and iteration with 16-byte plane loads.
__device__ __forceinline__ void count_cell(const GsPlan& p, int* hist, int cap, int s, int r, int32_t* rank,
                                           uint16_t* lrank, long long i, bool in) {
  if (!in) return;
  const bool occ = (unsigned)s < (unsigned)cap;
  if (occ) lrank[i] = (uint16_t)atomicAdd(&hist[gs_bin(p, s, r)], 1);  // rank inside the CTA's group
  if (rank) rank[i] = occ ? (int)i : -1;
}

__global__ void __launch_bounds__(kGsThreads) k_gs_count(const StepGeom g, const Planes f, const GsPlan p, int cap,
                                                          int32_t* cta_hist, uint16_t* lrank, float* tex,
                                                          int32_t* rank) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * p.rows_per_cta, r1 = min(g.H, r0 + p.rows_per_cta);
  const long long W = g.W, st = g.stride;
  // the records cover the ghost rows too (first / last CTA)
  const long long lo = (blockIdx.x == 0 ? -1 : r0) * W, hi = (r1 == g.H ? g.H + 1 : r1) * W;
  const long long c0 = (long long)r0 * W, c1 = (long long)r1 * W;
  if ((g.W & 3) == 0) {
    for (long long i = lo + 4 * threadIdx.x; i < hi; i += 4 * blockDim.x) {
      const long long o = i + W;  // element offset from ghost row -1
      const bool in = i >= c0 && i < c1;
      int4 G = make_int4(-1, -1, -1, -1);
      unsigned R = 0;
      if (in) {
        G = __ldg(reinterpret_cast<const int4*>(f.gi + o));
        R = __ldg(reinterpret_cast<const unsigned*>(f.rot + o));
      }
        const float4 E = __ldg(reinterpret_cast<const float4*>(f.E + o));
        const float4 I = __ldg(reinterpret_cast<const float4*>(f.I + o));
        const float4 C0 = __ldg(reinterpret_cast<const float4*>(f.C + o));
        const float4 C1 = __ldg(reinterpret_cast<const float4*>(f.C + st + o));
        const float4 C2 = __ldg(reinterpret_cast<const float4*>(f.C + 2 * st + o));
        float* t = tex + o * 8;
        st_rec(t, E.x, I.x, C0.x, C1.x, C2.x);
        st_rec(t + 8, E.y, I.y, C0.y, C1.y, C2.y);
        st_rec(t + 16, E.z, I.z, C0.z, C1.z, C2.z);
        st_rec(t + 24, E.w, I.w, C0.w, C1.w, C2.w);
      count_cell(p, hist, cap, G.x, (int)(R & 0xFFu), rank, lrank, i, in);
      count_cell(p, hist, cap, G.y, (int)((R >> 8) & 0xFFu), rank, lrank, i + 1, in);
      count_cell(p, hist, cap, G.z, (int)((R >> 16) & 0xFFu), rank, lrank, i + 2, in);
      count_cell(p, hist, cap, G.w, (int)(R >> 24), rank, lrank, i + 3, in);
    }
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const long long o = i + W;
        st_rec(tex + o * 8, __ldg(f.E + o), __ldg(f.I + o), __ldg(f.C + o), __ldg(f.C + st + o),
               __ldg(f.C + 2 * st + o));
      const bool in = i >= c0 && i < c1;
      count_cell(p, hist, cap, in ? __ldg(f.gi + o) : -1, in ? __ldg(f.rot + o) : 0, rank, lrank, i, in);
    }
  }
  __syncthreads();
  int32_t* out = cta_hist + (size_t)blockIdx.x * p.bins;
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) out[b] = hist[b];
}

// Slot ranks alone, for a fused step whose texture already holds the state
// (written by the previous step's pass 2, FusedPhysics): the genome plane is
// all that is read; an unoccupied cell's pass-1 record comes from its texture
// record.  W % 4 == 0 (the fused step needs the TMA maps anyway).
__global__ void __launch_bounds__(kGsThreads) k_gs_rank(const StepGeom g, const int32_t* gi, const GsPlan p, int cap,
                                                         int32_t* cta_hist, uint16_t* lrank, const float* tex,
                                                         const FusedPhysics fp, float* mid_rec) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * p.rows_per_cta, r1 = min(g.H, r0 + p.rows_per_cta);
  const long long W = g.W, c0 = (long long)r0 * W, c1 = (long long)r1 * W;
  for (long long i = c0 + 4 * threadIdx.x; i < c1; i += 4 * blockDim.x) {
    const int4 G = __ldg(reinterpret_cast<const int4*>(gi + i + W));
    const int sl[4] = {G.x, G.y, G.z, G.w};
    uint16_t rk[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((unsigned)sl[j] < (unsigned)cap) {
        rk[j] = (uint16_t)atomicAdd(&hist[gs_bin(p, sl[j], 0)], 1);
      } else {
        const f8r r = ld_rec(tex + (size_t)(i + j + W) * 8);
        const CellState cs{r.v[tex_ch(0)], r.v[tex_ch(1)], r.v[tex_ch(2)], r.v[tex_ch(3)], r.v[tex_ch(4)], -1, 0};
        st_mid(mid_rec + (size_t)(i + j) * 8, cell_physics(fp.s, fp.phases, fp.src_map, i + j, cs, CellAct{}));
      }
    }
    *reinterpret_cast<uint2*>(lrank + i) = make_uint2(rk[0] | ((unsigned)rk[1] << 16), rk[2] | ((unsigned)rk[3] << 16));
  }
  __syncthreads();
  int32_t* out = cta_hist + (size_t)blockIdx.x * p.bins;
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) out[b] = hist[b];
}

// Front E, I, C planes (ghost rows included) from the texture, when a lazy
// fused step left the state there (evoca_abi.cu: materialize).
__global__ void __launch_bounds__(256) k_tex_to_planes(const StepGeom g, const float* tex, const Planes f) {
  const long long n = (long long)(g.H + 2) * g.W, st = g.stride;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < n; o += (long long)gridDim.x * blockDim.x) {
    const f8r r = ld_rec(tex + (size_t)o * 8);
    f.E[o] = r.v[tex_ch(0)];
    f.I[o] = r.v[tex_ch(1)];
    f.C[o] = r.v[tex_ch(2)];
    f.C[st + o] = r.v[tex_ch(3)];
    f.C[2 * st + o] = r.v[tex_ch(4)];
  }
}

// per band and bin: exclusive scan of the per-CTA counts over the band's CTAs
// (in place: each CTA's base inside its group) and the band's group totals.
// One CTA per (band, 32 bins): lane = bin (coalesced), warp w a contiguous
// chunk of the band's CTAs; chunk sums scanned across warps in shared memory.
__global__ void __launch_bounds__(1024) k_gs_colscan(const GsPlan p, int32_t* cta_hist, int32_t* band_hist) {
  __shared__ int part[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb32 = (p.bins + 31) / 32, band = blockIdx.x / nb32, b = (blockIdx.x % nb32) * 32 + lane;
  const int cb = band * p.ctas_per_band, ce = min(p.nctas, cb + p.ctas_per_band);
  const int per = (ce - cb + 31) / 32, c0 = cb + w * per, c1 = min(ce, c0 + per);
  int sum = 0;
  if (b < p.bins)
    for (int c = c0; c < c1; ++c) sum += cta_hist[(size_t)c * p.bins + b];
  part[w][lane] = sum;
  __syncthreads();
  if (w == 0) {
    int run = 0;
    for (int k = 0; k < 32; ++k) {
      const int v = part[k][lane];
      part[k][lane] = run;
      run += v;
    }
    if (b < p.bins) band_hist[(size_t)band * p.bins + b] = run;
  }
  __syncthreads();
  int run = part[w][lane];
  if (b < p.bins)
    for (int c = c0; c < c1; ++c) {
      int32_t* q = cta_hist + (size_t)c * p.bins + b;
      const int v = *q;
      *q = run;
      run += v;
    }
}

// The same texture build and slot ranking through TMA (the default when the
// step covers the whole strip): per CTA a two-stage pipeline over 256-cell
// row chunks - thread 0 issues the chunk's six plane boxes (E, I, C0, C1, C2,
// genome; cp.async.bulk.tensor, mbarrier complete_tx) one chunk ahead, every
// thread turns its cell into a record in shared memory and ranks it, and
// thread 0 writes the chunk's 256 records back with one TMA store.
constexpr int kTmThreads = 256;
constexpr int kTmChunk = 256;  // cells per box (one row)

struct __align__(128) TmStage {
  float pl[5][kTmChunk];
  int32_t gi[kTmChunk];
  float rec[kTmChunk * 8];
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"((uint64_t)m), "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, const void* src, int c, int x, int y) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"((uint64_t)m),
               "r"(c), "r"(x), "r"(y), "r"((uint32_t)__cvta_generic_to_shared(src))
               : "memory");
}

__global__ void __launch_bounds__(kTmThreads) k_gs_count_tma(const StepGeom g, const __grid_constant__ GatherMaps maps,
                                                            const GsPlan p, int cap, int32_t* cta_hist,
                                                            uint16_t* lrank, int32_t* rank,
                                                            const FusedPhysics fp, float* mid_rec) {
  extern __shared__ __align__(128) unsigned char dsm[];
  TmStage* stg = reinterpret_cast<TmStage*>(dsm);  // 2 stages
  int* hist = reinterpret_cast<int*>(dsm + 2 * sizeof(TmStage));
  __shared__ __align__(8) uint64_t full[2];
  const int tid = threadIdx.x;
  for (int b = tid; b < p.bins; b += kTmThreads) hist[b] = 0;
  const int r0 = blockIdx.x * p.rows_per_cta, r1 = min(g.H, r0 + p.rows_per_cta);
  // tensor rows (0 = ghost row -1): this CTA's rows, plus the ghost rows on
  // the first / last CTA (records only)
  const int y_lo = blockIdx.x == 0 ? 0 : r0 + 1, y_hi = r1 == g.H ? g.H + 2 : r1 + 1;
  const int per_row = (g.W + kTmChunk - 1) / kTmChunk;
  const int nchunks = (y_hi - y_lo) * per_row;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int c) {  // thread 0: chunk c's six boxes into stage c & 1
    TmStage& s = stg[c & 1];
    const int ty = y_lo + c / per_row, x0 = (c % per_row) * kTmChunk;
    uint64_t* bar = &full[c & 1];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(6 * kTmChunk * 4)
                 : "memory");
#pragma unroll
    for (int k = 0; k < 5; ++k) tma_load_2d(s.pl[k], &maps.plane[k], x0, ty, bar);
    tma_load_2d(s.gi, &maps.plane[5], x0, ty, bar);
  };
  if (tid == 0 && nchunks > 0) issue(0);
  uint32_t ph[2] = {0u, 0u};
  for (int c = 0; c < nchunks; ++c) {
    const int sb = c & 1;
    TmStage& s = stg[sb];
    if (tid == 0 && c + 1 < nchunks) issue(c + 1);  // its stage was read before the last barrier
    {
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&full[sb]);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(b), "r"(ph[sb])
            : "memory");
      ph[sb] ^= 1u;
    }
    const int ty = y_lo + c / per_row, x = (c % per_row) * kTmChunk + tid;
    // the record (two 16-byte halves; lanes 32 bytes apart)
    float4* rp = reinterpret_cast<float4*>(s.rec + tid * 8);
    rp[0] = make_float4(s.pl[0][tid], s.pl[2][tid], s.pl[3][tid], s.pl[4][tid]);  // {E, C0, C1, C2 | I, 0, 0, 0}
    rp[1] = make_float4(s.pl[1][tid], 0.0f, 0.0f, 0.0f);
    const int y = ty - 1;  // strip row
    if (x < g.W && y >= r0 && y < r1) {
      const long long i = (long long)y * g.W + x;
      const int sl = s.gi[tid];
      const bool occ = (unsigned)sl < (unsigned)cap;
      if (occ) lrank[i] = (uint16_t)atomicAdd(&hist[gs_bin(p, sl, 0)], 1);
      if (rank) rank[i] = occ ? (int)i : -1;
      if (mid_rec && !occ) {  // fused step: the net never sees an unoccupied cell, its physics runs here
        const CellState cs{s.pl[0][tid], s.pl[1][tid], s.pl[2][tid], s.pl[3][tid], s.pl[4][tid], -1, 0};
        st_mid(mid_rec + i * 8, cell_physics(fp.s, fp.phases, fp.src_map, i, cs, CellAct{}));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tma_store_3d(&maps.tex, s.rec, 0, (c % per_row) * kTmChunk, ty);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the store issued one chunk ago has read its stage: that stage's
      // record buffer is written again by the next chunk
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncthreads();
  int32_t* out = cta_hist + (size_t)blockIdx.x * p.bins;
  for (int b = tid; b < p.bins; b += kTmThreads) out[b] = hist[b];
}

// Block-wide exclusive scan of (cells, half-tiles) pairs, 1024 threads.
__device__ __forceinline__ void scan_pair(int c, int t, int& xc, int& xt, int& tot_c, int& tot_t, int* wc, int* wt) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  xc = c;
  xt = t;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int yc = __shfl_up_sync(0xffffffffu, xc, d), yt = __shfl_up_sync(0xffffffffu, xt, d);
    if (lane >= d) xc += yc, xt += yt;
  }
  if (lane == 31) wc[w] = xc, wt[w] = xt;
  __syncthreads();
  if (w == 0) {
    const int ac = wc[lane], at = wt[lane];
    int sc = ac, s2 = at;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int yc = __shfl_up_sync(0xffffffffu, sc, d), yt = __shfl_up_sync(0xffffffffu, s2, d);
      if (lane >= d) sc += yc, s2 += yt;
    }
    wc[lane] = sc - ac;
    wt[lane] = s2 - at;
    if (lane == 31) wc[32] = sc, wt[32] = s2;
  }
  __syncthreads();
  xc = wc[w] + xc - c;
  xt = wt[w] + xt - t;
  tot_c = wc[32];
  tot_t = wt[32];
  __syncthreads();
}

// one CTA per band: group offsets (cells, tiles) within the band; each
// thread scans a contiguous run of bins
__global__ void __launch_bounds__(1024) k_gs_scan_band(const GsPlan p, const int32_t* band_hist, int32_t* goff,
                                                       int32_t* ght, int32_t* band_tot) {
  __shared__ int wc[33], wt[33];
  const int band = blockIdx.x, bins = p.bins;
  const int32_t* bh = band_hist + (size_t)band * bins;
  int32_t* go = goff + (size_t)band * (bins + 1);
  int32_t* gt = ght + (size_t)band * (bins + 1);
  const int per = (bins + 1023) / 1024, b0 = threadIdx.x * per, b1 = min(bins, b0 + per);
  int cnt[16];  // per <= 16 (bins <= 16 K)
  int sc = 0, stl = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    cnt[j] = b0 + j < b1 ? bh[b0 + j] : 0;
    sc += cnt[j];
    stl += (cnt[j] + p.tile - 1) / p.tile;
  }
  int xc, xt, tc, tt;
  scan_pair(sc, stl, xc, xt, tc, tt, wc, wt);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (b0 + j < b1) {
      go[b0 + j] = xc;
      gt[b0 + j] = xt;
    }
    xc += cnt[j];
    xt += (cnt[j] + p.tile - 1) / p.tile;
  }
  if (threadIdx.x == 0) {
    go[bins] = tc;
    gt[bins] = tt;
    band_tot[2 * band] = tc;
    band_tot[2 * band + 1] = tt;
  }
}

// band bases: band_base[2 b] cells, [2 b + 1] half-tiles before band b;
// entry nbands holds the totals, *n_ht the half-tile count
__global__ void __launch_bounds__(1024) k_gs_scan_bands(const GsPlan p, const int32_t* band_tot, int32_t* band_base,
                                                        int32_t* n_ht) {
  __shared__ int wc[33], wt[33];
  int carry_c = 0, carry_t = 0;
  for (int b0 = 0; b0 < p.nbands; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int c = i < p.nbands ? band_tot[2 * i] : 0, t = i < p.nbands ? band_tot[2 * i + 1] : 0;
    int xc, xt, tc, tt;
    scan_pair(c, t, xc, xt, tc, tt, wc, wt);
    if (i < p.nbands) {
      band_base[2 * i] = carry_c + xc;
      band_base[2 * i + 1] = carry_t + xt;
    }
    carry_c += tc;
    carry_t += tt;
  }
  if (threadIdx.x == 0) {
    band_base[2 * p.nbands] = carry_c;
    band_base[2 * p.nbands + 1] = carry_t;
    n_ht[0] = carry_t;
    n_ht[1] = 0;  // k_direct_gather's work counter
  }
}

// Sorted cell list, no atomics: a cell's position is its band's base + its
// group's offset in the band + its count CTA's base in the group + its rank
// inside that CTA (k_gs_count).  Entry = (rot << 29) | (y << 15) | x
// (gather_supported: W <= 32768, H <= 16384).
__device__ __forceinline__ void scatter_cell(const GsPlan& p, int cap, int s, int r, long long i, long long W,
                                             const int32_t* base, const int32_t* go, const int32_t* ch,
                                             const uint16_t* lrank, uint32_t* sorted) {
  if ((unsigned)s >= (unsigned)cap) return;
  const int b = gs_bin(p, s, r);
  const int pos = base[0] + __ldg(go + b) + __ldg(ch + b) + (int)lrank[i];
  const unsigned y = (unsigned)i / (unsigned)W, x = (unsigned)i - y * (unsigned)W;  // cells < 2^31
  sorted[pos] = ((unsigned)(r & 7) << 29) | (y << 15) | x;
}

__global__ void __launch_bounds__(256) k_gs_scatter(const StepGeom g, const Planes f, const GsPlan p, int cap,
                                                    const int32_t* __restrict__ cta_hist,
                                                    const int32_t* __restrict__ goff,
                                                    const int32_t* __restrict__ band_base,
                                                    const uint16_t* __restrict__ lrank, uint32_t* __restrict__ sorted) {
  const long long W = g.W, n = W * g.H;
  if ((g.W & 3) == 0) {
    // eight cells per thread and iteration: every load of both quads (planes,
    // ranks, then the group / CTA bases) is issued before any store, so the
    // two dependent load rounds are paid once per eight cells
    for (long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8; i0 < n;
         i0 += (long long)gridDim.x * blockDim.x * 8) {
      int sl[8], rt[8], rk[8], pos[8];
      bool ok[8];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long i = i0 + 4 * q;
        const bool in = i < n;
        const int4 G = in ? __ldg(reinterpret_cast<const int4*>(f.gi + i + W)) : make_int4(-1, -1, -1, -1);
        const unsigned R = in ? __ldg(reinterpret_cast<const unsigned*>(f.rot + i + W)) : 0u;
        const uint2 L = in ? __ldg(reinterpret_cast<const uint2*>(lrank + i)) : make_uint2(0u, 0u);
        sl[4 * q] = G.x, sl[4 * q + 1] = G.y, sl[4 * q + 2] = G.z, sl[4 * q + 3] = G.w;
        rt[4 * q] = (int)(R & 0xFFu), rt[4 * q + 1] = (int)((R >> 8) & 0xFFu), rt[4 * q + 2] = (int)((R >> 16) & 0xFFu),
        rt[4 * q + 3] = (int)(R >> 24);
        rk[4 * q] = (int)(L.x & 0xFFFFu), rk[4 * q + 1] = (int)(L.x >> 16), rk[4 * q + 2] = (int)(L.y & 0xFFFFu),
        rk[4 * q + 3] = (int)(L.y >> 16);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long i = i0 + j;
        ok[j] = i < n && (unsigned)sl[j] < (unsigned)cap;
        const int cta = (int)((unsigned)(ok[j] ? i : 0) / (unsigned)W) / p.rows_per_cta, band = cta / p.ctas_per_band;
        const int b = ok[j] ? gs_bin(p, sl[j], rt[j]) : 0;
        pos[j] = __ldg(band_base + 2 * band) + __ldg(goff + (size_t)band * (p.bins + 1) + b) +
                 __ldg(cta_hist + (size_t)cta * p.bins + b) + rk[j];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (ok[j]) {
          const long long i = i0 + j;
          const unsigned y = (unsigned)i / (unsigned)W, x = (unsigned)i - y * (unsigned)W;  // cells < 2^31
          sorted[pos[j]] = ((unsigned)(rt[j] & 7) << 29) | (y << 15) | x;
        }
    }
    return;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int cta = (int)((unsigned)i / (unsigned)W) / p.rows_per_cta, band = cta / p.ctas_per_band;
    scatter_cell(p, cap, __ldg(f.gi + i + W), __ldg(f.rot + i + W), i, W, band_base + 2 * band,
                 goff + (size_t)band * (p.bins + 1), cta_hist + (size_t)cta * p.bins, lrank, sorted);
  }
}

// tile h -> {bin = slot * rb + rot, first list position, cells (1 .. p.tile), 0}
__global__ void k_gs_tilemap(const GsPlan p, const int32_t* goff, const int32_t* ght, const int32_t* band_base,
                             const int32_t* n_ht, int4* info) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= *n_ht) return;
  int lo = 0, hi = p.nbands;  // largest band with base_ht <= h
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(band_base + 2 * mid + 1) <= h) lo = mid; else hi = mid;
  }
  const int band = lo, local = h - __ldg(band_base + 2 * band + 1);
  const int32_t* gt = ght + (size_t)band * (p.bins + 1);
  const int32_t* go = goff + (size_t)band * (p.bins + 1);
  lo = 0;
  hi = p.bins;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(gt + mid) <= local) lo = mid; else hi = mid;
  }
  const int k = local - __ldg(gt + lo);
  const int start = __ldg(go + lo) + k * p.tile;
  info[h] = make_int4(lo, __ldg(band_base + 2 * band) + start, min(p.tile, __ldg(go + lo + 1) - start), 0);
}

// ---------------------------------------------------------------------------
// the net
constexpr int kGwWarps = 4;
constexpr int kGwThreads = kGwWarps * 32;
constexpr int kGwChunk = 8;  // consecutive half-tiles per warp turn (band locality: one turn of all warps ~1.2 M cells)
constexpr int kGwW = kSensors * 12 + 48 + kOutPad;  // W12 [45][12] | W1 [48] | bias [16]

struct GatherArgs {
  Params net;
  const float* tex;  // FFMA kernel: single-cell records from ghost row -1; tensor-core kernel: column triples
  int W;
  const uint32_t* sorted;
  const int4* info;
  int32_t* n_ht;  // [0] half-tiles, [1] work counter (chunks handed out)
  float* act;
  int export_rows;  // 0: 8-float decided records, 1: 16-float actuator rows (cell index)
  FusedPhysics fp;  // kGwFused: the physics runs in the epilogue, act receives the pass-1 records
};
constexpr int kGwDecided = 0, kGwExport = 1, kGwFused = 2;  // k_direct_gather output forms

// C cells per lane (a warp takes a tile of 32 C cells of one slot); D Moore
// records per cell in flight.  C = 2, D = 3: 16 warps per SM (four resident
// CTAs).  Measured: C = 4 (half the weight broadcasts per cell, 12 warps per
// SM, 168 registers) took 1.54 ms against 1.05 ms on config 3 - fewer,
// larger tiles in flight spread over more of the band and the DRAM reads of
// the texture doubled.
template <int C, int D, int MODE>
__global__ void __launch_bounds__(kGwThreads, C == 2 ? 4 : 3) k_direct_gather(const GatherArgs a) {
  constexpr bool EXPORT = MODE == kGwExport;
  if (MODE == kGwFused && blockIdx.x == 0 && threadIdx.x == 0 && a.fp.stats) {
    a.fp.stats[0] = 0;
    a.fp.stats[1] = 0;
  }
  __shared__ __align__(16) float wsm[kGwWarps][kGwW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* W12 = wsm[warp];
  float* W1 = W12 + kSensors * 12;
  float* Bs = W1 + 48;
  const int n = a.n_ht[0], W = a.W;
  // Tiles are handed out in runs of kGwChunk from one counter, so all warps
  // work on neighbouring runs: the texture band they gather from and the
  // records they write stay in L2.  The run after next is claimed when a
  // run starts, hiding the atomic's latency.
  auto claim = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(a.n_ht + 1, 1);
    return __shfl_sync(0xffffffffu, v, 0) * kGwChunk;
  };
  int h = claim();
  int queued = claim();
  if (h >= n) return;
  auto step = [&](int h) {
    ++h;
    if (h % kGwChunk) return h;
    const int q = queued;
    queued = claim();
    return q;
  };
  // the next tile's cells stay packed list entries until their records are
  // asked for (decoded cells cost five registers each)
  auto entries_of = [&](const int4& t, uint32_t (&e)[C]) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int r = lane + 32 * j;
      e[j] = __ldg(a.sorted + t.y + (r < t.z ? r : 0));
    }
  };
  int cur = -1;
  int4 ti = __ldg(a.info + h);
  GCell cc[C];
  uint32_t ne[C];
  entries_of(ti, ne);
#pragma unroll
  for (int j = 0; j < C; ++j) cc[j] = gcell(ne[j], W);
  f8r q[C][3];  // ring of the D = 3 Moore records in flight per cell
#pragma unroll
  for (int s = 0; s < D; ++s)
#pragma unroll
    for (int j = 0; j < C; ++j) q[j][s] = ld_rec(rec_ptr(a.tex, cc[j], W, cc[j].rot, s));
  // the tile info is read two tiles ahead and the cell list one tile ahead,
  // so neither of the two dependent loads (info -> sorted entries -> record
  // addresses) is waited for (13 % of the stall samples sat on that chain)
  int hn = step(h);
  int4 tn = make_int4(0, 0, 1, 0);
  if (hn < n) tn = __ldg(a.info + hn);
  while (h < n) {
    const bool more = hn < n;
    if (more) entries_of(tn, ne);  // else: the last tile reloads its own cells
    const int hnn = more ? step(hn) : hn;
    int4 tnn = make_int4(0, 0, 1, 0);
    if (hnn < n) tnn = __ldg(a.info + hnn);
    const int slot = ti.x;  // groups are (band, slot): each lane gathers in its own cell's Moore order
    if (slot != cur) {
      cur = slot;
      __syncwarp();
      const float4* w12 = reinterpret_cast<const float4*>(a.net.wA + (size_t)cur * kSensors * 12);
      for (int i = lane; i < kSensors * 3; i += 32) reinterpret_cast<float4*>(W12)[i] = __ldg(w12 + i);
      for (int i = lane; i < kSensors; i += 32) W1[i] = __ldg(a.net.wB + (size_t)cur * kSensors + i);
      if (lane < kOutPad) Bs[lane] = __ldg(a.net.bA + (size_t)cur * kOutPad + lane);
      __syncwarp();
    }
    u64 acc[C][6];
    float acc12[C];
    float ce[C], ci[C];  // fused: the cell's own E and I (Moore slot 0), kept for the physics
#pragma unroll
    for (int c = 0; c < C; ++c) {
      ce[c] = q[c][0].v[tex_ch(0)];
      ci[c] = q[c][0].v[tex_ch(1)];
      acc12[c] = 0.0f;
#pragma unroll
      for (int p = 0; p < 6; ++p) acc[c][p] = 0ull;
    }
    // nine Moore slots in three rolled rounds of three (a third of the code
    // of the fully unrolled loop: no_instructions stalls); ring slot j holds
    // Moore slot 3 i + j, refilled with slot 3 i + j + 3 (or the next tile's
    // slot j) as soon as it is consumed
    static_assert(D == 3, "the rolled slot loop keeps three records per cell in flight");
#pragma unroll 1
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int s = 3 * i + j;
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) {
          const int k = 5 * s + ch;
          const float4* w4 = reinterpret_cast<const float4*>(W12 + k * 12);
          const float4 wa = w4[0], wb = w4[1], wc = w4[2];
          const u64 wp[6] = {pk2(wa.x, wa.y), pk2(wa.z, wa.w), pk2(wb.x, wb.y),
                             pk2(wb.z, wb.w), pk2(wc.x, wc.y), pk2(wc.z, wc.w)};
          const float w12 = W1[k];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const float x = q[c][j].v[tex_ch(ch)];
#pragma unroll
            for (int p = 0; p < 6; ++p) ffma2(acc[c][p], x, wp[p]);
            acc12[c] = fmaf(x, w12, acc12[c]);
          }
        }
        // refill (unconditional for the next tile: the last tile reloads its
        // own cells, which keeps a single copy of the loop body)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const GCell gc = i < 2 ? cc[c] : gcell(ne[c], W);
          q[c][j] = ld_rec(rec_ptr(a.tex, gc, W, gc.rot, i < 2 ? s + 3 : j));
        }
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int r = lane + 32 * c;
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
      const int cell = cc[c].cell;
      if (MODE == kGwFused) {
        CellAct ac{};
        ac.acted = true;
        ac.inv = squash(z[0]);
        ac.liq = squash(z[1]);
        ac.m0 = squash(z[2]);
        ac.m1 = squash(z[3]);
        ac.m2 = squash(z[4]);
        explore_pick(z + 5, ac.kstar, ac.xmax);
        // the communication channels only matter when the phase is off or
        // the cell starves (rare): then the cell's record is read again
        const CellState cs{ce[c], ci[c], 0.0f, 0.0f, 0.0f, slot, cc[c].rot};
        CellOut o = cell_physics(a.fp.s, a.fp.phases, a.fp.src_map, cell, cs, ac);
        if (!(a.fp.phases & EVO_PH_COMM) || o.slot < 0) {  // write_communication of cell_physics on the real channels
          const f8r own = ld_rec(rec_ptr(a.tex, cc[c], W, cc[c].rot, 0));
          const bool decay = (a.fp.phases & EVO_PH_COMM) != 0;  // here: the cell starved (physics.py:245-247)
          o.c0 = decay ? __fmul_rn(own.v[tex_ch(2)], 0.9f) : own.v[tex_ch(2)];
          o.c1 = decay ? __fmul_rn(own.v[tex_ch(3)], 0.9f) : own.v[tex_ch(3)];
          o.c2 = decay ? __fmul_rn(own.v[tex_ch(4)], 0.9f) : own.v[tex_ch(4)];
        }
        st_mid(a.act + (size_t)cell * 8, o);
      } else if (!EXPORT) {  // 32 bytes at the cell index (explore_pick is exact)
        int ks;
        float xm;
        explore_pick(z + 5, ks, xm);
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a.act + (size_t)cell * 8),
                     "f"(squash(z[0])), "f"(squash(z[1])), "f"(squash(z[2])), "f"(squash(z[3])), "f"(squash(z[4])),
                     "f"(xm), "f"(__int_as_float(ks)), "f"(0.0f)
                     : "memory");
      } else {
        float v[16];
#pragma unroll
        for (int j = 0; j < 13; ++j) v[j] = squash(z[j]);
        v[13] = v[14] = v[15] = 0.0f;
        float4* dst = reinterpret_cast<float4*>(a.act + (size_t)cell * 16);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) dst[qq] = make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
      }
    }
    h = hn;
    ti = tn;
    hn = hnn;
    tn = tnn;
#pragma unroll
    for (int j = 0; j < C; ++j) cc[j] = gcell(ne[j], W);
  }
}

// ---------------------------------------------------------------------------
// The net on the tensor cores (k_direct_tc, EVO_F_TC_DIRECT).  One 128-cell
// tile of one (band, slot) group per MMA: thread t owns tile row t = TMEM
// lane t and gathers its cell's nine records in the cell's own Moore order
// (per-row rotation, so the rows need no uniformity); the 48 inputs are
// split x = hi + lo (hi = x with the low 13 mantissa bits cleared, lo = x -
// hi exact): A_hi goes into the thread's TMEM lane (tcgen05.st), A_lo into a
// canonical K-major shared-memory tile.  B' = [W_hi | W_lo] (N = 32), so per
// K step two tcgen05.mma kind::tf32 (M = 128, N = 32, K = 8) give
//   D[:, j] += (A_hi + A_lo) . W_hi[:, j],  D[:, 16 + j] += (A_hi + A_lo) . W_lo[:, j]
// (lo.lo included).  The tensor core accumulates with less than FP32
// accuracy (tools/microbench/tc_split.cu), so the W_lo terms keep their own
// columns and K steps 0-2 and 3-5 go to two accumulators, added in FP32 by
// the epilogue: z_j = ((D0[j] + D0[16 + j]) + (D1[j] + D1[16 + j])) + b_j.
// Measured: with all three cross products in one 16-column accumulator the
// error reached 3.3x that of the FP32 FFMA forward (over the 1e-5 tier-B
// target at BASELINE weights); this layout stays within 2x.  The summation
// order differs from the FFMA paths' (parity: tier B against the float64
// oracle).  TMEM per CTA: A_hi 48 + D0 32 + D1 32 columns (128 allocated),
// so 4 CTAs per SM.  Tiles are claimed in runs of kTcChunk from one counter (all CTAs
// sweep the bands together: the texture band stays in L2); each tile's info
// and row cell are loaded two tiles ahead, its records and weights one tile
// ahead, overlapping the previous tile's MMAs and epilogue.
constexpr int kTcThreads = 128;
constexpr int kTcCols = 128;
constexpr int kTcChunk = 4;  // consecutive tiles per claim (one slot's weights mostly stay staged)
constexpr int kTcK = 48;
constexpr int kTcWPer = 16 * kTcK / kTcThreads;  // weight elements staged per thread (6)
constexpr uint32_t kTcD0 = 64, kTcD1 = 96;  // TMEM accumulator columns (A_hi at 0..47)

struct __align__(1024) TcSmem {
  unsigned char Alo[128 * kTcK * 4];  // 24 KB, canonical K-major (R = 128)
  unsigned char B[32 * kTcK * 4];     // 6 KB: [W_hi | W_lo], canonical K-major (R = 32)
  float bias[16];
  int ring[4];  // claimed runs (first tile index), consumed in order
  uint32_t tmem;
  uint64_t bar;
};

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// weight element e (0 .. 16 * 48) of a slot: output n = e % 16, sensor k = e / 16
__device__ __forceinline__ float tc_weight(const Params& net, int slot, int e) {
  const int n = e & 15, k = e >> 4;
  if (k >= kSensors || n > 12) return 0.0f;
  return n < 12 ? __ldg(net.wA + ((size_t)slot * kSensors + k) * 12 + n) : __ldg(net.wB + (size_t)slot * kSensors + k);
}

// one MMA, A from TMEM, in warp-uniform control flow with an elected issuing
// lane (tools/microbench/tc_issue.cu: ~39 issue cycles per MMA, against ~73
// for a `tid == 0` loop that ptxas wraps in ELECT / BRA.U.ANY waterfalls)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
// the same with A from a shared-memory descriptor
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

__global__ void __launch_bounds__(kTcThreads, 4) k_direct_tc(const GatherArgs a) {
  __shared__ TcSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n = a.n_ht[0], W = a.W;
  auto claim = [&]() { return atomicAdd(a.n_ht + 1, 1) * kTcChunk; };
  if (warp == 0) tc::tmem_alloc<kTcCols>(&sm.tmem);
  if (tid == 0) {
    tc::mbar_init(&sm.bar, 1);
    sm.ring[3] = claim();  // this CTA's first run
    sm.ring[0] = claim();
    sm.ring[1] = claim();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tmem;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  uint32_t phase = 0;
  int cur = -1;
  int k = 0;  // ring slots consumed
  // the tile after h: the next one in the run, or the next claimed run
  // (whose slot is refilled two runs ahead by thread 0)
  auto next_tile = [&](int h) {
    if ((h + 1) % kTcChunk) return h + 1;
    const int r = sm.ring[k & 3];
    if (tid == 0) sm.ring[(k + 2) & 3] = claim();
    ++k;
    return r;
  };
  int h = sm.ring[3];
  int h1 = next_tile(h);
  int h2 = next_tile(h1);
  auto entry_of = [&](const int4& t) { return __ldg(a.sorted + t.y + (tid < t.z ? tid : 0)); };
  int4 ti = make_int4(-1, 0, 1, 0), t1 = ti, t2 = ti;
  uint32_t ecur = 0, e1 = 0, e2 = 0;
  f8r q[9];
  float wn[kTcWPer], bn = 0.0f;
  auto fetch_records = [&](const int4& t, uint32_t e, int have_slot) {
    const GCell c = gcell(e, W);
    if (tid < t.z) {
#pragma unroll
      for (int s = 0; s < 9; ++s) q[s] = ld_rec(rec_ptr(a.tex, c, W, c.rot, s));
    } else {
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int j = 0; j < 8; ++j) q[s].v[j] = 0.0f;
    }
    if (t.x != have_slot) {
#pragma unroll
      for (int j = 0; j < kTcWPer; ++j) wn[j] = tc_weight(a.net, t.x, tid + j * kTcThreads);
      bn = tid < 16 ? __ldg(a.net.bA + (size_t)t.x * kOutPad + tid) : 0.0f;
    }
  };
  if (h < n) {
    ti = __ldg(a.info + h);
    ecur = entry_of(ti);
    fetch_records(ti, ecur, -1);
  }
  if (h1 < n) {
    t1 = __ldg(a.info + h1);
    e1 = entry_of(t1);
  }
  while (h < n) {
    if (h2 < n) {  // two ahead: info + row entry
      t2 = __ldg(a.info + h2);
      e2 = entry_of(t2);
    }
    // (A) inputs split: hi into this thread's TMEM lane (columns 0..47), lo
    //     into row tid of the shared tile
    {
      uint32_t hv[48], lv[48];
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) {
          const float x = q[s].v[tex_ch(ch)];
          const uint32_t hb = __float_as_uint(x) & 0xFFFFE000u;
          hv[s * 5 + ch] = hb;
          lv[s * 5 + ch] = __float_as_uint(__fsub_rn(x, __uint_as_float(hb)));
        }
#pragma unroll
      for (int kk = 45; kk < 48; ++kk) hv[kk] = lv[kk] = 0u;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        uint32_t v16[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v16[j] = hv[16 * c + j];
        tmem_st16(lane_base + 16 * c, v16);
      }
#pragma unroll
      for (int c = 0; c < 12; ++c)
        *reinterpret_cast<uint4*>(sm.Alo + tc::canon_off(tid, 4 * c, 128)) =
            make_uint4(lv[4 * c], lv[4 * c + 1], lv[4 * c + 2], lv[4 * c + 3]);
    }
    // (B) the slot's weights (prefetched with the tile)
    if (ti.x != cur) {
      cur = ti.x;
#pragma unroll
      for (int j = 0; j < kTcWPer; ++j) {
        const int e = tid + j * kTcThreads, nn = e & 15, kk = e >> 4;
        const uint32_t hb = __float_as_uint(wn[j]) & 0xFFFFE000u;
        *reinterpret_cast<uint32_t*>(sm.B + tc::canon_off(nn, kk, 32)) = hb;
        *reinterpret_cast<float*>(sm.B + tc::canon_off(nn + 16, kk, 32)) = __fsub_rn(wn[j], __uint_as_float(hb));
      }
      if (tid < 16) sm.bias[tid] = bn;
    }
    tc::fence_async_smem();
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // (C) 12 MMAs by warp 0: per K step A_hi.B' (TMEM) and A_lo.B' (shared)
    if (warp == 0) {
      constexpr uint32_t id = tc::idesc_tf32(128, 32);
      constexpr uint32_t lB = 32 * 16, lA = 128 * 16;
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sm.B), lB, 128);
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sm.Alo), lA, 128);
#pragma unroll
      for (int ks = 0; ks < 6; ++ks) {
        const uint32_t d = tmem + (ks < 3 ? kTcD0 : kTcD1);
        const uint64_t b = bd + (uint64_t)((2 * ks * lB) >> 4);
        mma_ts(d, tmem + (uint32_t)(8 * ks), b, id, (uint32_t)(ks % 3 != 0));
        mma_ss(d, ad + (uint64_t)((2 * ks * lA) >> 4), b, id, 1u);
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
              tc::smem_u32(&sm.bar))
          : "memory");
    }
    // (D) the next tile's records and weights go out while the MMAs run
    const int4 tcur = ti;
    const int cell = gcell(ecur, W).cell;
    if (h1 < n) fetch_records(t1, e1, tcur.x);
    // (E) epilogue
    tc::mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    tc::fence_after();
    uint32_t d0[16], d0l[16], d1[16], d1l[16];
    tc::tmem_ld16_nw(lane_base + kTcD0, d0);
    tc::tmem_ld16_nw(lane_base + kTcD0 + 16, d0l);
    tc::tmem_ld16_nw(lane_base + kTcD1, d1);
    tc::tmem_ld16_nw(lane_base + kTcD1 + 16, d1l);
    tc::tmem_wait_ld();
    tc::reg_fence(d0);
    tc::reg_fence(d0l);
    tc::reg_fence(d1);
    tc::reg_fence(d1l);
    if (tid < tcur.z) {
      float z[13];
#pragma unroll
      for (int j = 0; j < 13; ++j) {
        const float p0 = __fadd_rn(__uint_as_float(d0[j]), __uint_as_float(d0l[j]));
        const float p1 = __fadd_rn(__uint_as_float(d1[j]), __uint_as_float(d1l[j]));
        z[j] = __fadd_rn(__fadd_rn(p0, p1), sm.bias[j]);
      }
      if (!a.export_rows) {
        int ks;
        float xm;
        explore_pick(z + 5, ks, xm);
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a.act + (size_t)cell * 8),
                     "f"(squash(z[0])), "f"(squash(z[1])), "f"(squash(z[2])), "f"(squash(z[3])), "f"(squash(z[4])),
                     "f"(xm), "f"(__int_as_float(ks)), "f"(0.0f)
                     : "memory");
      } else {
        float v[16];
#pragma unroll
        for (int j = 0; j < 13; ++j) v[j] = squash(z[j]);
        v[13] = v[14] = v[15] = 0.0f;
        float4* dst = reinterpret_cast<float4*>(a.act + (size_t)cell * 16);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) dst[qq] = make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM A_hi / D, the shared A_lo and B' free for the next tile
    tc::fence_after();
    h = h1;
    h1 = h2;
    h2 = h2 < n ? next_tile(h2) : n;
    ti = t1;
    ecur = e1;
    t1 = t2;
    e1 = e2;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTcCols>(tmem);
}

GsPlan make_plan(int W, int H, int cap, int num_sms, int tile, long long band_cells = band_cells_default()) {
  GsPlan p;
  p.rb = 1;  // both nets gather each row in its own Moore order
  p.tile = tile;
  const long long cells = (long long)W * H;
  int r = (int)((cells + 4LL * num_sms * W - 1) / (4LL * num_sms * W));
  r = std::max(1, std::min(r, std::max(1, 65536 / W)));
  p.rows_per_cta = r;
  p.ctas_per_band = (int)std::max(1LL, std::min((long long)(H + r - 1) / r, band_cells / ((long long)r * W)));
  p.nctas = (H + r - 1) / r;
  p.nbands = (p.nctas + p.ctas_per_band - 1) / p.ctas_per_band;
  p.bins = cap * p.rb;
  return p;
}

}  // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time libcuda dependency)
bool make_gather_maps(const Planes& f, const StepGeom& g, float* tex, GatherMaps* out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<Encode>(fn);
  }
  if ((g.W * 4) % 16 != 0) return false;  // TMA row pitch: a multiple of 16 bytes
  const cuuint64_t dims[2] = {(cuuint64_t)g.W, (cuuint64_t)g.H + 2};
  const cuuint64_t pitch[1] = {(cuuint64_t)g.W * 4};
  const cuuint32_t box[2] = {kTmChunk, 1}, es[2] = {1, 1};
  const void* base[6] = {f.E, f.I, f.C, f.C + g.stride, f.C + 2 * g.stride, f.gi};
  for (int k = 0; k < 6; ++k)
    if (encode(&out->plane[k], k == 5 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
               const_cast<void*>(base[k]), dims, pitch, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  const cuuint64_t tdims[3] = {8, (cuuint64_t)g.W, (cuuint64_t)g.H + 2};
  const cuuint64_t tpitch[2] = {32, (cuuint64_t)g.W * 32};
  const cuuint32_t tbox[3] = {8, kTmChunk, 1}, tes[3] = {1, 1, 1};
  return encode(&out->tex, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, tex, tdims, tpitch, tbox, tes,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool gather_supported(int W, int H, int cap) {
  return cap <= kGatherMaxCap && W >= 2 && W <= 32768 && H <= 16384 && (long long)W * H < (1LL << 31);
}

GatherSizes gather_sizes(int W, int H, int cap, int num_sms) {
  const GsPlan a = make_plan(W, H, cap, num_sms, 64), b = make_plan(W, H, cap, num_sms, 128);
  GatherSizes s;
  s.nbands = std::max(a.nbands, b.nbands);
  s.nctas = std::max(a.nctas, b.nctas);
  s.bins = std::max(a.bins, b.bins);
  s.max_ht = std::max((long long)W * H / a.tile + (long long)a.nbands * a.bins,
                      (long long)W * H / b.tile + (long long)b.nbands * b.bins) + 1;
  return s;
}

cudaError_t launch_gather_sort(const GatherBuffers& b, const StepGeom& g, const Planes& front, int cap, int num_sms,
                               int tile, bool one_band, int32_t* rank, cudaStream_t st, const GatherMaps* maps,
                               const FusedPhysics* fused, float* mid_rec, bool tex_is_state) {
  if (fused && !maps) return cudaErrorInvalidValue;  // the fused step's unoccupied cells go through the TMA build
  if (tex_is_state && (!fused || (g.W & 3))) return cudaErrorInvalidValue;
  const GsPlan p = make_plan(g.W, g.H, cap, num_sms, tile, one_band ? (long long)g.W * g.H : band_cells_default());
  if (tex_is_state) {  // ranks only: the texture holds the state (lazy fused steps)
    const size_t hsmem = (size_t)p.bins * 4;
    if (hsmem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_gs_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
      if (e != cudaSuccess) return e;
    }
    k_gs_rank<<<p.nctas, kGsThreads, hsmem, st>>>(g, front.gi, p, cap, b.cta_hist, b.lrank, b.tex, *fused, mid_rec);
  } else if (maps) {
    const size_t smem = 2 * sizeof(TmStage) + (size_t)p.bins * 4;
    cudaError_t e = cudaFuncSetAttribute(k_gs_count_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_gs_count_tma<<<p.nctas, kTmThreads, smem, st>>>(g, *maps, p, cap, b.cta_hist, b.lrank, rank,
                                                     fused ? *fused : FusedPhysics{}, fused ? mid_rec : nullptr);
  } else {
    const size_t hsmem = (size_t)p.bins * 4;
    if (hsmem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_gs_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
      if (e != cudaSuccess) return e;
    }
    k_gs_count<<<p.nctas, kGsThreads, hsmem, st>>>(g, front, p, cap, b.cta_hist, b.lrank, b.tex, rank);
  }
  k_gs_colscan<<<p.nbands * ((p.bins + 31) / 32), 1024, 0, st>>>(p, b.cta_hist, b.band_hist);
  k_gs_scan_band<<<p.nbands, 1024, 0, st>>>(p, b.band_hist, b.goff, b.ght, b.band_tot);
  k_gs_scan_bands<<<1, 1024, 0, st>>>(p, b.band_tot, b.band_base, b.n_ht);
  k_gs_scatter<<<num_sms * 8, 256, 0, st>>>(g, front, p, cap, b.cta_hist, b.goff, b.band_base, b.lrank, b.sorted);
  const long long max_ht = (long long)g.W * g.H / p.tile + (long long)p.nbands * p.bins + 1;
  k_gs_tilemap<<<(unsigned)((max_ht + 255) / 256), 256, 0, st>>>(p, b.goff, b.ght, b.band_base, b.n_ht, b.info);
  return cudaGetLastError();
}

cudaError_t launch_direct_gather(const GatherBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                                 int cap, int num_sms, int variant, bool export_rows, float* act, int32_t* rank,
                                 cudaStream_t st, const GatherMaps* maps, const FusedPhysics* fused,
                                 bool tex_is_state) {
  const bool tc = variant == kGatherTc;
  if (fused && (tc || export_rows)) return cudaErrorInvalidValue;
  cudaError_t e = launch_gather_sort(b, g, front, cap, num_sms, tc ? 128 : 64, false, export_rows ? rank : nullptr,
                                     st, maps, fused, act, tex_is_state);
  if (e != cudaSuccess) return e;
  GatherArgs a;
  a.net = net;
  a.tex = b.tex;
  a.W = g.W;
  a.sorted = b.sorted;
  a.info = b.info;
  a.n_ht = b.n_ht;
  a.act = act;
  a.export_rows = export_rows ? 1 : 0;
  a.fp = fused ? *fused : FusedPhysics{};
  if (fused)
    k_direct_gather<2, 3, kGwFused><<<num_sms * 4, kGwThreads, 0, st>>>(a);
  else if (tc)
    k_direct_tc<<<num_sms * 4, kTcThreads, 0, st>>>(a);  // 4 CTAs per SM, 128 TMEM columns each
  else if (export_rows)
    k_direct_gather<2, 3, kGwExport><<<num_sms * 4, kGwThreads, 0, st>>>(a);
  else
    k_direct_gather<2, 3, kGwDecided><<<num_sms * 4, kGwThreads, 0, st>>>(a);  // 16 warps per SM, one wave
  return cudaGetLastError();
}

cudaError_t launch_tex_to_planes(const float* tex, const StepGeom& g, const Planes& front, int num_sms,
                                 cudaStream_t st) {
  k_tex_to_planes<<<num_sms * 8, 256, 0, st>>>(g, tex, front);
  return cudaGetLastError();
}

}  // namespace evo
