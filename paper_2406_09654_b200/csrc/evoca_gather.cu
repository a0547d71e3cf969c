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
//   k_gs_count    per row band (~1 M cells, so the band's texture stays in
//                 the 126 MB L2): histogram of the occupied cells by
//                 (slot, rotation), and the 32-byte sense texture record of
//                 every cell {E, I, C0, C1, C2, 0, 0, 0} (one sector)
//   k_gs_scan_band / k_gs_scan_bands  group offsets within bands, band bases
//   k_gs_scatter  cell list sorted by (band, slot, rotation)
//   k_gs_tilemap  64-cell half-tiles of one (band, slot, rotation) group
//   k_direct_gather  one warp per half-tile: slot AND rotation are uniform,
//                 so the Moore slot order (PERM_TABLE[rot], physics.py:48-62)
//                 is a warp-uniform offset and the weights are warp-uniform
//                 broadcasts; each lane gathers its two cells' nine texture
//                 records (whole 32-byte sectors, L2 hits: half-tiles are
//                 handed out band by band) and runs the tile kernel's FFMA2
//                 chains in the same k order, so the actions are
//                 bit-identical to the tile and rows paths.  Output: the
//                 32-byte decided record at the cell index (k_physics_rows),
//                 or 16-float actuator rows at the cell index (export).

#include <algorithm>

#include "evoca_net.cuh"
#include "evoca_tc.cuh"

namespace evo {

namespace {

constexpr int kGsThreads = 512;  // count / scatter CTA
// GsPlan.rb: bins per slot (8 = one per rotation for the FFMA warp kernel,
// whose Moore order must be warp-uniform; 1 for the tensor-core kernel,
// which gathers each row in its own order); GsPlan.tile: cells per tile
// (64 = one warp, 128 = one MMA M).
constexpr int kGsBandCells = 1 << 20;

struct GsPlan {
  int rows_per_cta, ctas_per_band, nctas, nbands, bins, rb, tile;
};
__device__ __forceinline__ int gs_bin(const GsPlan& p, int s, int r) { return s * p.rb + (r & (p.rb - 1)); }

__device__ __forceinline__ void st_rec(float* p, float e, float i, float c0, float c1, float c2) {
  // (no "memory" clobber: nothing in the writing kernel reads the texture,
  //  and the clobber would pin every later load behind the store)
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%6,%6};" ::"l"(p), "f"(e), "f"(i), "f"(c0), "f"(c1),
               "f"(c2), "f"(0.0f));
}

// Texture records of the CTA's rows (plus ghost row -1 / H on the first /
// last CTA) and the band histogram by (slot, rotation).  Slots outside
// [0, cap) are left out (no out-of-bounds shared-memory write); the step's
// range check reports them.  Widths divisible by 4 move four cells per
// thread and iteration with 16-byte plane loads.
__device__ __forceinline__ void count_cell(const GsPlan& p, int* hist, int cap, int s, int r, int32_t* rank, long long i,
                                           bool in) {
  if (!in) return;
  const bool occ = (unsigned)s < (unsigned)cap;
  if (occ) atomicAdd(&hist[gs_bin(p, s, r)], 1);
  if (rank) rank[i] = occ ? (int)i : -1;
}

__global__ void __launch_bounds__(kGsThreads) k_gs_count(const StepGeom g, const Planes f, const GsPlan p,
                                                          int cap, int32_t* band_hist, float* tex, int32_t* rank) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * p.rows_per_cta, r1 = min(g.H, r0 + p.rows_per_cta);
  const long long W = g.W, st = g.stride;
  const long long lo = (blockIdx.x == 0 ? -1 : r0) * W, hi = (r1 == g.H ? g.H + 1 : r1) * W;
  const long long c0 = (long long)r0 * W, c1 = (long long)r1 * W;
  if ((g.W & 3) == 0) {
    for (long long i = lo + 4 * threadIdx.x; i < hi; i += 4 * blockDim.x) {
      const long long o = i + W;  // element offset from ghost row -1
      const float4 E = __ldg(reinterpret_cast<const float4*>(f.E + o));
      const float4 I = __ldg(reinterpret_cast<const float4*>(f.I + o));
      const float4 C0 = __ldg(reinterpret_cast<const float4*>(f.C + o));
      const float4 C1 = __ldg(reinterpret_cast<const float4*>(f.C + st + o));
      const float4 C2 = __ldg(reinterpret_cast<const float4*>(f.C + 2 * st + o));
      const bool in = i >= c0 && i < c1;
      int4 G = make_int4(-1, -1, -1, -1);
      unsigned R = 0;
      if (in) {
        G = __ldg(reinterpret_cast<const int4*>(f.gi + o));
        R = __ldg(reinterpret_cast<const unsigned*>(f.rot + o));
      }
      float* t = tex + o * 8;
      st_rec(t, E.x, I.x, C0.x, C1.x, C2.x);
      st_rec(t + 8, E.y, I.y, C0.y, C1.y, C2.y);
      st_rec(t + 16, E.z, I.z, C0.z, C1.z, C2.z);
      st_rec(t + 24, E.w, I.w, C0.w, C1.w, C2.w);
      count_cell(p, hist, cap, G.x, (int)(R & 0xFFu), rank, i, in);
      count_cell(p, hist, cap, G.y, (int)((R >> 8) & 0xFFu), rank, i + 1, in);
      count_cell(p, hist, cap, G.z, (int)((R >> 16) & 0xFFu), rank, i + 2, in);
      count_cell(p, hist, cap, G.w, (int)(R >> 24), rank, i + 3, in);
    }
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const long long o = i + W;
      st_rec(tex + o * 8, __ldg(f.E + o), __ldg(f.I + o), __ldg(f.C + o), __ldg(f.C + st + o),
             __ldg(f.C + 2 * st + o));
      const bool in = i >= c0 && i < c1;
      count_cell(p, hist, cap, in ? __ldg(f.gi + o) : -1, in ? __ldg(f.rot + o) : 0, rank, i, in);
    }
  }
  __syncthreads();
  int32_t* bh = band_hist + (size_t)(blockIdx.x / p.ctas_per_band) * p.bins;
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x)
    if (hist[b]) atomicAdd(bh + b, hist[b]);
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

// one CTA per band: group offsets (cells, half-tiles) within the band; each
// thread scans a contiguous run of bins; the band histogram is consumed
// (zeroed for the next step)
__global__ void __launch_bounds__(1024) k_gs_scan_band(const GsPlan p, int32_t* band_hist, int32_t* goff,
                                                       int32_t* ght, int32_t* cursor, int32_t* band_tot) {
  __shared__ int wc[33], wt[33];
  const int band = blockIdx.x, bins = p.bins;
  int32_t* bh = band_hist + (size_t)band * bins;
  int32_t* go = goff + (size_t)band * (bins + 1);
  int32_t* gt = ght + (size_t)band * (bins + 1);
  int32_t* cu = cursor + (size_t)band * bins;
  const int per = (bins + 1023) / 1024, b0 = threadIdx.x * per, b1 = min(bins, b0 + per);
  int sc = 0, stl = 0;
  for (int b = b0; b < b1; ++b) {
    const int c = bh[b];
    sc += c;
    stl += (c + p.tile - 1) / p.tile;
  }
  int xc, xt, tc, tt;
  scan_pair(sc, stl, xc, xt, tc, tt, wc, wt);
  for (int b = b0; b < b1; ++b) {
    const int c = bh[b];
    bh[b] = 0;
    go[b] = xc;
    gt[b] = xt;
    cu[b] = xc;
    xc += c;
    xt += (c + p.tile - 1) / p.tile;
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

// Sorted cell list: per CTA, one global reservation per non-empty (slot,
// rotation) group, then shared-memory ranks.  Order inside a group depends on
// atomic arrival, which changes no result (each cell's forward pass is
// independent of its neighbours in the list).  Entry = (rot << 29) | (y << 15)
// | x (gather_supported: W <= 32768, H <= 16384).
__device__ __forceinline__ void scatter_cell(const GsPlan& p, int* hist, int cap, int s, int r, long long i,
                                             long long W, uint32_t* sorted) {
  if ((unsigned)s >= (unsigned)cap) return;
  const int pos = atomicAdd(&hist[gs_bin(p, s, r)], 1);
  const unsigned y = (unsigned)i / (unsigned)W, x = (unsigned)i - y * (unsigned)W;  // cells < 2^31
  sorted[pos] = ((unsigned)(r & 7) << 29) | (y << 15) | x;
}

__global__ void __launch_bounds__(kGsThreads) k_gs_scatter(const StepGeom g, const Planes f, const GsPlan p, int cap,
                                                            int32_t* cursor, const int32_t* band_base,
                                                            uint32_t* sorted) {
  extern __shared__ int hist[];
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int r0 = blockIdx.x * p.rows_per_cta, r1 = min(g.H, r0 + p.rows_per_cta);
  const long long W = g.W;
  const long long c0 = (long long)r0 * W, c1 = (long long)r1 * W;
  const bool v4 = (g.W & 3) == 0;
  if (v4) {
    for (long long i = c0 + 4 * threadIdx.x; i < c1; i += 4 * blockDim.x) {
      const int4 G = __ldg(reinterpret_cast<const int4*>(f.gi + i + W));
      const unsigned R = __ldg(reinterpret_cast<const unsigned*>(f.rot + i + W));
      if ((unsigned)G.x < (unsigned)cap) atomicAdd(&hist[gs_bin(p, G.x, (int)R)], 1);
      if ((unsigned)G.y < (unsigned)cap) atomicAdd(&hist[gs_bin(p, G.y, (int)(R >> 8))], 1);
      if ((unsigned)G.z < (unsigned)cap) atomicAdd(&hist[gs_bin(p, G.z, (int)(R >> 16))], 1);
      if ((unsigned)G.w < (unsigned)cap) atomicAdd(&hist[gs_bin(p, G.w, (int)(R >> 24))], 1);
    }
  } else {
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
      const int s = __ldg(f.gi + i + W);
      if ((unsigned)s < (unsigned)cap) atomicAdd(&hist[gs_bin(p, s, __ldg(f.rot + i + W))], 1);
    }
  }
  __syncthreads();
  const int band = blockIdx.x / p.ctas_per_band;
  const int base = band_base[2 * band];
  int32_t* cur = cursor + (size_t)band * p.bins;
  for (int b = threadIdx.x; b < p.bins; b += blockDim.x)
    if (hist[b]) hist[b] = base + atomicAdd(cur + b, hist[b]);
  __syncthreads();
  if (v4) {
    for (long long i = c0 + 4 * threadIdx.x; i < c1; i += 4 * blockDim.x) {
      const int4 G = __ldg(reinterpret_cast<const int4*>(f.gi + i + W));
      const unsigned R = __ldg(reinterpret_cast<const unsigned*>(f.rot + i + W));
      scatter_cell(p, hist, cap, G.x, (int)(R & 0xFFu), i, W, sorted);
      scatter_cell(p, hist, cap, G.y, (int)((R >> 8) & 0xFFu), i + 1, W, sorted);
      scatter_cell(p, hist, cap, G.z, (int)((R >> 16) & 0xFFu), i + 2, W, sorted);
      scatter_cell(p, hist, cap, G.w, (int)(R >> 24), i + 3, W, sorted);
    }
  } else {
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x)
      scatter_cell(p, hist, cap, __ldg(f.gi + i + W), __ldg(f.rot + i + W), i, W, sorted);
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
constexpr int kGwDepth = 3;  // Moore-slot records per cell in flight
constexpr int kGwChunk = 8;  // consecutive half-tiles per warp turn (band locality: one turn of all warps ~1.2 M cells)
constexpr int kGwW = kSensors * 12 + 48 + kOutPad;  // W12 [45][12] | W1 [48] | bias [16]

struct GatherArgs {
  Params net;
  const float* tex;  // record of ghost row -1, column 0
  int W;
  const uint32_t* sorted;
  const int4* info;
  int32_t* n_ht;  // [0] half-tiles, [1] work counter (chunks handed out)
  float* act;
  int export_rows;  // 0: 8-float decided records, 1: 16-float actuator rows (cell index)
};

struct f8r {
  float v[8];
};
__device__ __forceinline__ f8r ld_rec(const float* p) {
  f8r r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                 "=f"(r.v[7])
               : "l"(p));
  return r;
}

// one lane's cell of a half-tile: texture index of its centre record and
// the wrap corrections for x - 1 / x + 1 on the torus seam
struct GCell {
  int idx;   // (y + 1) * W + x
  int wl;    // +W when x == 0 (a dx = -1 neighbour wraps)
  int wr;    // -W when x == W - 1
  int cell;  // y * W + x
};
__device__ __forceinline__ GCell gcell(uint32_t e, int W) {
  GCell c;
  const int y = (int)((e >> 15) & 0x3FFFu), x = (int)(e & 0x7FFFu);
  c.cell = y * W + x;
  c.idx = c.cell + W;
  c.wl = x == 0 ? W : 0;
  c.wr = x == W - 1 ? -W : 0;
  return c;
}
// Moore slot s of a (rot)-group: texture offset dy * W + dx and dx
__device__ __forceinline__ int slot_dx(int rot, int s) { return s == 0 ? 0 : dir_dx(perm_dir(rot, s - 1)); }
__device__ __forceinline__ int slot_dy(int rot, int s) { return s == 0 ? 0 : dir_dy(perm_dir(rot, s - 1)); }
__device__ __forceinline__ const float* rec_ptr(const float* tex, const GCell& c, int W, int rot, int s) {
  const int dx = slot_dx(rot, s), dy = slot_dy(rot, s);
  const int i = c.idx + dy * W + dx + (dx < 0 ? c.wl : 0) + (dx > 0 ? c.wr : 0);
  return tex + (size_t)i * 8;
}

__global__ void __launch_bounds__(kGwThreads, 4) k_direct_gather(const GatherArgs a) {
  __shared__ __align__(16) float wsm[kGwWarps][kGwW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* W12 = wsm[warp];
  float* W1 = W12 + kSensors * 12;
  float* Bs = W1 + 48;
  const int n = a.n_ht[0], W = a.W;
  // Half-tiles are handed out in runs of kGwChunk from one counter, so all
  // warps work on neighbouring runs: the texture band they gather from and
  // the records they write stay in L2.  The run after next is claimed when a
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
  int cur = -1;
  int4 ti = __ldg(a.info + h);
  GCell c0 = gcell(__ldg(a.sorted + ti.y + (lane < ti.z ? lane : 0)), W);
  GCell c1 = gcell(__ldg(a.sorted + ti.y + (lane + 32 < ti.z ? lane + 32 : 0)), W);
  f8r q0[9], q1[9];
  {
    const int rot = ti.x & 7;
#pragma unroll
    for (int s = 0; s < kGwDepth; ++s) {
      q0[s] = ld_rec(rec_ptr(a.tex, c0, W, rot, s));
      q1[s] = ld_rec(rec_ptr(a.tex, c1, W, rot, s));
    }
  }
  while (h < n) {
    const int hn = step(h);
    const bool more = hn < n;
    int4 tn = make_int4(0, 0, 1, 0);
    GCell n0 = c0, n1 = c1;
    if (more) {
      tn = __ldg(a.info + hn);
      n0 = gcell(__ldg(a.sorted + tn.y + (lane < tn.z ? lane : 0)), W);
      n1 = gcell(__ldg(a.sorted + tn.y + (lane + 32 < tn.z ? lane + 32 : 0)), W);
    }
    const int slot = ti.x >> 3, rot = ti.x & 7, rotn = tn.x & 7;
    if (slot != cur) {
      cur = slot;
      __syncwarp();
      const float4* w12 = reinterpret_cast<const float4*>(a.net.wA + (size_t)cur * kSensors * 12);
      for (int i = lane; i < kSensors * 3; i += 32) reinterpret_cast<float4*>(W12)[i] = __ldg(w12 + i);
      for (int i = lane; i < kSensors; i += 32) W1[i] = __ldg(a.net.wB + (size_t)cur * kSensors + i);
      if (lane < kOutPad) Bs[lane] = __ldg(a.net.bA + (size_t)cur * kOutPad + lane);
      __syncwarp();
    }
    u64 acc[2][6];
    float acc12[2] = {0.0f, 0.0f};
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int p = 0; p < 6; ++p) acc[c][p] = 0ull;
#pragma unroll
    for (int k = 0; k < kSensors; ++k) {
      const int s = k / 5, ch = k - 5 * s;
      if (ch == 0 && s + kGwDepth < 9) {  // keep kGwDepth records per cell in flight
        q0[s + kGwDepth] = ld_rec(rec_ptr(a.tex, c0, W, rot, s + kGwDepth));
        q1[s + kGwDepth] = ld_rec(rec_ptr(a.tex, c1, W, rot, s + kGwDepth));
      }
      if (ch == 0 && s >= 9 - kGwDepth && more) {  // the next half-tile's leading records
        const int sn = s - (9 - kGwDepth);
        q0[sn] = ld_rec(rec_ptr(a.tex, n0, W, rotn, sn));
        q1[sn] = ld_rec(rec_ptr(a.tex, n1, W, rotn, sn));
      }
      // (q[sn] was last read at slot sn < s: free)
      const float x0 = q0[s].v[ch];
      const float x1 = q1[s].v[ch];
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
      const int r = c ? lane + 32 : lane;
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
      const int cell = c ? c1.cell : c0.cell;
      if (!a.export_rows) {  // 32 bytes at the cell index (explore_pick is exact)
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
        for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
    h = hn;
    ti = tn;
    c0 = n0;
    c1 = n1;
  }
}

// ---------------------------------------------------------------------------
// The net on the tensor cores (k_direct_tc).  One 128-cell tile of one
// (band, slot) group per MMA: thread t owns tile row t = TMEM lane t, gathers
// its cell's nine records in the cell's own Moore order (per-row rotation:
// no uniformity needed), splits the 48 sensors x = hi + lo (hi = x with the
// low 13 mantissa bits cleared, lo = x - hi exact) and stores A' = [hi | lo]
// (K = 96) into its TMEM lane with tcgen05.st.  B' = [W_hi | W_lo] (N = 32,
// K = 48, canonical K-major in shared memory) serves both K halves, so 12
// tcgen05.mma kind::tf32 (M = 128, N = 32, K = 8) give
//   D[:, j] = (A_hi + A_lo) . W_hi[:, j],  D[:, 16 + j] = (A_hi + A_lo) . W_lo[:, j]
// and z_j = D[j] + D[16 + j] + b_j (every cross product of the split,
// lo.lo included).  The epilogue reads D with one tcgen05.ld and writes the
// decided record (or the 13 squashed actuators).  4 CTAs per SM, 128 TMEM
// columns each (A' 96 + D 32); the next tile's records and weights are in
// flight while this tile's MMAs and epilogue run.
constexpr int kTcThreads = 128;
constexpr int kTcCols = 128;
constexpr int kTcChunk = 4;  // consecutive tiles per claim (one slot's weights mostly stay staged)
constexpr int kTcK = 48;
constexpr int kTcN = 32;
constexpr int kTcWPer = 16 * kTcK / kTcThreads;  // weight elements staged per thread (6)

struct __align__(1024) TcSmem {
  unsigned char B[kTcN * kTcK * 4];  // 6 KB
  float bias[16];
  int next;
  uint32_t tmem;
  uint64_t bar;
};

__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}

// weight element e (0 .. 16 * 48) of a slot: output n = e % 16, sensor k = e / 16
__device__ __forceinline__ float tc_weight(const Params& net, int slot, int e) {
  const int n = e & 15, k = e >> 4;
  if (k >= kSensors || n > 12) return 0.0f;
  return n < 12 ? __ldg(net.wA + ((size_t)slot * kSensors + k) * 12 + n) : __ldg(net.wB + (size_t)slot * kSensors + k);
}

__global__ void __launch_bounds__(kTcThreads, 4) k_direct_tc(const GatherArgs a) {
  __shared__ TcSmem sm;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n = a.n_ht[0], W = a.W;
  if (warp == 0) tc::tmem_alloc<kTcCols>(&sm.tmem);
  if (tid == 0) {
    tc::mbar_init(&sm.bar, 1);
    sm.next = atomicAdd(a.n_ht + 1, 1) * kTcChunk;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tmem;
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  int h = sm.next;
  __syncthreads();
  if (tid == 0) sm.next = atomicAdd(a.n_ht + 1, 1) * kTcChunk;  // the run after this one
  uint32_t phase = 0;
  int cur = -1;
  // prefetched state of tile h: info, this row's cell, records, slot weights
  int4 ti = make_int4(0, 0, 1, 0);
  GCell cc{};
  int rot = 0;
  f8r q[9];
  float wn[kTcWPer], bn = 0.0f;
  auto fetch = [&](int hh, int4& t, GCell& c, int& r, int have_slot) {
    t = __ldg(a.info + hh);
    const uint32_t e = __ldg(a.sorted + t.y + (tid < t.z ? tid : 0));
    c = gcell(e, W);
    r = (int)(e >> 29);
#pragma unroll
    for (int s = 0; s < 9; ++s) q[s] = ld_rec(rec_ptr(a.tex, c, W, r, s));
    if (t.x != have_slot) {
#pragma unroll
      for (int j = 0; j < kTcWPer; ++j) wn[j] = tc_weight(a.net, t.x, tid + j * kTcThreads);
      bn = tid < 16 ? __ldg(a.net.bA + (size_t)t.x * kOutPad + tid) : 0.0f;
    }
  };
  if (h < n) fetch(h, ti, cc, rot, -1);
  while (h < n) {
    // (A) this row's sensors, split, into TMEM: hi at columns 0..47, lo at 48..95
    {
      uint32_t hv[48], lv[48];
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int ch = 0; ch < 5; ++ch) {
          const float x = q[s].v[ch];
          const uint32_t hb = __float_as_uint(x) & 0xFFFFE000u;
          hv[s * 5 + ch] = hb;
          lv[s * 5 + ch] = __float_as_uint(__fsub_rn(x, __uint_as_float(hb)));
        }
#pragma unroll
      for (int k = 45; k < 48; ++k) hv[k] = lv[k] = 0u;
      uint32_t c32[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) c32[j] = hv[j];
      tmem_st32(lane_base + 0, c32);
#pragma unroll
      for (int j = 0; j < 16; ++j) c32[j] = hv[32 + j];
#pragma unroll
      for (int j = 0; j < 16; ++j) c32[16 + j] = lv[j];
      tmem_st32(lane_base + 32, c32);
#pragma unroll
      for (int j = 0; j < 32; ++j) c32[j] = lv[16 + j];
      tmem_st32(lane_base + 64, c32);
    }
    // (B) the slot's weights into B' (prefetched with the tile)
    if (ti.x != cur) {
      cur = ti.x;
#pragma unroll
      for (int j = 0; j < kTcWPer; ++j) {
        const int e = tid + j * kTcThreads, nn = e & 15, k = e >> 4;
        const uint32_t hb = __float_as_uint(wn[j]) & 0xFFFFE000u;
        *reinterpret_cast<uint32_t*>(sm.B + tc::canon_off(nn, k, kTcN)) = hb;
        *reinterpret_cast<float*>(sm.B + tc::canon_off(nn + 16, k, kTcN)) = __fsub_rn(wn[j], __uint_as_float(hb));
      }
      if (tid < 16) sm.bias[tid] = bn;
      tc::fence_async_smem();
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // (C) 12 MMAs: K steps 0-5 from A_hi, 6-11 from A_lo, both against B'.
    //     Warp 0 runs the loop in warp-uniform control flow with operands
    //     derived from uniform values, one elected lane issuing inside each
    //     asm block (tools/microbench/tc_issue.cu: ~39 issue cycles per MMA
    //     against ~73 for a per-thread `if (tid == 0)` loop, which ptxas
    //     wraps in ELECT / BRA.U.ANY waterfalls)
    if (warp == 0) {
      constexpr uint32_t id = tc::idesc_tf32(128, kTcN);
      constexpr uint32_t lB = kTcN * 16;
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sm.B), lB, 128);
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const int ks = j % 6;
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + 96u),
            "r"(tmem + (uint32_t)((j < 6 ? 0 : 48) + 8 * ks)), "l"(bd + (uint64_t)((2 * ks * lB) >> 4)), "r"(id),
            "r"((uint32_t)(j > 0)));
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
              tc::smem_u32(&sm.bar))
          : "memory");
    }
    // (D) the next tile's records and weights go out while the MMAs run
    const int4 tcur = ti;
    const GCell ccur = cc;
    int hn = h + 1;
    if (hn % kTcChunk == 0) {
      hn = sm.next;  // read before the barrier below lets thread 0 overwrite it
    }
    const bool more = hn < n;
    if (more) fetch(hn, ti, cc, rot, tcur.x);
    // (E) epilogue
    tc::mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    tc::fence_after();
    uint32_t d[32];
    tmem_ld32(lane_base + 96, d);
    tc::tmem_wait_ld();
    if (tid < tcur.z) {
      float z[13];
#pragma unroll
      for (int j = 0; j < 13; ++j)
        z[j] = __fadd_rn(__fadd_rn(__uint_as_float(d[j]), __uint_as_float(d[16 + j])), sm.bias[j]);
      if (!a.export_rows) {
        int ks;
        float xm;
        explore_pick(z + 5, ks, xm);
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a.act + (size_t)ccur.cell * 8),
                     "f"(squash(z[0])), "f"(squash(z[1])), "f"(squash(z[2])), "f"(squash(z[3])), "f"(squash(z[4])),
                     "f"(xm), "f"(__int_as_float(ks)), "f"(0.0f)
                     : "memory");
      } else {
        float v[16];
#pragma unroll
        for (int j = 0; j < 13; ++j) v[j] = squash(z[j]);
        v[13] = v[14] = v[15] = 0.0f;
        float4* dst = reinterpret_cast<float4*>(a.act + (size_t)ccur.cell * 16);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) dst[qq] = make_float4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM A' / D and B' free; every thread has read sm.next
    tc::fence_after();
    if ((h + 1) % kTcChunk == 0 && tid == 0) sm.next = atomicAdd(a.n_ht + 1, 1) * kTcChunk;
    h = hn;
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kTcCols>(tmem);
}

GsPlan make_plan(int W, int H, int cap, int num_sms, bool tc) {
  GsPlan p;
  p.rb = tc ? 1 : 8;
  p.tile = tc ? 128 : 64;
  const long long cells = (long long)W * H;
  int r = (int)((cells + 4LL * num_sms * W - 1) / (4LL * num_sms * W));
  r = std::max(1, std::min(r, std::max(1, 65536 / W)));
  p.rows_per_cta = r;
  p.ctas_per_band = std::max(1, (int)(kGsBandCells / ((long long)r * W)));
  p.nctas = (H + r - 1) / r;
  p.nbands = (p.nctas + p.ctas_per_band - 1) / p.ctas_per_band;
  p.bins = cap * p.rb;
  return p;
}

}  // namespace

bool gather_supported(int W, int H, int cap) {
  return cap <= kGatherMaxCap && W >= 2 && W <= 32768 && H <= 16384 && (long long)W * H < (1LL << 31);
}

GatherSizes gather_sizes(int W, int H, int cap, int num_sms) {
  const GsPlan p = make_plan(W, H, cap, num_sms, false);  // the larger of the two layouts
  GatherSizes s;
  s.nbands = p.nbands;
  s.bins = p.bins;
  s.max_ht = (long long)W * H / p.tile + (long long)p.nbands * p.bins + 1;
  return s;
}

cudaError_t launch_direct_gather(const GatherBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                                 int cap, int num_sms, bool tc, bool export_rows, float* act, int32_t* rank,
                                 cudaStream_t st) {
  const GsPlan p = make_plan(g.W, g.H, cap, num_sms, tc);
  const size_t hsmem = (size_t)p.bins * 4;
  cudaError_t e = cudaSuccess;
  if (hsmem > 48 * 1024) {
    e = cudaFuncSetAttribute(k_gs_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gs_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem);
    if (e != cudaSuccess) return e;
  }
  k_gs_count<<<p.nctas, kGsThreads, hsmem, st>>>(g, front, p, cap, b.band_hist, b.tex, export_rows ? rank : nullptr);
  k_gs_scan_band<<<p.nbands, 1024, 0, st>>>(p, b.band_hist, b.goff, b.ght, b.cursor, b.band_tot);
  k_gs_scan_bands<<<1, 1024, 0, st>>>(p, b.band_tot, b.band_base, b.n_ht);
  k_gs_scatter<<<p.nctas, kGsThreads, hsmem, st>>>(g, front, p, cap, b.cursor, b.band_base, b.sorted);
  const long long max_ht = (long long)g.W * g.H / p.tile + (long long)p.nbands * p.bins + 1;
  k_gs_tilemap<<<(unsigned)((max_ht + 255) / 256), 256, 0, st>>>(p, b.goff, b.ght, b.band_base, b.n_ht, b.info);
  GatherArgs a;
  a.net = net;
  a.tex = b.tex;
  a.W = g.W;
  a.sorted = b.sorted;
  a.info = b.info;
  a.n_ht = b.n_ht;
  a.act = act;
  a.export_rows = export_rows ? 1 : 0;
  if (tc)
    k_direct_tc<<<num_sms * 4, kTcThreads, 0, st>>>(a);  // 4 CTAs per SM, 128 TMEM columns each
  else
    k_direct_gather<<<num_sms * 4, kGwThreads, 0, st>>>(a);  // 16 warps per SM, one wave
  return cudaGetLastError();
}

}  // namespace evo
