// Tile staging helpers shared by the persistent pass-1 kernels
// (k_pass1_direct, k_pass1_mma in evoca_kernels.cu; k_pass1_shard in
// evoca_shard.cu): the 32x32 tile plus its 1-cell Moore halo of the five
// sensed front planes, loaded into registers a tile ahead and committed to
// shared memory as interleaved float4 {E, I, C0, C1} + C2.
#pragma once

#include "evoca_net.cuh"

namespace evo {

// Halo cell i of the tile at (x0, y0): global plane offset (rows -1..H exist).
__device__ __forceinline__ unsigned halo_src(const StepGeom& g, int x0, int y0, int i) {
  const int hy = i / kHaloW, hx = i - hy * kHaloW;
  int y = y0 + hy - 1;
  if (y > g.H) y = g.H;  // beyond a partial tile: never read
  int x = x0 + hx - 1;
  x = x < 0 ? x + g.W : (x >= g.W ? x - g.W : x);
  if (x >= g.W) x = g.W - 1;
  return (unsigned)((y + 1) * g.W + x);
}

template <int THREADS>
struct PrefetchT {
  static constexpr int kHalo = (kHaloCells + THREADS - 1) / THREADS;
  static constexpr int kCells = (kTileCells + THREADS - 1) / THREADS;
  float v[kHalo][5];
  int gi[kCells];
  int rot[kCells];
};

template <int THREADS>
__device__ __forceinline__ void prefetch_tile(const Pass1Args& a, int tile, int tiles_x, PrefetchT<THREADS>& pf) {
  constexpr int kPreHalo = PrefetchT<THREADS>::kHalo, kPreCells = PrefetchT<THREADS>::kCells;
  const StepGeom& g = a.g;
  const int tid = threadIdx.x;
  const int x0 = (tile % tiles_x) * kTileW;
  const int y0 = (tile / tiles_x) * kTileH;
  const unsigned st = (unsigned)g.stride;
#pragma unroll
  for (int j = 0; j < kPreHalo; ++j) {
    const int i = tid + j * THREADS;
    if (i < kHaloCells) {
      const unsigned o = halo_src(g, x0, y0, i);
      pf.v[j][0] = ld_na(a.front.E + o);
      pf.v[j][1] = ld_na(a.front.I + o);
      pf.v[j][2] = ld_na(a.front.C + o);
      pf.v[j][3] = ld_na(a.front.C + st + o);
      pf.v[j][4] = ld_na(a.front.C + 2 * st + o);
    }
  }
#pragma unroll
  for (int j = 0; j < kPreCells; ++j) {
    const int i = tid + j * THREADS;
    const int ty = i / kTileW, tx = i - ty * kTileW;
    const int y = y0 + ty, x = x0 + tx;
    const bool in = (i < kTileCells) && (y < g.H) && (x < g.W);
    const unsigned o = in ? (unsigned)((y + 1) * g.W + x) : 0u;
    pf.gi[j] = in ? __ldg(a.front.gi + o) : -1;
    pf.rot[j] = in ? (int)__ldg(a.front.rot + o) : 0;
  }
}

template <int THREADS, typename SM>
__device__ __forceinline__ void commit_tile(SM& sm, const PrefetchT<THREADS>& pf) {
  constexpr int kPreHalo = PrefetchT<THREADS>::kHalo, kPreCells = PrefetchT<THREADS>::kCells;
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < kPreHalo; ++j) {
    const int i = tid + j * THREADS;
    if (i < kHaloCells) {
      sm.eic[i] = make_float4(pf.v[j][0], pf.v[j][1], pf.v[j][2], pf.v[j][3]);
      sm.c2[i] = pf.v[j][4];
    }
  }
#pragma unroll
  for (int j = 0; j < kPreCells; ++j) {
    const int i = tid + j * THREADS;
    if (i < kTileCells) {
      sm.gi[i] = pf.gi[j];
      sm.rot[i] = (uint8_t)pf.rot[j];
    }
  }
}

// L2 prefetch of a tile's halo rows (5 planes) and interior genome/rotation
// rows: no registers, issued a whole tile ahead of the register loads.
template <int THREADS>
__device__ __forceinline__ void prefetch_tile_l2(const Pass1Args& a, int tile, int tiles_x) {
  const StepGeom& g = a.g;
  const int x0 = (tile % tiles_x) * kTileW;
  const int y0 = (tile / tiles_x) * kTileH;
  // per plane row: [x0-1, x0+33) -> at most 2 x 128-byte lines (floats)
  constexpr int kLines = kHaloH * 2;  // per float plane
  for (int i = threadIdx.x; i < kLines * 5 + kTileH * 2; i += THREADS) {
    const char* p;
    if (i < kLines * 5) {
      const int plane = i / kLines, r = (i - plane * kLines) >> 1, half = i & 1;
      int y = y0 + r - 1;
      if (y > g.H) y = g.H;
      int x = x0 - 1 + half * 32;
      x = x < 0 ? 0 : (x >= g.W ? g.W - 1 : x);
      const float* base = plane == 0 ? a.front.E : (plane == 1 ? a.front.I : a.front.C + (plane - 2) * g.stride);
      p = reinterpret_cast<const char*>(base + (unsigned)((y + 1) * g.W + x));
    } else {
      const int j = i - kLines * 5, r = j >> 1;
      int y = y0 + r;
      if (y >= g.H) y = g.H - 1;
      p = (j & 1) ? reinterpret_cast<const char*>(a.front.rot + (unsigned)((y + 1) * g.W + x0))
                  : reinterpret_cast<const char*>(a.front.gi + (unsigned)((y + 1) * g.W + x0));
    }
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}

// Asynchronous copy of the slot weight tables into shared memory (16-byte cp.async).
template <int THREADS>
__device__ __forceinline__ void stage_weights(float* dst, const float* src, int nfloats) {
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(dst);
  for (int i = threadIdx.x * 4; i < nfloats; i += THREADS * 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + i * 4), "l"(src + i));
}


}  // namespace evo
