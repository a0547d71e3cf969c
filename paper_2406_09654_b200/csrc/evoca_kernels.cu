// B200 (sm_100a) kernels for the evoca per-step substrate update.
//
// Pass 1  (k_act_physics)  reference engine.py:193-230 + physics.py:178-309
//   One CTA per 32x32 tile.  The tile plus its 1-cell Moore halo of the five
//   sensed front planes (E, I, C0..C2) is staged in shared memory; occupied
//   cells are bucketed by genome slot inside the CTA (radix sort, groups
//   padded to cell quads) so that each thread evaluates four cells of ONE
//   genome and every weight fetched from L1 feeds four fixed-order fp32 FMA
//   chains.  Sensors are gathered from shared memory in the rotation order
//   PERM[rot] (physics.py:48-62, engine.py:164-177) and never touch HBM.
//   Actions land in shared memory in spatial order; the fused physics tail
//   (energy, invest/liquidate/upkeep/death, communication, explore proposal)
//   then runs in spatial order with coalesced stores.  Physics uses only
//   __f*_rn intrinsics (no FMA contraction) in the reference's op order so
//   that, given the same actions, results are bit-identical to NumPy.
//
// Pass 2  (k_resolve)  reference physics.py:286-343 + 395-404
//   Each target cell PULLS the shipments aimed at it from its 8 neighbours'
//   proposal bytes.  Arrivals are ordered by the packed 64-bit key
//   (bits(q) << 32) | (0xFFFFFFFF - global_source_index), i.e. q descending,
//   source ascending — the reference's lexsort order — and summed
//   sequentially in that order (bit-exact, deterministic, no atomics); the
//   maximal key is the winner, which adopts the target iff q > infra there.
//   The final genome plane feeds a shared-memory census histogram; the last
//   CTA to finish publishes counts and retires slots (neuroevo.py:521-542).

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "evoca_internal.h"

namespace evo {

// Moore offsets (dx, dy) for direction j (physics.py:40-43), packed.
// Halo-tile offset of direction j: dy*kHaloW + dx, stored biased by +64 in a byte.
__host__ __device__ constexpr unsigned long long pack_halo_offsets() {
  const int dx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
  const int dy[8] = {0, 1, 1, 1, 0, -1, -1, -1};
  unsigned long long p = 0;
  for (int j = 0; j < 8; ++j) p |= (unsigned long long)(dy[j] * kHaloW + dx[j] + 64) << (8 * j);
  return p;
}
constexpr unsigned long long kHaloOffPack = pack_halo_offsets();
// rotation_permutation deltas (0, +1, -1, +2, -2, +3, -3, +4) mod 8, 4 bits each.
constexpr unsigned kDeltaPack = (0u << 0) | (1u << 4) | (7u << 8) | (2u << 12) | (6u << 16) | (3u << 20) |
                                (5u << 24) | (4u << 28);
// dx+1 and dy+1 per direction, 4 bits each.
constexpr unsigned kDxPack = (2u << 0) | (2u << 4) | (1u << 8) | (0u << 12) | (0u << 16) | (0u << 20) |
                             (1u << 24) | (2u << 28);
constexpr unsigned kDyPack = (1u << 0) | (2u << 4) | (2u << 8) | (2u << 12) | (1u << 16) | (0u << 20) |
                             (0u << 24) | (0u << 28);

__device__ __forceinline__ int perm_dir(int rot, int slot) {  // PERM_TABLE[rot][slot]
  return (rot + ((kDeltaPack >> (4 * slot)) & 7u)) & 7;
}
__device__ __forceinline__ int halo_off(int dir) {
  return (int)((kHaloOffPack >> (8 * dir)) & 0xFFu) - 64;
}
__device__ __forceinline__ int dir_dx(int d) { return (int)((kDxPack >> (4 * d)) & 0xFu) - 1; }
__device__ __forceinline__ int dir_dy(int d) { return (int)((kDyPack >> (4 * d)) & 0xFu) - 1; }

// Output nonlinearity exactly as hypernet.py:246-251: negate, exp, +1,
// correctly rounded reciprocal, clip to [2^-126, 1-2^-24].
__device__ __forceinline__ float squash(float z) {
  const float e = expf(-z);
  const float d = __fadd_rn(e, 1.0f);
  const float r = __frcp_rn(d);
  return fminf(fmaxf(r, 1.17549435082228750797e-38f), 0.99999994039535522461f);
}

__device__ __forceinline__ long long plane_row(const StepGeom& g, int y) { return (long long)(y + 1) * g.W; }

// ---------------------------------------------------------------------------
// Pass 1

struct Pass1Smem {
  float4 eic[kHaloCells];  // E, I, C0, C1 of tile + halo
  float c2[kHaloCells];    // C2
  int gi[kTileCells];
  uint8_t rot[kTileCells];
  unsigned short order[4 * kTileCells];  // genome-sorted cell list, groups padded to quads
  int n_quads;
  union {
    typename cub::BlockRadixSort<unsigned, kThreads1, 4>::TempStorage sort;
    typename cub::BlockScan<int, kThreads1>::TempStorage scan;
    struct {
      float inv[kTileCells], liq[kTileCells], c0[kTileCells], c1[kTileCells], c2[kTileCells], xmax[kTileCells];
      uint8_t kstar[kTileCells];
    } act;
  } u;
  unsigned last_code[kThreads1 + 1];  // [t+1] = last code held by thread t
  unsigned first_code[kThreads1 + 1]; // [t] = first code held by thread t
};

// Bucket the tile's occupied cells by genome slot; write the padded order.
__device__ void bucket_by_genome(Pass1Smem& sm, int capacity) {
  const int tid = threadIdx.x;
  int nbits = 1;
  while ((1 << nbits) <= capacity) ++nbits;
  unsigned keys[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pos = tid * 4 + i;
    const int g = sm.gi[pos];
    const unsigned code = g >= 0 ? (unsigned)g : (unsigned)capacity;
    keys[i] = (code << 12) | (unsigned)pos;
  }
  cub::BlockRadixSort<unsigned, kThreads1, 4>(sm.u.sort).Sort(keys, 12, 12 + nbits);
  __syncthreads();
  unsigned code[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) code[i] = keys[i] >> 12;
  sm.last_code[tid + 1] = code[3];
  sm.first_code[tid] = code[0];
  if (tid == 0) {
    sm.last_code[0] = 0xFFFFFFFFu;
    sm.first_code[kThreads1] = 0xFFFFFFFFu;
  }
  __syncthreads();
  // group starts (max-scan of start positions) and group-end padding
  int start_in[4], start_of[4];
  unsigned prev = sm.last_code[tid];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    start_in[i] = (code[i] != prev) ? tid * 4 + i : 0;
    prev = code[i];
  }
  cub::BlockScan<int, kThreads1>(sm.u.scan).InclusiveScan(start_in, start_of, cub::Max());
  __syncthreads();
  const unsigned next_code = sm.first_code[tid + 1];
  int pad[4], pad_before[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = tid * 4 + i;
    const unsigned nx = (i < 3) ? code[i + 1] : next_code;
    const bool valid = code[i] < (unsigned)capacity;
    const bool is_end = valid && (nx != code[i]);
    const int size = p - start_of[i] + 1;
    pad[i] = is_end ? ((4 - (size & 3)) & 3) : 0;
  }
  int total_pad;
  cub::BlockScan<int, kThreads1>(sm.u.scan).ExclusiveSum(pad, pad_before, total_pad);
  __syncthreads();
  // count occupied: number of valid codes
  int nvalid = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) nvalid += (code[i] < (unsigned)capacity) ? 1 : 0;
  // order[] is pre-filled with 0xFFFF by the caller
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (code[i] < (unsigned)capacity) sm.order[tid * 4 + i + pad_before[i]] = (unsigned short)(keys[i] & 0xFFFu);
  }
  // the last valid item's padded end gives the list length
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = tid * 4 + i;
    const unsigned nx = (i < 3) ? code[i + 1] : next_code;
    if (code[i] < (unsigned)capacity && !(nx < (unsigned)capacity)) {
      sm.n_quads = (p + pad_before[i] + pad[i] + 1) / 4;
    }
  }
  (void)nvalid;
  (void)total_pad;
}

// Direct 45->13 controller over one quad of same-genome cells.
__device__ __forceinline__ void net_direct_quad(const Pass1Smem& sm, const float* __restrict__ W,
                                                const float* __restrict__ B, const int hb[4], const int rot[4],
                                                float out[4][kActuators]) {
  float acc[4][kActuators];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < kActuators; ++j) acc[c][j] = 0.0f;
#pragma unroll 1
  for (int s = 0; s < 9; ++s) {
    float x[4][5];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int nb = (s == 0) ? hb[c] : hb[c] + halo_off(perm_dir(rot[c], s - 1));
      const float4 v = sm.eic[nb];
      x[c][0] = v.x;
      x[c][1] = v.y;
      x[c][2] = v.z;
      x[c][3] = v.w;
      x[c][4] = sm.c2[nb];
    }
    const float4* wrow = reinterpret_cast<const float4*>(W + (size_t)s * 5 * kOutPad);
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
      const float4 w0 = __ldg(wrow + ch * 4 + 0);
      const float4 w1 = __ldg(wrow + ch * 4 + 1);
      const float4 w2 = __ldg(wrow + ch * 4 + 2);
      const float4 w3 = __ldg(wrow + ch * 4 + 3);
      const float w[13] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w, w3.x};
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < kActuators; ++j) acc[c][j] = fmaf(x[c][ch], w[j], acc[c][j]);
    }
  }
  const float4* b4 = reinterpret_cast<const float4*>(B);
  const float4 b0 = __ldg(b4), b1 = __ldg(b4 + 1), b2 = __ldg(b4 + 2), b3 = __ldg(b4 + 3);
  const float b[13] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w, b3.x};
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int j = 0; j < kActuators; ++j) out[c][j] = squash(__fadd_rn(acc[c][j], b[j]));
}

// Hidden-layer controller 45->H(tanh)->13 for one cell (reference DenseParams).
__device__ __forceinline__ void net_hidden_cell(const Pass1Smem& sm, const Params& P, int g, int hb, int rot,
                                                float out[kActuators]) {
  float x[kSensors];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int nb = (s == 0) ? hb : hb + halo_off(perm_dir(rot, s - 1));
    const float4 v = sm.eic[nb];
    x[s * 5 + 0] = v.x;
    x[s * 5 + 1] = v.y;
    x[s * 5 + 2] = v.z;
    x[s * 5 + 3] = v.w;
    x[s * 5 + 4] = sm.c2[nb];
  }
  float acc[kActuators];
#pragma unroll
  for (int j = 0; j < kActuators; ++j) acc[j] = 0.0f;
  const float* W1 = P.wA + (size_t)g * kSensors * P.hpad;
  const float* B1 = P.bA + (size_t)g * P.hpad;
  const float* W2 = P.wB + (size_t)g * P.hpad * kOutPad;
#pragma unroll 1
  for (int hc = 0; hc < P.hpad; hc += 8) {
    float z[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) z[h] = 0.0f;
#pragma unroll
    for (int k = 0; k < kSensors; ++k) {
      const float4* wr = reinterpret_cast<const float4*>(W1 + (size_t)k * P.hpad + hc);
      const float4 wa = __ldg(wr), wb = __ldg(wr + 1);
      const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int h = 0; h < 8; ++h) z[h] = fmaf(x[k], w[h], z[h]);
    }
    const float4* b4 = reinterpret_cast<const float4*>(B1 + hc);
    const float4 ba = __ldg(b4), bb = __ldg(b4 + 1);
    const float bh[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const float th = tanhf(__fadd_rn(z[h], bh[h]));
      const float4* w2 = reinterpret_cast<const float4*>(W2 + (size_t)(hc + h) * kOutPad);
      const float4 u0 = __ldg(w2), u1 = __ldg(w2 + 1), u2 = __ldg(w2 + 2), u3 = __ldg(w2 + 3);
      const float u[13] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w, u2.x, u2.y, u2.z, u2.w, u3.x};
#pragma unroll
      for (int j = 0; j < kActuators; ++j) acc[j] = fmaf(th, u[j], acc[j]);
    }
  }
  const float4* b4 = reinterpret_cast<const float4*>(P.bB + (size_t)g * kOutPad);
  const float4 b0 = __ldg(b4), b1 = __ldg(b4 + 1), b2 = __ldg(b4 + 2), b3 = __ldg(b4 + 3);
  const float b[13] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w, b3.x};
#pragma unroll
  for (int j = 0; j < kActuators; ++j) out[j] = squash(__fadd_rn(acc[j], b[j]));
}

// first maximal explore actuator (np.argmax: lowest index on ties)
__device__ __forceinline__ void explore_argmax(const float* ex, int& kstar, float& xmax) {
  kstar = 0;
  xmax = ex[0];
#pragma unroll
  for (int k = 1; k < 8; ++k)
    if (ex[k] > xmax) {
      xmax = ex[k];
      kstar = k;
    }
}

template <bool kExport>
__device__ __forceinline__ void store_actions(Pass1Smem& sm, const Pass1Args& a, int p, int x0, int y0,
                                              const float* out) {
  sm.u.act.inv[p] = out[0];
  sm.u.act.liq[p] = out[1];
  sm.u.act.c0[p] = out[2];
  sm.u.act.c1[p] = out[3];
  sm.u.act.c2[p] = out[4];
  int ks;
  float xm;
  explore_argmax(out + 5, ks, xm);
  sm.u.act.xmax[p] = xm;
  sm.u.act.kstar[p] = (uint8_t)ks;
  if (kExport) {
    const int ty = p / kTileW, tx = p - ty * kTileW;
    const long long cell = (long long)(y0 + ty) * a.g.W + (x0 + tx);
    float* dst = a.act_out + cell * kActuators;
#pragma unroll
    for (int j = 0; j < kActuators; ++j) dst[j] = out[j];
    a.act_out_flag[cell] = 1;
  }
}

template <bool kInject, bool kExport, bool kHidden>
__global__ void __launch_bounds__(kThreads1, 2) k_act_physics(const Pass1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pass1Smem& sm = *reinterpret_cast<Pass1Smem*>(smem_raw);
  const StepGeom& g = a.g;
  const int tid = threadIdx.x;
  const int tiles_x = (g.W + kTileW - 1) / kTileW;
  const int x0 = (blockIdx.x % tiles_x) * kTileW;
  const int y0 = (blockIdx.x / tiles_x) * kTileH;
  if (blockIdx.x == 0 && tid == 0 && a.stats) {
    a.stats[0] = 0;
    a.stats[1] = 0;
  }

  // -- stage tile + halo of the sensed front planes (rows -1..H exist: ghosts)
  for (int i = tid; i < kHaloCells; i += kThreads1) {
    const int hy = i / kHaloW, hx = i - hy * kHaloW;
    int y = y0 + hy - 1;
    if (y > g.H) y = g.H;  // beyond a partial tile: never read
    int x = x0 + hx - 1;
    x = x < 0 ? x + g.W : (x >= g.W ? x - g.W : x);
    if (x >= g.W) x = g.W - 1;
    const long long o = plane_row(g, y) + x;
    sm.eic[i] = make_float4(__ldg(a.front.E + o), __ldg(a.front.I + o), __ldg(a.front.C + o),
                            __ldg(a.front.C + g.stride + o));
    sm.c2[i] = __ldg(a.front.C + 2 * g.stride + o);
  }
  for (int i = tid; i < kTileCells; i += kThreads1) {
    const int ty = i / kTileW, tx = i - ty * kTileW;
    const int y = y0 + ty, x = x0 + tx;
    const bool in = (y < g.H) && (x < g.W);
    const long long o = plane_row(g, in ? y : 0) + (in ? x : 0);
    sm.gi[i] = in ? __ldg(a.front.gi + o) : -1;
    sm.rot[i] = in ? __ldg(a.front.rot + o) : 0;
  }
  if (!kInject) {
    for (int i = tid; i < 4 * kTileCells; i += kThreads1) sm.order[i] = 0xFFFF;
    if (tid == 0) sm.n_quads = 0;
  }
  __syncthreads();

  // -- sense + controller, genome-bucketed
  if (!kInject) {
    bucket_by_genome(sm, a.capacity);
    __syncthreads();
    const int nq = sm.n_quads;
    for (int q = tid; q < nq; q += kThreads1) {
      const ushort4 o4 = reinterpret_cast<const ushort4*>(sm.order)[q];
      const unsigned short ord[4] = {o4.x, o4.y, o4.z, o4.w};
      int pos[4], hb[4], rot[4];
      bool valid[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        valid[c] = ord[c] != 0xFFFF;
        pos[c] = valid[c] ? ord[c] : ord[0];
        const int ty = pos[c] / kTileW, tx = pos[c] - ty * kTileW;
        hb[c] = (ty + 1) * kHaloW + tx + 1;
        rot[c] = sm.rot[pos[c]];
      }
      const int slot = sm.gi[pos[0]];
      if (!kHidden) {
        float out[4][kActuators];
        net_direct_quad(sm, a.net.wA + (size_t)slot * kSensors * kOutPad, a.net.bA + (size_t)slot * kOutPad, hb,
                        rot, out);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (valid[c]) store_actions<kExport>(sm, a, pos[c], x0, y0, out[c]);
      } else {
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          if (!valid[c]) continue;
          float out[kActuators];
          net_hidden_cell(sm, a.net, slot, hb[c], rot[c], out);
          store_actions<kExport>(sm, a, pos[c], x0, y0, out);
        }
      }
    }
    __syncthreads();
  }

  // -- fused physics tail in spatial order (physics.py:178-290)
  const Scalars& s = a.s;
  for (int i = tid; i < kTileCells; i += kThreads1) {
    const int ty = i / kTileW, tx = i - ty * kTileW;
    const int y = y0 + ty, x = x0 + tx;
    if (y >= g.H || x >= g.W) continue;
    const long long cell = (long long)y * g.W + x;
    const long long o = plane_row(g, y) + x;
    const int hp = (ty + 1) * kHaloW + tx + 1;
    const float4 f = sm.eic[hp];
    float e = f.x, inf = f.y, c0 = f.z, c1 = f.w, c2 = sm.c2[hp];
    const int slot = sm.gi[i];
    const int r = sm.rot[i];
    bool acted;
    float inv = 0.f, liq = 0.f, m0 = 0.f, m1 = 0.f, m2 = 0.f, xm = 0.f;
    int ks = 0;
    if (kExport && slot < 0) a.act_out_flag[cell] = 0;
    if (kInject) {
      acted = a.act_flag[cell] != 0;
      if (acted) {
        const float* row = a.act_in + cell * kActuators;
        inv = row[0];
        liq = row[1];
        m0 = row[2];
        m1 = row[3];
        m2 = row[4];
        explore_argmax(row + 5, ks, xm);
      }
    } else {
      acted = slot >= 0;
      if (acted) {
        inv = sm.u.act.inv[i];
        liq = sm.u.act.liq[i];
        m0 = sm.u.act.c0[i];
        m1 = sm.u.act.c1[i];
        m2 = sm.u.act.c2[i];
        xm = sm.u.act.xmax[i];
        ks = sm.u.act.kstar[i];
      }
    }
    // energy_cycle: all cells (physics.py:186-194)
    if (a.phases & EVO_PH_ENERGY) {
      if (s.mode == 1) {
        const float add = a.src_map ? __fmul_rn(s.rho, a.src_map[cell]) : s.rho;
        e = __fadd_rn(e, add);
      } else if (s.mode == 2) {
        e = __fsub_rn(e, __fmul_rn(s.drain, e));
      }
    }
    int slot2 = slot;
    // apply_invest_liquidate: listed cells still occupied (physics.py:212-233)
    if ((a.phases & EVO_PH_INVEST) && acted && slot >= 0) {
      const float de = __fmul_rn(inv, fminf(e, s.kinv));
      e = __fsub_rn(e, de);
      inf = __fadd_rn(inf, __fmul_rn(s.einv, de));
      const float di = __fmul_rn(liq, fminf(inf, s.kliq));
      inf = __fsub_rn(inf, di);
      e = __fadd_rn(e, __fmul_rn(s.eliq, di));
      const float cost = __fmul_rn(s.upkeep, inf);
      const bool fed = e >= cost;
      e = fed ? __fsub_rn(e, cost) : 0.0f;
      inf = fed ? inf : __fsub_rn(inf, __fmul_rn(s.dstarve, inf));
      if (inf < s.imin) slot2 = -1;
    }
    // write_communication (physics.py:240-247)
    if (a.phases & EVO_PH_COMM) {
      if (acted && slot2 >= 0) {
        c0 = m0;
        c1 = m1;
        c2 = m2;
      } else if (slot2 < 0) {
        c0 = __fmul_rn(c0, 0.9f);
        c1 = __fmul_rn(c1, 0.9f);
        c2 = __fmul_rn(c2, 0.9f);
      }
    }
    // exploration proposal + withdrawal (physics.py:276-290)
    uint8_t rp = (uint8_t)r;
    float q = 0.0f;
    if ((a.phases & EVO_PH_EXPLORE) && acted && slot2 >= 0) {
      const int dir = perm_dir(r, ks);
      q = __fmul_rn(__fmul_rn(s.alpha, xm), inf);
      inf = __fsub_rn(inf, q);
      rp = (uint8_t)(r | (dir << 3) | kShipBit);
    }
    a.back.E[o] = e;
    a.back.C[o] = c0;
    a.back.C[g.stride + o] = c1;
    a.back.C[2 * g.stride + o] = c2;
    a.mid.I[o] = inf;
    a.mid.gi[o] = slot2;
    a.mid.rp[o] = rp;
    a.mid.q[o] = q;
    if (g.own_ghosts) {
      // wrapped copies for the next pass / step: row 0 -> ghost row H, row H-1 -> ghost row -1
#pragma unroll 1
      for (int rep = 0; rep < 2; ++rep) {
        const bool hit = rep == 0 ? (y == 0) : (y == g.H - 1);
        if (!hit) continue;
        const long long og = plane_row(g, rep == 0 ? g.H : -1) + x;
        a.back.E[og] = e;
        a.back.C[og] = c0;
        a.back.C[g.stride + og] = c1;
        a.back.C[2 * g.stride + og] = c2;
        a.mid.gi[og] = slot2;
        a.mid.rp[og] = rp;
        a.mid.q[og] = q;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 2

template <bool kRecord>
__global__ void __launch_bounds__(kThreads2) k_resolve(const Pass2Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* hist = reinterpret_cast<int*>(smem_raw);
  __shared__ int s_adopt;
  __shared__ bool s_last;
  const StepGeom& g = a.g;
  const int tid = threadIdx.x;
  for (int b = tid; b < a.capacity; b += kThreads2) hist[b] = 0;
  if (tid == 0) s_adopt = 0;
  __syncthreads();

  const long long ncell = (long long)g.W * g.H;
  int my_adopt = 0;
  for (long long cell = (long long)blockIdx.x * kThreads2 + tid; cell < ncell; cell += (long long)gridDim.x * kThreads2) {
    const int y = (int)(cell / g.W);
    const int x = (int)(cell - (long long)y * g.W);
    const long long o = plane_row(g, y) + x;
    const float before = a.mid.I[o];
    const int own = a.mid.gi[o];
    const int r = a.mid.rp[o] & 7;
    unsigned long long key[8];
    int n = 0;
    unsigned long long best = 0;
    int best_d = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const int sy = y - dir_dy(d);
      int sx = x - dir_dx(d);
      sx = sx < 0 ? sx + g.W : (sx >= g.W ? sx - g.W : sx);
      const long long so = plane_row(g, sy) + sx;
      const uint8_t rp = a.mid.rp[so];
      key[d] = 0;
      if ((rp & kShipBit) && ((rp >> 3) & 7) == d) {
        const float qv = __fadd_rn(a.mid.q[so], 0.0f);  // canonical +0
        long long grow = g.row0 + sy;
        if (grow < 0) grow += g.Hg;
        if (grow >= g.Hg) grow -= g.Hg;
        const unsigned gsrc = (unsigned)(grow * g.W + sx);
        key[d] = ((unsigned long long)__float_as_uint(qv) << 32) | (unsigned long long)(0xFFFFFFFFu - gsrc);
        ++n;
        if (key[d] > best) {
          best = key[d];
          best_d = d;
        }
      }
    }
    float acc = before;
    // sequential sum in (q desc, source asc) order (physics.py:294, 321-324)
    for (int it = 0; it < n; ++it) {
      unsigned long long m = 0;
      int md = 0;
#pragma unroll
      for (int d = 0; d < 8; ++d)
        if (key[d] > m) {
          m = key[d];
          md = d;
        }
#pragma unroll
      for (int d = 0; d < 8; ++d)
        if (d == md) key[d] = 0;
      acc = __fadd_rn(acc, __uint_as_float((unsigned)(m >> 32)));
    }
    int gnew = own;
    int rnew = r;
    bool adopt = false;
    if (n > 0) {
      const float qw = __uint_as_float((unsigned)(best >> 32));
      if (qw > before) {
        adopt = true;
        const int sy = y - dir_dy(best_d);
        int sx = x - dir_dx(best_d);
        sx = sx < 0 ? sx + g.W : (sx >= g.W ? sx - g.W : sx);
        gnew = a.mid.gi[plane_row(g, sy) + sx];
        rnew = best_d;
        if (kRecord) {
          a.ev.src[cell] = (long long)(0xFFFFFFFFu - (unsigned)(best & 0xFFFFFFFFu));
          a.ev.q[cell] = qw;
          a.ev.def[cell] = own;
        }
      }
    }
    if (kRecord && !adopt) a.ev.src[cell] = -1;
    my_adopt += adopt ? 1 : 0;
    a.back.I[o] = acc;
    a.back.gi[o] = gnew;
    a.back.rot[o] = (uint8_t)rnew;
    if (g.own_ghosts) {
      if (y == 0) {
        const long long og = plane_row(g, g.H) + x;
        a.back.I[og] = acc;
        a.back.gi[og] = gnew;
        a.back.rot[og] = (uint8_t)rnew;
      }
      if (y == g.H - 1) {
        const long long og = plane_row(g, -1) + x;
        a.back.I[og] = acc;
        a.back.gi[og] = gnew;
        a.back.rot[og] = (uint8_t)rnew;
      }
    }
    if (gnew >= 0 && gnew < a.capacity) atomicAdd(&hist[gnew], 1);
  }
  // block reductions -> global
  for (int off = 16; off > 0; off >>= 1) my_adopt += __shfl_xor_sync(0xffffffffu, my_adopt, off);
  if ((tid & 31) == 0 && my_adopt) atomicAdd(&s_adopt, my_adopt);
  __syncthreads();
  if (tid == 0 && s_adopt) atomicAdd((unsigned long long*)&a.census.stats[0], (unsigned long long)s_adopt);
  for (int b = tid; b < a.capacity; b += kThreads2)
    if (hist[b]) atomicAdd(&a.census.counts[b], hist[b]);
  if (!a.run_census) return;
  // last CTA: census epilogue (physics.py:395-404, neuroevo.py:521-542)
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned ticket = atomicAdd(a.census.done, 1u);
    s_last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  int dead = 0;
  for (int b = tid; b < a.capacity; b += kThreads2) {
    const int c = atomicExch(&a.census.counts[b], 0);
    a.census.counts_last[b] = c;
    if (a.census.state[b] == 1) {
      if (c == 0) {
        a.census.state[b] = 2;
        a.census.death_step[b] = a.t + 1;
        ++dead;
      } else if (c > a.census.peak[b]) {
        a.census.peak[b] = c;
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) dead += __shfl_xor_sync(0xffffffffu, dead, off);
  if ((tid & 31) == 0 && dead) atomicAdd((unsigned long long*)&a.census.stats[1], (unsigned long long)dead);
  if (tid == 0) *a.census.done = 0u;
}

// Census epilogue as its own launch (strip mode: after the cross-rank sum of counts).
__global__ void k_census_finish(const Census c, int capacity, long long t) {
  int dead = 0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < capacity; b += gridDim.x * blockDim.x) {
    const int n = c.counts[b];
    c.counts[b] = 0;
    c.counts_last[b] = n;
    if (c.state[b] == 1) {
      if (n == 0) {
        c.state[b] = 2;
        c.death_step[b] = t + 1;
        ++dead;
      } else if (n > c.peak[b]) {
        c.peak[b] = n;
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) dead += __shfl_xor_sync(0xffffffffu, dead, off);
  if ((threadIdx.x & 31) == 0 && dead) atomicAdd((unsigned long long*)&c.stats[1], (unsigned long long)dead);
}

__global__ void k_refresh_ghosts(const Planes p, const StepGeom g) {
  // single strip: ghost row -1 <- row H-1, ghost row H <- row 0, for E, I, C0..2, gi, rot
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.W; x += gridDim.x * blockDim.x) {
    const long long top = plane_row(g, -1) + x, last = plane_row(g, g.H - 1) + x;
    const long long bot = plane_row(g, g.H) + x, first = plane_row(g, 0) + x;
    p.E[top] = p.E[last];
    p.E[bot] = p.E[first];
    p.I[top] = p.I[last];
    p.I[bot] = p.I[first];
    for (int k = 0; k < 3; ++k) {
      p.C[k * g.stride + top] = p.C[k * g.stride + last];
      p.C[k * g.stride + bot] = p.C[k * g.stride + first];
    }
    p.gi[top] = p.gi[last];
    p.gi[bot] = p.gi[first];
    p.rot[top] = p.rot[last];
    p.rot[bot] = p.rot[first];
  }
}

__global__ void k_scatter_actions(float* act, uint8_t* flag, const int64_t* cells, const float* rows, long long n,
                                  long long ncell) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long c = cells[i];
    if (c < 0 || c >= ncell) continue;
    flag[c] = 1;
    for (int j = 0; j < kActuators; ++j) act[c * kActuators + j] = rows[i * kActuators + j];
  }
}

__global__ void k_patch_genomes(int32_t* gi, int W, const int64_t* cells, const int32_t* slots, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long c = cells[i];
    gi[c + W] = slots[i];  // +W: skip ghost row -1
  }
}

// ---------------------------------------------------------------------------
// launchers

template <bool I, bool E, bool H>
static cudaError_t launch1(const Pass1Args& a, cudaStream_t st) {
  const size_t smem = sizeof(Pass1Smem);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_act_physics<I, E, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = ((a.g.W + kTileW - 1) / kTileW) * ((a.g.H + kTileH - 1) / kTileH);
  k_act_physics<I, E, H><<<tiles, kThreads1, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pass1(const Pass1Args& a, bool inject, bool export_actions, cudaStream_t st) {
  const bool hidden = a.net.hidden > 0;
  if (inject) return launch1<true, false, false>(a, st);
  if (hidden) return export_actions ? launch1<false, true, true>(a, st) : launch1<false, false, true>(a, st);
  return export_actions ? launch1<false, true, false>(a, st) : launch1<false, false, false>(a, st);
}

cudaError_t launch_pass2(const Pass2Args& a, cudaStream_t st) {
  const long long ncell = (long long)a.g.W * a.g.H;
  long long blocks = (ncell + kThreads2 * 4 - 1) / (kThreads2 * 4);
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const size_t smem = (size_t)a.capacity * sizeof(int);
  if (a.ev.src) {
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(k_resolve<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cfg = true;
    }
    k_resolve<true><<<(unsigned)blocks, kThreads2, smem, st>>>(a);
  } else {
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(k_resolve<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cfg = true;
    }
    k_resolve<false><<<(unsigned)blocks, kThreads2, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_census_finish(const Census& c, int capacity, long long t, cudaStream_t st) {
  const int blocks = (capacity + 255) / 256;
  k_census_finish<<<blocks, 256, 0, st>>>(c, capacity, t);
  return cudaGetLastError();
}

cudaError_t launch_refresh_ghosts(const Planes& p, const StepGeom& g, cudaStream_t st) {
  const int blocks = (g.W + 255) / 256;
  k_refresh_ghosts<<<blocks, 256, 0, st>>>(p, g);
  return cudaGetLastError();
}

cudaError_t launch_scatter_actions(float* act, uint8_t* flag, const int64_t* cells, const float* rows, long long n,
                                   long long ncell, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  k_scatter_actions<<<(unsigned)(blocks > 4096 ? 4096 : blocks), 256, 0, st>>>(act, flag, cells, rows, n, ncell);
  return cudaGetLastError();
}

cudaError_t launch_patch_genomes(int32_t* gi, int W, const int64_t* cells, const int32_t* slots, long long n,
                                 cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  k_patch_genomes<<<(unsigned)(blocks > 4096 ? 4096 : blocks), 256, 0, st>>>(gi, W, cells, slots, n);
  return cudaGetLastError();
}

}  // namespace evo
