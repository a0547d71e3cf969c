// B200 (sm_100a) kernels for the evoca per-step substrate update.
//
// Pass 1 (reference engine.py:193-230 + physics.py:178-309): sense, controller
// and the fused physics tail, per 32x32 tile.  The tile plus its 1-cell Moore
// halo of the five sensed front planes (E, I, C0..C2) is staged in shared
// memory; occupied cells are bucketed by genome slot inside the CTA (counting
// sort, each genome group padded to an even number of two-cell units) so
// that each thread evaluates two cells of ONE genome and every weight loaded
// feeds two fixed-order fp32 FMA chains.  Sensors are gathered from shared
// memory in the rotation order PERM[rot] (physics.py:48-62,
// engine.py:164-177) and never touch HBM.  Actions land in shared memory in
// spatial order; the physics tail then runs in spatial order with coalesced
// stores, using only __f*_rn intrinsics (no FMA contraction) in the
// reference's op order so that, given the same actions, results are
// bit-identical to NumPy.
//   k_pass1_direct  hot path (direct 45->13 net, pools <= 68 slots):
//                   persistent CTA per SM, weight table resident in shared
//                   memory, packed FFMA2 (fma.rn.f32x2), next tile's halo
//                   prefetched into L2 and registers during compute.
//   k_pass1_generic injected actions (parity tier A / the phase-function API)
//                   and the CUDA-core 45->H(tanh)->13 net.
//   k_physics_rows  physics of the genome-sorted paths (evoca_hidden_tc.cu).
//
// Pass 2 (k_resolve, physics.py:286-343 + 395-404): each target cell PULLS
// the shipments aimed at it from its 8 neighbours' one-hot proposal bytes.
// Arrivals are ordered by the packed 64-bit key (bits(q) << 32) | (0xFFFFFFFF -
// global_source_index), i.e. q descending then source ascending - the
// reference's lexsort order - and summed sequentially in that order
// (bit-exact, deterministic, no atomics); the maximal key is the winner,
// which adopts the target iff q > infra standing there.  The final genome
// plane feeds a shared-memory census histogram; the last CTA to finish
// publishes counts and retires slots (neuroevo.py:521-542).

#include <algorithm>

#include "evoca_gather.cuh"
#include "evoca_tile.cuh"

namespace evo {

// Optional per-phase cycle accounting of the hot pass-1 kernel (diagnostics
// build: -DEVO_PHASE_TIMING; read with evo_debug_phase_cycles).
__device__ unsigned long long g_phase_cycles[8];
#ifdef EVO_PHASE_TIMING
#define PHASE_MARK(k)                                               \
  if (threadIdx.x == 0) {                                           \
    const long long now = clock64();                                \
    atomicAdd(&g_phase_cycles[k], (unsigned long long)(now - t_mark)); \
    t_mark = now;                                                   \
  }
#else
#define PHASE_MARK(k)
#endif

__device__ __forceinline__ void zero_stats(const Pass1Args& a) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.stats) {
    a.stats[0] = 0;
    a.stats[1] = 0;
  }
}

// Pass 1 of the genome-sorted paths (tensor-core hidden nets, large-pool
// direct nets): the actions already sit in rank-ordered rows, so the physics
// tail runs per cell straight from the planes - coalesced state reads, one
// 64-byte actuator row read per occupied cell, coalesced stores - with no
// shared-memory staging.
__device__ __forceinline__ CellAct row_actions(const Pass1Args& a, int r) {
  CellAct ac{};
  ac.acted = r >= 0;
  if (ac.acted && a.act_decided) {  // one 32-byte sector at the cell index: {inv, liq, m0, m1, m2, xmax, kstar, 0}
    float v[8];
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(a.act_in + (size_t)r * 8));
    ac.inv = v[0];
    ac.liq = v[1];
    ac.m0 = v[2];
    ac.m1 = v[3];
    ac.m2 = v[4];
    ac.xmax = v[5];
    ac.kstar = __float_as_int(v[6]);
  } else if (ac.acted) {
    const float4* row = reinterpret_cast<const float4*>(a.act_in + (size_t)r * 16);
    const float4 r0 = __ldg(row), r1 = __ldg(row + 1), r2 = __ldg(row + 2), r3 = __ldg(row + 3);
    ac.inv = r0.x;
    ac.liq = r0.y;
    ac.m0 = r0.z;
    ac.m1 = r0.w;
    ac.m2 = r1.x;
    const float ex[8] = {r1.y, r1.z, r1.w, r2.x, r2.y, r2.z, r2.w, r3.x};
    explore_argmax(ex, ac.kstar, ac.xmax);
  }
  return ac;
}

// Four consecutive cells per thread (W % 4 == 0): 16-byte plane loads and
// stores, one load instruction per plane per four cells (the per-cell
// version was LSU-queue bound: lg_throttle 28 %, long_scoreboard 60 %).
// Direct nets write their decided records at the cell's own index, so those
// reads are coalesced too (rows at the sorted rank made this kernel
// gather-bound: long_scoreboard 83 %).
__global__ void __launch_bounds__(256) k_physics_rows(const Pass1Args a) {
  zero_stats(a);
  const StepGeom& g = a.g;
  const int n = g.W * g.H;
  const unsigned st = (unsigned)g.stride;
  if ((g.W & 3) == 0) {
    for (int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4; c0 < n; c0 += gridDim.x * blockDim.x * 4) {
      const int y = c0 / g.W, x = c0 - y * g.W;
      const unsigned o = (unsigned)((y + 1) * g.W + x);
      const float4 E = __ldg(reinterpret_cast<const float4*>(a.front.E + o));
      const float4 I = __ldg(reinterpret_cast<const float4*>(a.front.I + o));
      const float4 C0 = __ldg(reinterpret_cast<const float4*>(a.front.C + o));
      const float4 C1 = __ldg(reinterpret_cast<const float4*>(a.front.C + st + o));
      const float4 C2 = __ldg(reinterpret_cast<const float4*>(a.front.C + 2 * st + o));
      const int4 G = __ldg(reinterpret_cast<const int4*>(a.front.gi + o));
      const unsigned R = __ldg(reinterpret_cast<const unsigned*>(a.front.rot + o));
      const int4 RK = a.act_decided ? make_int4(G.x >= 0 ? c0 : -1, G.y >= 0 ? c0 + 1 : -1, G.z >= 0 ? c0 + 2 : -1,
                                                G.w >= 0 ? c0 + 3 : -1)
                                    : __ldg(reinterpret_cast<const int4*>(a.act_rank + c0));
      const float e[4] = {E.x, E.y, E.z, E.w}, in[4] = {I.x, I.y, I.z, I.w};
      const float c0v[4] = {C0.x, C0.y, C0.z, C0.w}, c1v[4] = {C1.x, C1.y, C1.z, C1.w},
                  c2v[4] = {C2.x, C2.y, C2.z, C2.w};
      const int gv[4] = {G.x, G.y, G.z, G.w}, rk[4] = {RK.x, RK.y, RK.z, RK.w};
      CellOut out[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const CellState cs{e[j], in[j], c0v[j], c1v[j], c2v[j], gv[j], (int)((R >> (8 * j)) & 0xFFu)};
        out[j] = cell_physics(a.s, a.phases, a.src_map, c0 + j, cs, row_actions(a, rk[j]));
      }
      if (g.own_ghosts && (y == 0 || y == g.H - 1)) {  // seam rows: per-cell stores with the wrapped copies
#pragma unroll
        for (int j = 0; j < 4; ++j) store_pass1(a, y, x + j, out[j]);
        continue;
      }
      *reinterpret_cast<float4*>(a.back.E + o) = make_float4(out[0].e, out[1].e, out[2].e, out[3].e);
      *reinterpret_cast<float4*>(a.back.C + o) = make_float4(out[0].c0, out[1].c0, out[2].c0, out[3].c0);
      *reinterpret_cast<float4*>(a.back.C + st + o) = make_float4(out[0].c1, out[1].c1, out[2].c1, out[3].c1);
      *reinterpret_cast<float4*>(a.back.C + 2 * st + o) = make_float4(out[0].c2, out[1].c2, out[2].c2, out[3].c2);
      *reinterpret_cast<float4*>(a.mid.I + o) = make_float4(out[0].inf, out[1].inf, out[2].inf, out[3].inf);
      *reinterpret_cast<int4*>(a.mid.gi + o) = make_int4(out[0].slot, out[1].slot, out[2].slot, out[3].slot);
      *reinterpret_cast<unsigned*>(a.mid.rp + o) =
          (unsigned)out[0].rp | ((unsigned)out[1].rp << 8) | ((unsigned)out[2].rp << 16) | ((unsigned)out[3].rp << 24);
      *reinterpret_cast<float4*>(a.mid.q + o) = make_float4(out[0].q, out[1].q, out[2].q, out[3].q);
    }
    return;
  }
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int y = c / g.W, x = c - y * g.W;
    const unsigned o = (unsigned)((y + 1) * g.W + x);
    const CellState cs{__ldg(a.front.E + o), __ldg(a.front.I + o), __ldg(a.front.C + o),
                       __ldg(a.front.C + st + o), __ldg(a.front.C + 2 * st + o), __ldg(a.front.gi + o),
                       (int)__ldg(a.front.rot + o)};
    const int r = a.act_decided ? (cs.slot >= 0 ? c : -1) : __ldg(a.act_rank + c);
    store_pass1(a, y, x, cell_physics(a.s, a.phases, a.src_map, c, cs, row_actions(a, r)));
  }
}

// Physics tail of one tile in spatial order (shared by both pass-1 kernels).
template <bool kInject, bool kExport, int THREADS, typename SM>
__device__ __forceinline__ void tile_physics(const Pass1Args& a, const SM& sm, int x0, int y0) {
  const StepGeom& g = a.g;
#pragma unroll 1
  for (int i = threadIdx.x; i < kTileCells; i += THREADS) {
    const int ty = i / kTileW, tx = i - ty * kTileW;
    const int y = y0 + ty, x = x0 + tx;
    if (y >= g.H || x >= g.W) continue;
    const long long cell = (long long)y * g.W + x;
    const int hp = (ty + 1) * kHaloW + tx + 1;
    const float4 f = sm.eic[hp];
    CellState st{f.x, f.y, f.z, f.w, sm.c2[hp], sm.gi[i], sm.rot[i]};
    CellAct ac{};
    if (kExport && st.slot < 0) a.act_out_flag[cell] = 0;
    if (kInject) {
      const float* row;
      if (a.act_rank) {  // rows of the genome-sorted paths, 16 floats each
        const int r = a.act_rank[cell];
        ac.acted = r >= 0;
        row = a.act_in + (size_t)(r >= 0 ? r : 0) * 16;
      } else {
        ac.acted = a.act_flag[cell] != 0;
        row = a.act_in + cell * kActuators;
      }
      if (ac.acted) {
        ac.inv = row[0];
        ac.liq = row[1];
        ac.m0 = row[2];
        ac.m1 = row[3];
        ac.m2 = row[4];
        explore_argmax(row + 5, ac.kstar, ac.xmax);
      }
    } else {
      ac.acted = st.slot >= 0;
      if (ac.acted) {
        ac.inv = sm.u.act.inv[i];
        ac.liq = sm.u.act.liq[i];
        ac.m0 = sm.u.act.c0[i];
        ac.m1 = sm.u.act.c1[i];
        ac.m2 = sm.u.act.c2[i];
        ac.xmax = sm.u.act.xmax[i];
        ac.kstar = sm.u.act.kstar[i];
      }
    }
#ifdef EVO_DIAG_NO_STORE  // diagnostics builds only: results are wrong
    const CellOut o = cell_physics(a.s, a.phases, a.src_map, cell, st, ac);
    if (__float_as_uint(o.e) == 0x7fc00001u + (unsigned)a.g.W) store_pass1(a, y, x, o);
#else
    store_pass1(a, y, x, cell_physics(a.s, a.phases, a.src_map, cell, st, ac));
#endif
  }
}

// Unit loop of the controller over the bucketed tile (U cells per thread).
template <bool kExport, bool kHidden, int THREADS, int U, bool kSmemW = false, typename SM>
__device__ __forceinline__ void tile_controller(const Pass1Args& a, SM& sm, int x0, int y0,
                                                const float* W12 = nullptr, const float* W1 = nullptr,
                                                const float* B = nullptr) {
  if (!kSmemW) {
    W12 = a.net.wA;
    W1 = a.net.wB;
    B = a.net.bA;
  }
#ifdef EVO_DIAG_NO_CTRL  // diagnostics builds only (no controller work): results are wrong
  const int nu = a.g.W < 0 ? sm.n_units : 0;
#else
  const int nu = sm.n_units;
#endif
  for (int q = threadIdx.x; q < nu; q += THREADS) {
    unsigned short ord[U];
    if constexpr (U % 2 == 0) {
#pragma unroll
      for (int c = 0; c < U; c += 2) {  // order entries are 16-bit, read in 32-bit pairs
        const unsigned w = reinterpret_cast<const unsigned*>(sm.order)[(q * U + c) >> 1];
        ord[c] = (unsigned short)(w & 0xFFFFu);
        ord[c + 1] = (unsigned short)(w >> 16);
      }
    } else {
#pragma unroll
      for (int c = 0; c < U; ++c) ord[c] = sm.order[q * U + c];
    }
    if (ord[0] == 0xFFFF) continue;  // a pure padding unit (groups padded past U cells)
    int pos[U], hb[U], rot[U];
    bool valid[U];
#pragma unroll
    for (int c = 0; c < U; ++c) {
      valid[c] = ord[c] != 0xFFFF;
      pos[c] = valid[c] ? ord[c] : ord[0];
      const int ty = pos[c] / kTileW, tx = pos[c] - ty * kTileW;
      hb[c] = (ty + 1) * kHaloW + tx + 1;
      rot[c] = sm.rot[pos[c]];
    }
    const int slot = sm.gi[pos[0]];
#ifdef EVO_PHASE_TIMING
    {  // diagnostics: distinct genome slots per warp-iteration of the unit loop
      const unsigned act = __activemask();
      const unsigned grp = __match_any_sync(act, slot);
      if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&g_phase_cycles[6], 1ull);
      if ((threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(&g_phase_cycles[7], 1ull);
    }
#endif
    if (!kHidden) {
      float out[U][kActuators];
      net_direct_unit<U, kSmemW>(sm, W12 + (size_t)slot * kSensors * 12, W1 + (size_t)slot * kSensors,
                                 B + (size_t)slot * kOutPad, hb, rot, out);
#pragma unroll
      for (int c = 0; c < U; ++c)
        if (valid[c]) finish_actions<kExport>(sm.u.act, a, pos[c], x0, y0, out[c]);
    } else {
#pragma unroll 1
      for (int c = 0; c < U; ++c) {
        if (!valid[c]) continue;
        float out[kActuators];
        net_hidden_cell(sm, a.net, slot, hb[c], rot[c], out);
        finish_actions<kExport>(sm.u.act, a, pos[c], x0, y0, out);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 1, generic (injected actions / hidden-layer net / export)

struct GenericSmem {
  float4 eic[kHaloCells];
  float c2[kHaloCells];
  int gi[kTileCells];
  uint8_t rot[kTileCells];
  unsigned short order[4 * kTileCells];
  int slot_off[72];
  int scratch[kThreads1 / 32];
  int n_units;
  union {
    ActSmem act;
  } u;
  int bins[1];  // capacity ints (dynamic tail)
};

template <bool kInject, bool kExport, bool kHidden>
__global__ void __launch_bounds__(kThreads1, 2) k_pass1_generic(const Pass1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GenericSmem& sm = *reinterpret_cast<GenericSmem*>(smem_raw);
  const StepGeom& g = a.g;
  const int tid = threadIdx.x;
  const int tiles_x = (g.W + kTileW - 1) / kTileW;
  const int x0 = (blockIdx.x % tiles_x) * kTileW;
  const int y0 = (blockIdx.x / tiles_x) * kTileH;
  zero_stats(a);
  fill_slot_offsets(sm.slot_off);
  for (int i = tid; i < kHaloCells; i += kThreads1) {
    const unsigned o = halo_src(g, x0, y0, i);
    sm.eic[i] = make_float4(__ldg(a.front.E + o), __ldg(a.front.I + o), __ldg(a.front.C + o),
                            __ldg(a.front.C + g.stride + o));
    sm.c2[i] = __ldg(a.front.C + 2 * g.stride + o);
  }
  for (int i = tid; i < kTileCells; i += kThreads1) {
    const int ty = i / kTileW, tx = i - ty * kTileW;
    const int y = y0 + ty, x = x0 + tx;
    const bool in = (y < g.H) && (x < g.W);
    const unsigned o = in ? (unsigned)((y + 1) * g.W + x) : 0u;
    sm.gi[i] = in ? __ldg(a.front.gi + o) : -1;
    sm.rot[i] = in ? __ldg(a.front.rot + o) : 0;
  }
  __syncthreads();
  if (!kInject) {
    bucket_by_genome<kThreads1, kTileCells / kThreads1, 4>(sm.bins, sm.scratch, sm.gi, sm.order, &sm.n_units,
                                                           a.capacity);
    tile_controller<kExport, kHidden, kThreads1, 4>(a, sm, x0, y0);
    __syncthreads();
  }
  tile_physics<kInject, kExport, kThreads1>(a, sm, x0, y0);
}

// ---------------------------------------------------------------------------
// Pass 1, hot path: persistent, direct net, FFMA2

constexpr int kThreadsP = 640;  // >= units of a tile for pools <= 64 slots: one controller round
#ifndef EVO_UNIT_CELLS
#define EVO_UNIT_CELLS 2
#endif
constexpr int kUnitP = EVO_UNIT_CELLS;  // cells per thread in the controller (same genome)
constexpr int kPreCells = (kTileCells + kThreadsP - 1) / kThreadsP;

struct DirectSmem {
  float4 eic[kHaloCells];
  float c2[kHaloCells];
  int gi[kTileCells];
  uint8_t rot[kTileCells];
  unsigned short order[4 * kTileCells];
  int slot_off[72];
  int scratch[kThreadsP / 32];
  int n_units;
  union {
    ActSmem act;
  } u;
  int bins[1];  // capacity ints (dynamic tail)
};

using Prefetch = PrefetchT<kThreadsP>;

template <bool kExport, bool kSmemW>
__global__ void __launch_bounds__(kThreadsP, 1) k_pass1_direct(const Pass1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DirectSmem& sm = *reinterpret_cast<DirectSmem*>(smem_raw);
  const StepGeom& g = a.g;
  const int tiles_x = (g.W + kTileW - 1) / kTileW;
  const int ntiles = tiles_x * ((g.H + kTileH - 1) / kTileH);
  zero_stats(a);
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  // weight tables resident in shared memory for small pools: W12 | W1 | bias
  float* sW12 = nullptr;
  float* sW1 = nullptr;
  float* sB = nullptr;
  if (kSmemW) {
    const size_t off = (sizeof(DirectSmem) + (size_t)a.capacity * sizeof(int) + 15) & ~(size_t)15;
    sW12 = reinterpret_cast<float*>(smem_raw + off);
    sW1 = sW12 + (size_t)a.capacity * kSensors * 12;
    sB = sW1 + (((size_t)a.capacity * kSensors + 3) & ~(size_t)3);
    stage_weights<kThreadsP>(sW12, a.net.wA, a.capacity * kSensors * 12);
    stage_weights<kThreadsP>(sW1, a.net.wB, (a.capacity * kSensors + 3) & ~3);
    stage_weights<kThreadsP>(sB, a.net.bA, a.capacity * kOutPad);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  fill_slot_offsets(sm.slot_off);
  int rank[kPreCells];
  {
    Prefetch pf;
    prefetch_tile(a, tile, tiles_x, pf);
    commit_tile(sm, pf);
    for (int b = threadIdx.x; b < a.capacity; b += kThreadsP) sm.bins[b] = 0;
    __syncthreads();
    bucket_count<kThreadsP, kPreCells>(sm.bins, pf.gi, rank);
    __syncthreads();
    bucket_offsets<kThreadsP, 2 * kUnitP, kUnitP>(sm.bins, sm.scratch, sm.order, &sm.n_units, a.capacity);
    __syncthreads();
    bucket_scatter<kThreadsP, kPreCells>(sm.bins, pf.gi, rank, sm.order);
  }
  __syncthreads();
  long long t_mark = clock64();
  (void)t_mark;
  PHASE_MARK(4);
  // Per tile: controller | physics + next tile's genome count (from its
  // prefetch registers) | offsets | scatter + halo commit of the next tile.
  for (; tile < ntiles; tile += gridDim.x) {
    const int x0 = (tile % tiles_x) * kTileW;
    const int y0 = (tile / tiles_x) * kTileH;
    const int next = tile + gridDim.x;
    if (next < ntiles) prefetch_tile_l2<kThreadsP>(a, next, tiles_x);
    for (int b = threadIdx.x; b < a.capacity; b += kThreadsP) sm.bins[b] = 0;  // for the next count
    if (kSmemW && tile == (int)blockIdx.x) {  // weight staging overlapped the first halo load + bucketing
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    PHASE_MARK(0);
    tile_controller<kExport, false, kThreadsP, kUnitP, kSmemW>(a, sm, x0, y0, sW12, sW1, sB);
    __syncthreads();
    PHASE_MARK(1);
    Prefetch pf;
    if (next < ntiles) prefetch_tile(a, next, tiles_x, pf);  // L2 hits by now
    tile_physics<false, kExport, kThreadsP>(a, sm, x0, y0);
    if (next < ntiles) bucket_count<kThreadsP, kPreCells>(sm.bins, pf.gi, rank);
    __syncthreads();
    PHASE_MARK(2);
    if (next < ntiles) {
      bucket_offsets<kThreadsP, 2 * kUnitP, kUnitP>(sm.bins, sm.scratch, sm.order, &sm.n_units, a.capacity);
      __syncthreads();
      bucket_scatter<kThreadsP, kPreCells>(sm.bins, pf.gi, rank, sm.order);
      commit_tile(sm, pf);
    }
    __syncthreads();
    PHASE_MARK(3);
  }
}

// Largest pool whose weight tables fit in shared memory next to the tile.
constexpr int kSmemWeightSlots = kSmemWeightSlotsAbi;
constexpr size_t weight_smem_bytes(int capacity) {
  return ((size_t)capacity * (kSensors * 12 + kOutPad) + (((size_t)capacity * kSensors + 3) & ~(size_t)3)) * sizeof(float);
}

// ---------------------------------------------------------------------------
// Pass 1, direct net as mma.sync m16n8k8 TF32 (EVO_F_MMA_NET; a measured
// alternative, not the default: on config 2 it runs the step in 157 us against
// the FFMA2 kernel's 115 us - 81M warp instructions per launch against 43M,
// because per 8-cell block every lane splits its 12 sensor values, computes 12
// rotated addresses and squashes 2-4 outputs, ~3x the sigmoid evaluations of
// the pruned per-cell epilogue)
//
// The 45->13 contraction of an 8-cell block of one genome is D[16 x 8] =
// W[16 outputs x 48] . S[48 x 8 cells]: outputs on M (13 of 16 rows used),
// cells on N, so genome groups are padded to 8 cells (not 16).  fp32
// accuracy from the 3xTF32 split x = hi + lo: hi.hi into one accumulator
// (bias-initialised), hi.lo + lo.hi into a second, summed in FP32 (the TF32
// MMA accumulates with worse than FP32 rounding, tools/microbench/tc_split.cu).
// The K order is permuted so that lane (r = lane/4, q = lane%4) loads
// channel q of the 9 Moore slots straight from the interleaved halo tile
// (one 16-byte {E, I, C0, C1} chunk per cell and slot is read by the cell's
// four lanes) plus three C2 values:
//   K-steps 0-3: rows 8j+q -> slot 2j channel q, 8j+4+q -> slot 2j+1 channel q
//   K-step 4:    32+q -> slot 8 channel q,      36+q -> slot q channel C2
//   K-step 5:    40+q -> slot 4+q channel C2,   44+q -> slot 8 C2 (q = 0), pad
// Weights live in shared memory in A-fragment order (k_frag_relayout), loaded
// into registers (split hi/lo) when a warp's block changes genome; warps walk
// contiguous ranges of blocks.  Epilogue: each lane squashes its outputs (the
// reference sigmoid sequence), the explore argmax (first-max over squashed
// values) is a 3-step shuffle reduction over the 8 lanes of a cell pair.

constexpr int kThreadsM = 512;
constexpr int kWarpsM = kThreadsM / 32;
constexpr int kOrderM = (kTileCells + kMmaSlots * 7 + 7) & ~7;

struct MmaSmem {
  float4 eic[kHaloCells];
  float c2[kHaloCells];
  int gi[kTileCells];
  uint8_t rot[kTileCells];
  unsigned short order[kOrderM];
  int scratch[kThreadsM / 32];
  int n_units;
  union {
    ActSmem act;
  } u;
  int bins[kMmaSlots];
};

// logical K row -> physical sensor index slot*5 + channel (-1: padding)
__host__ __device__ constexpr int mma_k_phys(int kk) {
  const int j = kk >> 3, h = (kk >> 2) & 1, q = kk & 3;
  return j < 4 ? (2 * j + h) * 5 + q
               : (j == 4 ? (h == 0 ? 40 + q : q * 5 + 4) : (h == 0 ? (4 + q) * 5 + 4 : (q == 0 ? 44 : -1)));
}

// Compact direct weights (W12 [cap][45][12], W1 [cap][45], bias [cap][16])
// -> fragment-order table [cap][kFragGenome].
__global__ void k_frag_relayout(const Params net, int capacity, float* wF) {
  const int n = capacity * kFragGenome;
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const int g = d / kFragGenome, e = d - g * kFragGenome;
    float v = 0.0f;
    if (e >= 6 * kFragStep) {
      v = net.bA[(size_t)g * kOutPad + (e - 6 * kFragStep)];
    } else {
      const int j = e / kFragStep, r2 = e - j * kFragStep;
      int lane, comp;
      if (r2 < 80) {
        lane = r2 >> 2;
        comp = r2 & 3;
      } else {
        lane = 20 + ((r2 - 80) >> 1);
        comp = ((r2 - 80) & 1) * 2;  // a0, a2
      }
      const int o = (lane >> 2) + ((comp & 1) ? 8 : 0);
      const int kk = 8 * j + (lane & 3) + ((comp & 2) ? 4 : 0);
      const int ph = mma_k_phys(kk);
      if (ph >= 0 && o < kActuators)
        v = o < 12 ? net.wA[((size_t)g * kSensors + ph) * 12 + o] : net.wB[(size_t)g * kSensors + ph];
    }
    wF[d] = v;
  }
}

// x = hi + lo with hi exactly TF32 (11 significant bits, rounded to nearest)
// by Veltkamp splitting on the FMA pipe (cvt.rna.tf32 runs on the slow XU
// pipe, which bound the first version of this kernel): t = x * (2^13 + 1),
// hi = t - (t - x), lo = x - hi exact (<= 12 significant bits; the MMA reads
// its top 11, an error <= 2^-22 |x|).
__device__ __forceinline__ void split_tf32(float x, unsigned& hi, unsigned& lo) {
  const float t = __fmul_rn(x, 8193.0f);
  const float h = __fsub_rn(t, __fsub_rn(t, x));
  hi = __float_as_uint(h);
  lo = __float_as_uint(__fsub_rn(x, h));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float lds_f32(unsigned addr) {
  float r;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(addr));
  return r;
}

// halo-tile offset (biased by +64) of Moore slot s for rotation rot, from the
// byte-rotated direction pack
__device__ __forceinline__ unsigned long long rotated_offsets(int rot) {
  const unsigned long long p = kHaloOffPack;
  const int sh = 8 * rot;
  return sh ? (p >> sh) | (p << (64 - sh)) : p;
}

template <bool kExport>
__device__ __forceinline__ void tile_controller_mma(const Pass1Args& a, MmaSmem& sm, const float* sF, int x0,
                                                    int y0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int nblk = sm.n_units;
  const int b_begin = warp * nblk / kWarpsM, b_end = (warp + 1) * nblk / kWarpsM;
  // lane constants: rotation deltas of C2 slots q and 4+q (slot 0 has none)
  const int dq1 = (int)((kDeltaPack >> (4 * ((q + 7) & 7))) & 7u);  // slot q (q >= 1): delta index q-1
  const int dq2 = (int)((kDeltaPack >> (4 * (q + 3))) & 7u);        // slot 4+q: delta index 3+q
  const unsigned eic_base = (unsigned)__cvta_generic_to_shared(sm.eic) + 4u * q;
  const unsigned c2_base = (unsigned)__cvta_generic_to_shared(sm.c2);
  const bool lo_lane = lane < 20;  // rows r and r+8 (r+8 <= 12); lanes 20-31 hold rows 5-7 only
  const float* fr_base = sF + (lo_lane ? lane * 4 : 80 + (lane - 20) * 2);
  unsigned ah[6][4], al[6][4];
  float bias0 = 0.0f, bias1 = 0.0f;
  int cur = -1;
  float* actf = reinterpret_cast<float*>(&sm.u.act);
  for (int b = b_begin; b < b_end; ++b) {
    const unsigned short* ob = sm.order + b * 8;
    const int p0 = ob[0];
    const int slot = sm.gi[p0];
    if (slot != cur) {  // warp-uniform: reload this genome's fragments
      cur = slot;
      const float* fg = fr_base + (size_t)slot * kFragGenome;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        float w[4];
        if (lo_lane) {
          const float4 v = *reinterpret_cast<const float4*>(fg + j * kFragStep);
          w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
        } else {
          const float2 v = *reinterpret_cast<const float2*>(fg + j * kFragStep);
          w[0] = v.x, w[1] = 0.0f, w[2] = v.y, w[3] = 0.0f;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) split_tf32(w[c], ah[j][c], al[j][c]);
      }
      const float* bg = sF + (size_t)slot * kFragGenome + 6 * kFragStep;
      bias0 = bg[r];
      bias1 = bg[r + 8];
    }
    // sensors of cell r (padding entries read cell p0; their results are dropped)
    const int pr = ob[r];
    const int pc = pr == 0xFFFF ? p0 : pr;
    const int ty = pc >> 5, tx = pc & 31;
    const int hb = (ty + 1) * kHaloW + tx + 1 - 64;
    const unsigned long long rp = rotated_offsets(sm.rot[pc]);
    int nbr[9];
    nbr[0] = hb + 64;
#pragma unroll
    for (int s = 1; s < 9; ++s) nbr[s] = hb + (int)((rp >> (8 * ((kDeltaPack >> (4 * (s - 1))) & 7u))) & 0xFFu);
    float v[12];
#pragma unroll
    for (int s = 0; s < 9; ++s) v[s] = lds_f32(eic_base + 16u * (unsigned)nbr[s]);
    const int nq1 = q == 0 ? hb + 64 : hb + (int)((rp >> (8 * dq1)) & 0xFFu);
    const int nq2 = hb + (int)((rp >> (8 * dq2)) & 0xFFu);
    v[9] = lds_f32(c2_base + 4u * (unsigned)nq1);
    v[10] = lds_f32(c2_base + 4u * (unsigned)nq2);
    v[11] = q == 0 ? lds_f32(c2_base + 4u * (unsigned)nbr[8]) : 0.0f;
    float dh[4] = {bias0, bias0, bias1, bias1};
    float dc[4] = {0.0f, 0.0f, 0.0f, 0.0f}, dd[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      unsigned bh0, bl0, bh1, bl1;
      split_tf32(v[2 * j], bh0, bl0);
      split_tf32(v[2 * j + 1], bh1, bl1);
      mma_tf32(dh, ah[j], bh0, bh1);
      mma_tf32(dc, ah[j], bl0, bl1);
      mma_tf32(dd, al[j], bh0, bh1);
    }
    float z[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) z[c] = __fadd_rn(dh[c], __fadd_rn(dc[c], dd[c]));
    // z[0], z[1]: output r of cells 2q, 2q+1; z[2], z[3]: output r+8
    const unsigned pair = *reinterpret_cast<const unsigned*>(ob + 2 * q);
    const int pa = (int)(pair & 0xFFFFu), pb = (int)(pair >> 16);
    const bool act_lane = r < 5;
    float sa = squash(act_lane ? z[2] : z[0]);
    float sb = squash(act_lane ? z[3] : z[1]);
    int ea = act_lane ? r + 3 : r - 5;
    int eb = ea;
    float ua = 0.0f, ub = 0.0f;
    if (act_lane) {
      ua = squash(z[0]);
      ub = squash(z[1]);
    }
    if (kExport) {  // all 13 squashed actuators of the exported cells
      const int oa = act_lane ? r : -1;  // action output held in ua/ub
      const int ox = ea + 5;             // explore output held in sa/sb
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int p = c ? pb : pa;
        if (p == 0xFFFF) continue;
        const int ty2 = p >> 5, tx2 = p - (ty2 << 5);
        const long long cell = (long long)(y0 + ty2) * a.g.W + (x0 + tx2);
        float* dst = a.act_out + cell * kActuators;
        if (oa >= 0) dst[oa] = c ? ub : ua;
        dst[ox] = c ? sb : sa;
        if (r == 0) a.act_out_flag[cell] = 1;
      }
    }
#pragma unroll
    for (int m = 4; m <= 16; m <<= 1) {
      const float oa = __shfl_xor_sync(0xFFFFFFFFu, sa, m), ob2 = __shfl_xor_sync(0xFFFFFFFFu, sb, m);
      const int xa = __shfl_xor_sync(0xFFFFFFFFu, ea, m), xb = __shfl_xor_sync(0xFFFFFFFFu, eb, m);
      if (oa > sa || (oa == sa && xa < ea)) sa = oa, ea = xa;
      if (ob2 > sb || (ob2 == sb && xb < eb)) sb = ob2, eb = xb;
    }
    if (pa != 0xFFFF) {
      if (act_lane) actf[r * kTileCells + pa] = ua;
      if (r == 5) {
        actf[5 * kTileCells + pa] = sa;
        sm.u.act.kstar[pa] = (uint8_t)ea;
      }
    }
    if (pb != 0xFFFF) {
      if (act_lane) actf[r * kTileCells + pb] = ub;
      if (r == 6) {
        actf[5 * kTileCells + pb] = sb;
        sm.u.act.kstar[pb] = (uint8_t)eb;
      }
    }
  }
}

template <bool kExport>
__global__ void __launch_bounds__(kThreadsM, 1) k_pass1_mma(const Pass1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MmaSmem& sm = *reinterpret_cast<MmaSmem*>(smem_raw);
  const StepGeom& g = a.g;
  const int tiles_x = (g.W + kTileW - 1) / kTileW;
  const int ntiles = tiles_x * ((g.H + kTileH - 1) / kTileH);
  zero_stats(a);
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  float* sF = reinterpret_cast<float*>(smem_raw + ((sizeof(MmaSmem) + 15) & ~(size_t)15));
  stage_weights<kThreadsM>(sF, a.net.wF, a.capacity * kFragGenome);
  asm volatile("cp.async.commit_group;" ::: "memory");
  using PF = PrefetchT<kThreadsM>;
  constexpr int kPreCellsM = PF::kCells;
  int rank[kPreCellsM];
  {
    PF pf;
    prefetch_tile(a, tile, tiles_x, pf);
    commit_tile(sm, pf);
    for (int b = threadIdx.x; b < a.capacity; b += kThreadsM) sm.bins[b] = 0;
    __syncthreads();
    bucket_count<kThreadsM, kPreCellsM>(sm.bins, pf.gi, rank);
    __syncthreads();
    bucket_offsets<kThreadsM, 8, 8>(sm.bins, sm.scratch, sm.order, &sm.n_units, a.capacity);
    __syncthreads();
    bucket_scatter<kThreadsM, kPreCellsM>(sm.bins, pf.gi, rank, sm.order);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  long long t_mark = clock64();
  (void)t_mark;
  PHASE_MARK(4);
  for (; tile < ntiles; tile += gridDim.x) {
    const int x0 = (tile % tiles_x) * kTileW;
    const int y0 = (tile / tiles_x) * kTileH;
    const int next = tile + gridDim.x;
    if (next < ntiles) prefetch_tile_l2<kThreadsM>(a, next, tiles_x);
    for (int b = threadIdx.x; b < a.capacity; b += kThreadsM) sm.bins[b] = 0;  // for the next count
    PHASE_MARK(0);
    tile_controller_mma<kExport>(a, sm, sF, x0, y0);
    __syncthreads();
    PHASE_MARK(1);
    PF pf;
    if (next < ntiles) prefetch_tile(a, next, tiles_x, pf);
    tile_physics<false, kExport, kThreadsM>(a, sm, x0, y0);
    if (next < ntiles) bucket_count<kThreadsM, kPreCellsM>(sm.bins, pf.gi, rank);
    __syncthreads();
    PHASE_MARK(2);
    if (next < ntiles) {
      bucket_offsets<kThreadsM, 8, 8>(sm.bins, sm.scratch, sm.order, &sm.n_units, a.capacity);
      __syncthreads();
      bucket_scatter<kThreadsM, kPreCellsM>(sm.bins, pf.gi, rank, sm.order);
      commit_tile(sm, pf);
    }
    __syncthreads();
    PHASE_MARK(3);
  }
}

// ---------------------------------------------------------------------------
// Pass 2

// Pass 2 works on warp tiles of 32 x 4 cells: each warp stages its own tile
// plus 1-cell halo (proposal byte, quantity, post-death genome; infra of the
// tile) in a private shared-memory slice and resolves it without any CTA
// barrier, so the latency of one warp's loads overlaps the others' work.
constexpr int kWtW = 32, kWtH = 4;  // warp tile
constexpr int kWtCells = kWtW * kWtH;
constexpr int kWtHW = kWtW + 2;
constexpr int kWtHalo = (kWtH + 2) * kWtHW;
constexpr int kWarps2 = kThreads2 / 32;

struct WarpTile {
  uint8_t rp[kWtHalo];
  uint8_t rot[kWtCells];
  float q[kWtHalo];
  int gi[kWtHalo];
  float inf[kWtCells];
  unsigned short queue[kWtCells];
};

// Shipment arriving at tile cell (ty, tx) from direction d: halo index of the
// source, its quantity and the 64-bit ordering key (q desc, global source asc).
struct Arrival {
  int h;
  float q;
  u64 key;
};

__device__ __forceinline__ Arrival arrival(const StepGeom& g, const WarpTile& wt, int y, int x, int ty, int tx,
                                           int d) {
  Arrival r;
  r.h = (ty + 1 - dir_dy(d)) * kWtHW + tx + 1 - dir_dx(d);
  r.q = __fadd_rn(wt.q[r.h], 0.0f);  // canonical +0
  const int sy = y - dir_dy(d);
  int sx = x - dir_dx(d);
  sx = sx < 0 ? sx + g.W : (sx >= g.W ? sx - g.W : sx);
  int grow = (int)g.row0 + sy;
  grow = grow < 0 ? grow + g.Hg : (grow >= g.Hg ? grow - g.Hg : grow);
  const unsigned gsrc = (unsigned)grow * (unsigned)g.W + (unsigned)sx;
  r.key = ((u64)__float_as_uint(r.q) << 32) | (u64)(0xFFFFFFFFu - gsrc);
  return r;
}

__device__ __forceinline__ unsigned arrival_mask(const WarpTile& wt, int ty, int tx) {
  unsigned m = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) m |= wt.rp[(ty + 1 - dir_dy(d)) * kWtHW + tx + 1 - dir_dx(d)] & (1u << d);
  return m;
}

// Resolve one target cell whose arrival mask is m (bit d: the neighbour at
// t - off[d] ships in direction d): ordered sum, winner, adoption, stores.
// Returns the cell's final genome slot.  KIND restricts the compiled paths
// (1: at most one arrival, 2: exactly two, 3: three or more) so that a warp
// never executes predicated-off code of the other cases.
__device__ __forceinline__ void st_tex(float* p, const float4& f, float inf) {  // {E, C0, C1, C2 | I, 0, 0, 0}
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%6,%6};" ::"l"(p), "f"(f.x), "f"(f.y), "f"(f.z), "f"(f.w),
               "f"(inf), "f"(0.0f)
               : "memory");
}

template <bool kRecord, int KIND, bool kLazy = false>
__device__ __forceinline__ int resolve_cell(const Pass2Args& a, const WarpTile& wt, int ty, int tx, int y, int x,
                                            unsigned m, int& adopted, bool edge_tile, const float4* ec = nullptr) {
  const StepGeom& g = a.g;
  const int hc = (ty + 1) * kWtHW + tx + 1;
  const float before = wt.inf[ty * kWtW + tx];
  const int own = wt.gi[hc];
  const int r = wt.rot[ty * kWtW + tx];
  float acc = before;
  int gnew = own, rnew = r;
  bool adopt = false;
  if (m) {
    const int n = KIND == 1 ? 1 : (KIND == 2 ? 2 : 3);
    u64 win;
    int wd, wh;
    if (n == 1) {  // single arrival: no ordering, source index only for the event record
      wd = __ffs(m) - 1;
      wh = (ty + 1 - dir_dy(wd)) * kWtHW + tx + 1 - dir_dx(wd);
      const float q = __fadd_rn(wt.q[wh], 0.0f);
      acc = __fadd_rn(acc, q);
      win = (u64)__float_as_uint(q) << 32;
      if (kRecord) win = arrival(g, wt, y, x, ty, tx, wd).key;
    } else if (n == 2) {  // order by q; the global source index only breaks exact ties
      const int d0 = __ffs(m) - 1, d1 = __ffs(m & (m - 1)) - 1;
      const int h0 = (ty + 1 - dir_dy(d0)) * kWtHW + tx + 1 - dir_dx(d0);
      const int h1 = (ty + 1 - dir_dy(d1)) * kWtHW + tx + 1 - dir_dx(d1);
      const float q0 = __fadd_rn(wt.q[h0], 0.0f), q1 = __fadd_rn(wt.q[h1], 0.0f);
      bool first0 = q0 > q1;
      if (q0 == q1) first0 = arrival(g, wt, y, x, ty, tx, d0).key > arrival(g, wt, y, x, ty, tx, d1).key;
      acc = __fadd_rn(__fadd_rn(acc, first0 ? q0 : q1), first0 ? q1 : q0);
      wd = first0 ? d0 : d1;
      wh = first0 ? h0 : h1;
      win = (u64)__float_as_uint(first0 ? q0 : q1) << 32;
      if (kRecord) win = arrival(g, wt, y, x, ty, tx, wd).key;
    } else {
      // general (>= 3 arrivals).  Quantities are >= 0, so their f32 bit
      // patterns order like the values; equal quantities add identically in
      // any order, so the sum only needs the quantities sorted descending
      // (32-bit min/max network, 19 comparators) and the source index only
      // breaks ties for the winner.  Present zero quantities sort last and
      // add +0 (which only turns a -0 sum into +0).
      unsigned qb[8];
      unsigned qmax = 0, zeros = 0;
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const bool pres = (m >> d) & 1u;
        const unsigned b = pres ? __float_as_uint(__fadd_rn(wt.q[(ty + 1 - dir_dy(d)) * kWtHW + tx + 1 - dir_dx(d)],
                                                            0.0f))
                                : 0u;
        qb[d] = b;
        qmax = max(qmax, b);
        zeros |= (pres && b == 0u) ? 1u : 0u;
      }
      unsigned tie = 0;
#pragma unroll
      for (int d = 0; d < 8; ++d) tie |= ((m >> d) & 1u) && qb[d] == qmax ? (1u << d) : 0u;
      wd = __ffs(tie) - 1;
      if (tie & (tie - 1)) {  // exact tie on the maximum: lowest global source wins
        u64 best = arrival(g, wt, y, x, ty, tx, wd).key;
        for (unsigned rest = tie & (tie - 1); rest; rest &= rest - 1) {
          const int d = __ffs(rest) - 1;
          const u64 k = arrival(g, wt, y, x, ty, tx, d).key;
          if (k > best) {
            best = k;
            wd = d;
          }
        }
      }
      wh = (ty + 1 - dir_dy(wd)) * kWtHW + tx + 1 - dir_dx(wd);
      win = (u64)qmax << 32;
      if (kRecord) win = arrival(g, wt, y, x, ty, tx, wd).key;
#define EVO_CE(a, b)                 \
  {                                  \
    const unsigned hi = max(a, b);   \
    b = min(a, b);                   \
    a = hi;                          \
  }
      EVO_CE(qb[0], qb[1]) EVO_CE(qb[2], qb[3]) EVO_CE(qb[4], qb[5]) EVO_CE(qb[6], qb[7])
      EVO_CE(qb[0], qb[2]) EVO_CE(qb[1], qb[3]) EVO_CE(qb[4], qb[6]) EVO_CE(qb[5], qb[7])
      EVO_CE(qb[1], qb[2]) EVO_CE(qb[5], qb[6])
      EVO_CE(qb[0], qb[4]) EVO_CE(qb[1], qb[5]) EVO_CE(qb[2], qb[6]) EVO_CE(qb[3], qb[7])
      EVO_CE(qb[2], qb[4]) EVO_CE(qb[3], qb[5])
      EVO_CE(qb[1], qb[2]) EVO_CE(qb[3], qb[4]) EVO_CE(qb[5], qb[6])
#undef EVO_CE
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (qb[i]) acc = __fadd_rn(acc, __uint_as_float(qb[i]));
      if (zeros) acc = __fadd_rn(acc, 0.0f);
    }
    const float qw = __uint_as_float((unsigned)(win >> 32));
    if (qw > before) {  // physics.py:325
      adopt = true;
      gnew = wt.gi[wh];
      rnew = wd;
      if (kRecord) {
        const long long cell = (long long)y * g.W + x;
        a.ev.src[cell] = (long long)(0xFFFFFFFFu - (unsigned)(win & 0xFFFFFFFFull));
        a.ev.q[cell] = qw;
        a.ev.def[cell] = own;
      }
    }
  }
  if (kRecord && !adopt) a.ev.src[(long long)y * g.W + x] = -1;
  adopted += adopt ? 1 : 0;
  const unsigned o = (unsigned)((y + 1) * g.W + x);
  // lazy fused steps: the final infrastructure is the second half of the
  // next step's texture record {E, C0, C1, C2 | I, 0, 0, 0}
  // (whole 32-byte records: half-sector stores made L2 fill the other half from DRAM)
  float4 f4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (kLazy) {
    f4 = ec[ty * kWtW + tx];
    st_tex(a.tex_out + (size_t)o * 8, f4, acc);
  } else {
    a.back.I[o] = acc;
  }
  a.back.gi[o] = gnew;
  a.back.rot[o] = (uint8_t)rnew;
  if (edge_tile && (y == 0 || y == g.H - 1)) {  // warp-uniform pre-test per tile
    if (y == 0) {
      const unsigned og = (unsigned)((g.H + 1) * g.W + x);
      if (kLazy)
        st_tex(a.tex_out + (size_t)og * 8, f4, acc);
      else
        a.back.I[og] = acc;
      a.back.gi[og] = gnew;
      a.back.rot[og] = (uint8_t)rnew;
    }
    if (y == g.H - 1) {
      if (kLazy)
        st_tex(a.tex_out + (size_t)x * 8, f4, acc);
      else
        a.back.I[x] = acc;
      a.back.gi[x] = gnew;
      a.back.rot[x] = (uint8_t)rnew;
    }
  }
  return gnew;
}

// kMidRec: pass 1 left 32-byte records {E', C0', C1', C2' | I', q, genome,
// proposal byte} at the cell index (the fused gather step, FusedPhysics)
// instead of the mid planes: the halo rows read the records' second halves
// (rows wrap by index: single-strip steps only), the tile rows also copy the
// first halves into the back E and C planes.
// kMid 2 (lazy): the same, but E', C' and the final I go to the texture
// records (the next step's sense texture) and the back E, I, C planes are
// not written (evoca_abi.cu materialises them on demand).
template <bool kRecord, int kMid>
// 4 resident CTAs per SM (64 registers, no spills): the 4 x num_sms grid is
// one wave; at 80 registers only 3 fitted and the last quarter of the grid ran
// as a tail (k_resolve 22.5 -> 20.9 us on config 2, config 3 step 2.44 -> 2.40 ms)
#ifndef EVO_K2_MIN_BLOCKS
#define EVO_K2_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kThreads2, EVO_K2_MIN_BLOCKS) k_resolve(const Pass2Args a) {
  constexpr bool kMidRec = kMid != 0, kLazy = kMid == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpTile* wts = reinterpret_cast<WarpTile*>(smem_raw);
  int* hist = reinterpret_cast<int*>(smem_raw + ((sizeof(WarpTile) * kWarps2 + 15) & ~(size_t)15));
  // lazy: {E', C0', C1', C2'} of the warp's tile cells, behind the histogram
  float4* ec = reinterpret_cast<float4*>(smem_raw + ((sizeof(WarpTile) * kWarps2 + 15) & ~(size_t)15) +
                                         (((size_t)a.capacity * sizeof(int) + 15) & ~(size_t)15)) +
               (threadIdx.x >> 5) * kWtCells;
  __shared__ int s_adopt;
  __shared__ bool s_last;
  const StepGeom& g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpTile& wt = wts[warp];
  for (int b = tid; b < a.capacity; b += kThreads2) hist[b] = 0;
  if (tid == 0) s_adopt = 0;
  __syncthreads();
  const int tiles_x = (g.W + kWtW - 1) / kWtW;
  const int ntiles = tiles_x * ((g.H + kWtH - 1) / kWtH);
  int my_adopt = 0;
  for (int tile = blockIdx.x * kWarps2 + warp; tile < ntiles; tile += gridDim.x * kWarps2) {
    const int x0 = (tile % tiles_x) * kWtW;
    const int y0 = (tile / tiles_x) * kWtH;
    const bool edge_tile = g.own_ghosts && (y0 == 0 || y0 + kWtH >= g.H);
    if (kMidRec) {
      constexpr int kRows = kWtH + 2;
      int xa = x0 - 1 + lane;
      xa = xa < 0 ? xa + g.W : (xa >= g.W ? xa - g.W : xa);
      if (xa >= g.W) xa = g.W - 1;
      // halo columns 32 and 33 of the six halo rows: one load on lanes 0..11
      const bool extra = lane < 2 * kRows;
      const int er = extra ? lane >> 1 : 0;
      int xb = x0 + 31 + (lane & 1);
      xb = xb >= g.W ? xb - g.W : xb;
      if (xb >= g.W) xb = g.W - 1;
      // halo row r of the tile -> record row: a single strip wraps by index;
      // strips keep their neighbours' rows (evo_halo_unpack) behind the last
      // one: row H = ghost below, row H + 1 = ghost above
      auto rec_row = [&](int r) {
        const int y = min(y0 + r - 1, g.H);
        if (g.own_ghosts) return y < 0 ? g.H - 1 : (y >= g.H ? 0 : y);
        return y < 0 ? g.H + 1 : y;
      };
      float4 hv[kRows], hx = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int r = 0; r < kRows; ++r)
        hv[r] = __ldg(reinterpret_cast<const float4*>(a.mid_rec + ((size_t)rec_row(r) * g.W + xa) * 8) + 1);
      if (extra) hx = __ldg(reinterpret_cast<const float4*>(a.mid_rec + ((size_t)rec_row(er) * g.W + xb) * 8) + 1);
      const int xi = min(x0 + lane, g.W - 1);
      float4 fv[kWtH];
      uint8_t vr[kWtH];
#pragma unroll
      for (int j = 0; j < kWtH; ++j) {
        const int yj = min(y0 + j, g.H - 1);
        fv[j] = __ldg(reinterpret_cast<const float4*>(a.mid_rec + ((size_t)yj * g.W + xi) * 8));
        vr[j] = __ldg(a.rot_front + (unsigned)((yj + 1) * g.W + xi));
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        wt.rp[r * kWtHW + lane] = (uint8_t)__float_as_int(hv[r].w);
        wt.q[r * kWtHW + lane] = hv[r].y;
        wt.gi[r * kWtHW + lane] = __float_as_int(hv[r].z);
        if (r >= 1 && r <= kWtH && lane >= 1) wt.inf[(r - 1) * kWtW + lane - 1] = hv[r].x;
      }
      if (extra) {
        wt.rp[er * kWtHW + 32 + (lane & 1)] = (uint8_t)__float_as_int(hx.w);
        wt.q[er * kWtHW + 32 + (lane & 1)] = hx.y;
        wt.gi[er * kWtHW + 32 + (lane & 1)] = __float_as_int(hx.z);
        if (!(lane & 1) && er >= 1 && er <= kWtH) wt.inf[(er - 1) * kWtW + 31] = hx.x;
      }
      const unsigned pst = (unsigned)g.stride;
#pragma unroll
      for (int j = 0; j < kWtH; ++j) {
        wt.rot[j * kWtW + lane] = vr[j];
        const int y = y0 + j, x = x0 + lane;
        if (kLazy) {  // first half of the next texture record, stored with the final I by resolve_cell
          ec[j * kWtW + lane] = fv[j];
        } else if (y < g.H && x < g.W) {  // final E and C of the cell (pass 2 does not change them)
          const unsigned o = (unsigned)((y + 1) * g.W + x);
          a.back.E[o] = fv[j].x;
          a.back.C[o] = fv[j].y;
          a.back.C[pst + o] = fv[j].z;
          a.back.C[2 * pst + o] = fv[j].w;
          if (edge_tile && (y == 0 || y == g.H - 1)) {
            if (y == 0) {
              const unsigned og = (unsigned)((g.H + 1) * g.W + x);
              a.back.E[og] = fv[j].x;
              a.back.C[og] = fv[j].y;
              a.back.C[pst + og] = fv[j].z;
              a.back.C[2 * pst + og] = fv[j].w;
            }
            if (y == g.H - 1) {
              a.back.E[x] = fv[j].x;
              a.back.C[x] = fv[j].y;
              a.back.C[pst + x] = fv[j].z;
              a.back.C[2 * pst + x] = fv[j].w;
            }
          }
        }
      }
      __syncwarp();
    } else {
      // all staging loads of the warp tile issued before any shared store
      // halo column lane (x0-1+lane) of every halo row, plus halo columns 32
      // and 33 on lanes 0 and 1; ghost rows make the vertical wrap implicit
      constexpr int kRows = kWtH + 2;
      int xa = x0 - 1 + lane;
      xa = xa < 0 ? xa + g.W : (xa >= g.W ? xa - g.W : xa);
      if (xa >= g.W) xa = g.W - 1;
      int xb = x0 + 31 + (lane & 1);
      xb = xb >= g.W ? xb - g.W : xb;
      if (xb >= g.W) xb = g.W - 1;
      const bool extra = lane < 2;
      uint8_t vrp[kRows], wrp[kRows];
      float vq[kRows], wq[kRows], vi[kWtH];
      int vg[kRows], wg[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int y = min(y0 + r - 1, g.H);
        const unsigned row = (unsigned)((y + 1) * g.W);
        vrp[r] = __ldg(a.mid.rp + row + xa);
        vq[r] = __ldg(a.mid.q + row + xa);
        vg[r] = __ldg(a.mid.gi + row + xa);
        if (extra) {
          wrp[r] = __ldg(a.mid.rp + row + xb);
          wq[r] = __ldg(a.mid.q + row + xb);
          wg[r] = __ldg(a.mid.gi + row + xb);
        }
      }
      const int xi = min(x0 + lane, g.W - 1);
      uint8_t vr[kWtH];
#pragma unroll
      for (int j = 0; j < kWtH; ++j) {
        const unsigned o = (unsigned)((min(y0 + j, g.H - 1) + 1) * g.W + xi);
        vi[j] = __ldg(a.mid.I + o);
        vr[j] = __ldg(a.rot_front + o);
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        wt.rp[r * kWtHW + lane] = vrp[r];
        wt.q[r * kWtHW + lane] = vq[r];
        wt.gi[r * kWtHW + lane] = vg[r];
        if (extra) {
          wt.rp[r * kWtHW + 32 + lane] = wrp[r];
          wt.q[r * kWtHW + 32 + lane] = wq[r];
          wt.gi[r * kWtHW + 32 + lane] = wg[r];
        }
      }
#pragma unroll
      for (int j = 0; j < kWtH; ++j) {
        wt.inf[j * kWtW + lane] = vi[j];
        wt.rot[j * kWtW + lane] = vr[j];
      }
      __syncwarp();
    }
    // cells with <= 1 arrival resolve in place; the rest are queued so that
    // the ordering work runs on whole warps
    // queue[0..n2): exactly two arrivals; queue[kWtCells-n3..): three or more
    int n2 = 0, n3 = 0;
#pragma unroll
    for (int j = 0; j < kWtH; ++j) {
      const int ty = j, tx = lane;
      const int y = y0 + ty, x = x0 + tx;
      int key = -1;
      int kind = 0;  // 0 resolved here, 2 / 3 deferred
      if (y < g.H && x < g.W) {
        const unsigned m = arrival_mask(wt, ty, tx);
        if ((m & (m - 1)) == 0) {
          const int gn = resolve_cell<kRecord, 1, kLazy>(a, wt, ty, tx, y, x, m, my_adopt, edge_tile, ec);
          key = (gn >= 0 && gn < a.capacity) ? gn : -1;
        } else {
          kind = __popc(m) == 2 ? 2 : 3;
        }
      }
      const unsigned b2 = __ballot_sync(0xffffffffu, kind == 2);
      const unsigned b3 = __ballot_sync(0xffffffffu, kind == 3);
      const unsigned below = (1u << lane) - 1u;
      if (kind == 2) wt.queue[n2 + __popc(b2 & below)] = (unsigned short)(ty * kWtW + tx);
      if (kind == 3) wt.queue[kWtCells - 1 - (n3 + __popc(b3 & below))] = (unsigned short)(ty * kWtW + tx);
      n2 += __popc(b2);
      n3 += __popc(b3);
      if (key >= 0) atomicAdd(&hist[key], 1);
    }
    __syncwarp();
#pragma unroll 1
    for (int e = lane; e < n2; e += 32) {
      const int i = wt.queue[e];
      const int ty = i / kWtW, tx = i - ty * kWtW;
      const int gn = resolve_cell<kRecord, 2, kLazy>(a, wt, ty, tx, y0 + ty, x0 + tx, arrival_mask(wt, ty, tx), my_adopt,
                                              edge_tile, ec);
      if (gn >= 0 && gn < a.capacity) atomicAdd(&hist[gn], 1);
    }
#pragma unroll 1
    for (int e = lane; e < n3; e += 32) {
      const int i = wt.queue[kWtCells - 1 - e];
      const int ty = i / kWtW, tx = i - ty * kWtW;
      const int gn = resolve_cell<kRecord, 3, kLazy>(a, wt, ty, tx, y0 + ty, x0 + tx, arrival_mask(wt, ty, tx), my_adopt,
                                              edge_tile, ec);
      if (gn >= 0 && gn < a.capacity) atomicAdd(&hist[gn], 1);
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) my_adopt += __shfl_xor_sync(0xffffffffu, my_adopt, off);
  if (lane == 0 && my_adopt) atomicAdd(&s_adopt, my_adopt);
  __syncthreads();
  if (tid == 0 && s_adopt) atomicAdd((unsigned long long*)&a.census.stats[0], (unsigned long long)s_adopt);
#ifndef EVO_DIAG_NO_FLUSH
  for (int b = tid; b < a.capacity; b += kThreads2)
    if (hist[b]) atomicAdd(&a.census.counts[b], hist[b]);
#endif
#ifdef EVO_DIAG_NO_TICKET  // diagnostics builds only: census not finished
  return;
#endif
  if (!a.run_census) return;
  // last CTA: census epilogue (physics.py:395-404, neuroevo.py:521-542).
  // One cumulative release fence by thread 0 after the barrier publishes the
  // whole CTA's count atomics before its ticket (a fence in every thread
  // stalled every warp on a full memory drain).
  __syncthreads();
  if (tid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const unsigned ticket = atomicAdd(a.census.done, 1u);
    s_last = (ticket == gridDim.x - 1);
    if (s_last) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  if (!s_last) return;
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


// Census epilogue as its own launch (strip mode: after the cross-rank sum of
// counts).  A set *skip (rejected host planes, evo_step_host) only clears
// the accumulators: slot states are left as they were before the step.
__global__ void k_census_finish(const Census c, int capacity, long long t, const int* skip) {
  const bool discard = skip && *skip;
  int dead = 0;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < capacity; b += gridDim.x * blockDim.x) {
    const int n = c.counts[b];
    c.counts[b] = 0;
    if (discard) continue;
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

// Row-band (host-pipelined) steps of a single strip: the bands run as
// strips of one context whose ghost rows are the neighbouring bands' real
// rows, so only the torus seam needs the pass-1 outputs pass 2 reads
// (post-death genome, shipped quantity, proposal byte) wrapped.
__global__ void k_wrap_mid(const Mid m, const StepGeom g) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.W; x += gridDim.x * blockDim.x) {
    const long long top = plane_row(g, -1) + x, last = plane_row(g, g.H - 1) + x;
    const long long bot = plane_row(g, g.H) + x, first = plane_row(g, 0) + x;
    m.gi[top] = m.gi[last];
    m.gi[bot] = m.gi[first];
    m.q[top] = m.q[last];
    m.q[bot] = m.q[first];
    m.rp[top] = m.rp[last];
    m.rp[bot] = m.rp[first];
  }
}

// RGBA frame of the front buffer (substrate.py:147-165): red = energy and
// green = infrastructure scaled by their display norms, clamped to [0, 1],
// x255, rounded half-to-even; blue = the genome slot's golden-ratio hue
// (slot * 0.6180339887498949 mod 1, 0 when empty); alpha 255.  All in f64 with
// the reference's operation order (a true division by the norm), so frames
// are bit-identical to numpy's; 12 B read + 4 B written per cell.
__device__ __forceinline__ unsigned render_channel(double v) {
  v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);  // np.clip (NaN passes through)
  v = rint(v * 255.0);
  return v == v ? (unsigned)v : 0u;
}

__global__ void k_render_rgb(const Planes f, const StepGeom g, double norm_e, double norm_i, uint32_t* out) {
  const long long n = (long long)g.W * g.H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long o = g.W + i;  // skip ghost row -1
    const unsigned r = render_channel((double)f.E[o] / norm_e);
    const unsigned gr = render_channel((double)f.I[o] / norm_i);
    const int slot = f.gi[o];
    const double hue = slot < 0 ? 0.0 : fmod((double)slot * 0.6180339887498949, 1.0);
    const unsigned b = (unsigned)rint(hue * 255.0);
    out[i] = r | (gr << 8) | (b << 16) | (255u << 24);
  }
}

// Range check of uploaded genome / rotation planes (the host upload's
// ValueError, done on the device so the host never scans the planes):
// out-of-range entries are cleared (genome -1, rotation & 7) so no kernel
// indexes outside the tables, and *bad is set; the host reports the error.
__global__ void k_check_cells(int32_t* gi, uint8_t* rot, long long n, int capacity, int* bad) {
  int b = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int g = gi[i];
    if (g < -1 || g >= capacity) {
      gi[i] = -1;
      b = 1;
    }
    const uint8_t r = rot[i];
    if (r > 7) {
      rot[i] = r & 7;
      b = 1;
    }
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// Strip halo staging (multi-GPU row strips).  which 0: the five sensed
// front planes E, I, C0..C2 (f32); which 1: the pass-1 outputs a
// neighbour's pass 2 reads - post-death genome (i32), shipped quantity (f32
// bits), proposal byte (widened to a 32-bit word).  A buffer holds two rows
// of `planes x W` 32-bit words: [0] = this strip's first row (pack) / the
// ghost row above (unpack), [1] = last row / ghost row below.
__global__ void k_halo_pack(const Planes f, const Mid m, const StepGeom g, int which, uint32_t* buf) {
  const int np = which == 0 ? 5 : 3;
  const int n = 2 * np * g.W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int side = i / (np * g.W), r = i - side * np * g.W, pl = r / g.W, x = r - pl * g.W;
    const long long o = plane_row(g, side ? g.H - 1 : 0) + x;
    uint32_t v;
    if (which == 0) {
      const float* src = pl == 0 ? f.E : (pl == 1 ? f.I : f.C + (pl - 2) * g.stride);
      v = __float_as_uint(src[o]);
    } else {
      v = pl == 0 ? (uint32_t)m.gi[o] : (pl == 1 ? __float_as_uint(m.q[o]) : (uint32_t)m.rp[o]);
    }
    buf[i] = v;
  }
}

__global__ void k_halo_unpack(const Planes f, const Mid m, const StepGeom g, int which, const uint32_t* buf) {
  const int np = which == 0 ? 5 : 3;
  const int n = 2 * np * g.W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int side = i / (np * g.W), r = i - side * np * g.W, pl = r / g.W, x = r - pl * g.W;
    const long long o = plane_row(g, side ? g.H : -1) + x;
    const uint32_t v = buf[i];
    if (which == 0) {
      float* dst = pl == 0 ? f.E : (pl == 1 ? f.I : f.C + (pl - 2) * g.stride);
      dst[o] = __uint_as_float(v);
    } else if (pl == 0) {
      m.gi[o] = (int32_t)v;
    } else if (pl == 1) {
      m.q[o] = __uint_as_float(v);
    } else {
      m.rp[o] = (uint8_t)v;
    }
  }
}

// The same wire format from / to the fused step's buffers: which = 0 with the
// state in the sense texture (lazy steps: E, I, C of rows 0 / H-1 out of, and
// into the ghost rows of, the texture records), which = 1 with pass-1 records
// (genome, quantity, proposal byte of rows 0 / H-1; the neighbours' rows go to
// record rows H + 1 (above) and H (below), which k_resolve reads as its halo).
__global__ void k_halo_pack_rec(const float* tex, const float* rec, const StepGeom g, int which, uint32_t* buf) {
  const int np = which == 0 ? 5 : 3;
  const int n = 2 * np * g.W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int side = i / (np * g.W), r = i - side * np * g.W, pl = r / g.W, x = r - pl * g.W;
    const int y = side ? g.H - 1 : 0;
    uint32_t v;
    if (which == 0) {
      const int f = pl == 0 ? 0 : (pl == 1 ? 4 : pl - 1);  // gs::tex_ch
      v = __float_as_uint(tex[((size_t)(y + 1) * g.W + x) * 8 + f]);
    } else {
      v = __float_as_uint(rec[((size_t)y * g.W + x) * 8 + (pl == 0 ? 6 : (pl == 1 ? 5 : 7))]);
    }
    buf[i] = v;
  }
}

__global__ void k_halo_unpack_rec(float* tex, float* rec, const StepGeom g, int which, const uint32_t* buf) {
  const int np = which == 0 ? 5 : 3;
  const int n = 2 * np * g.W;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int side = i / (np * g.W), r = i - side * np * g.W, pl = r / g.W, x = r - pl * g.W;
    const float v = __uint_as_float(buf[i]);
    if (which == 0) {
      const int f = pl == 0 ? 0 : (pl == 1 ? 4 : pl - 1);
      tex[((size_t)(side ? g.H + 1 : 0) * g.W + x) * 8 + f] = v;
    } else {
      rec[((size_t)(side ? g.H : g.H + 1) * g.W + x) * 8 + (pl == 0 ? 6 : (pl == 1 ? 5 : 7))] = v;
    }
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
    gi[cells[i] + W] = slots[i];  // +W: skip ghost row -1
  }
}

// ---------------------------------------------------------------------------
// launchers

// Per-device launch configuration: the SM count and every kernel's opted-in
// dynamic shared-memory size are properties of the device (context), so they
// are cached per device ordinal - a process may drive several GPUs.
constexpr int kMaxDevices = 64;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
static int num_sms() {
  static int sms[kMaxDevices] = {0};
  const int dev = current_device();
  if (!sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = n > 0 ? n : 148;
  }
  return sms[dev];
}

struct SmemOptIn {
  int bytes[kMaxDevices] = {0};
};
// Raise `kernel`'s dynamic shared-memory limit on the current device if
// `smem` exceeds what was configured there; *first is set when this device
// configures the kernel for the first time.
template <typename K>
static cudaError_t set_smem(K kernel, size_t smem, SmemOptIn& cfg, bool* first = nullptr) {
  int& configured = cfg.bytes[current_device()];
  if (first) *first = configured == 0;
  if ((int)smem <= configured) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) configured = (int)smem;
  return e;
}

template <bool I, bool E, bool H>
static cudaError_t launch_generic(const Pass1Args& a, cudaStream_t st) {
  const size_t smem = sizeof(GenericSmem) + (size_t)a.capacity * sizeof(int);
  static SmemOptIn cfg;
  cudaError_t e = set_smem(k_pass1_generic<I, E, H>, smem, cfg);
  if (e != cudaSuccess) return e;
  const int tiles = ((a.g.W + kTileW - 1) / kTileW) * ((a.g.H + kTileH - 1) / kTileH);
  k_pass1_generic<I, E, H><<<tiles, kThreads1, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool E, bool S>
static cudaError_t launch_direct(const Pass1Args& a, cudaStream_t st) {
  size_t smem = sizeof(DirectSmem) + (size_t)a.capacity * sizeof(int);
  if (S) smem = ((smem + 15) & ~(size_t)15) + weight_smem_bytes(a.capacity);
  static SmemOptIn cfg;
  bool first = false;
  cudaError_t e = set_smem(k_pass1_direct<E, S>, smem, cfg, &first);
  if (e != cudaSuccess) return e;
  if (first) {
    if (!S) {
      // smallest shared-memory carveout that holds one CTA: the rest of the
      // 256 KB per SM stays L1, where the per-genome weight table lives.
      const int pct = (int)((smem + 8 * 1024) * 100 / (228 * 1024)) + 1;
      cudaFuncSetAttribute(k_pass1_direct<E, S>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           pct > 100 ? 100 : pct);
    }
  }
  const int tiles = ((a.g.W + kTileW - 1) / kTileW) * ((a.g.H + kTileH - 1) / kTileH);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  k_pass1_direct<E, S><<<grid, kThreadsP, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool E>
static cudaError_t launch_mma(const Pass1Args& a, cudaStream_t st) {
  const size_t smem = ((sizeof(MmaSmem) + 15) & ~(size_t)15) + (size_t)a.capacity * kFragGenome * sizeof(float);
  static SmemOptIn cfg;
  cudaError_t e = set_smem(k_pass1_mma<E>, smem, cfg);
  if (e != cudaSuccess) return e;
  const int tiles = ((a.g.W + kTileW - 1) / kTileW) * ((a.g.H + kTileH - 1) / kTileH);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  k_pass1_mma<E><<<grid, kThreadsM, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_frag_relayout(const Params& net, int capacity, float* wF, cudaStream_t st) {
  const int n = capacity * kFragGenome;
  k_frag_relayout<<<(n + 255) / 256, 256, 0, st>>>(net, capacity, wF);
  return cudaGetLastError();
}

cudaError_t launch_pass1(const Pass1Args& a, bool inject, bool export_actions, cudaStream_t st) {
  if (inject && a.act_rank) {
    const long long n = (long long)a.g.W * a.g.H;
    const int grid = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 8);
    k_physics_rows<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  if (inject) return launch_generic<true, false, false>(a, st);
  if (a.net.hidden > 0)
    return export_actions ? launch_generic<false, true, true>(a, st) : launch_generic<false, false, true>(a, st);
  if (a.net.wF && a.capacity <= kMmaSlots)
    return export_actions ? launch_mma<true>(a, st) : launch_mma<false>(a, st);
  if (a.capacity <= kSmemWeightSlots)
    return export_actions ? launch_direct<true, true>(a, st) : launch_direct<false, true>(a, st);
  return export_actions ? launch_direct<true, false>(a, st) : launch_direct<false, false>(a, st);
}

cudaError_t launch_census_finish(const Census& c, int capacity, long long t, cudaStream_t st, const int* skip);

cudaError_t launch_resolve_rows(const Pass2Args& a, int num_sms, cudaStream_t st);

cudaError_t launch_pass2(const Pass2Args& a_in, cudaStream_t st) {
  Pass2Args a = a_in;
#ifdef EVO_K2_STREAM
  // measured alternative (evoca_resolve.cu): the register-window streaming
  // form - 9.0 warp instructions per cell against 9.6 here, 0.24 ms against
  // 0.22 ms on config 3 and 49 us against 24 us on config 2
  return launch_resolve_rows(a, num_sms(), st);
#endif
#ifdef EVO_K2_SPLIT_CENSUS
  // census epilogue as its own launch instead of the last-CTA ticket: the
  // ticket's per-CTA GPU-scope fence costs ~4 us of k_resolve, the extra
  // launch about the same (measured), so the ticket stays the default
  const bool finish = a.run_census != 0;
  a.run_census = 0;
#endif
  const int tiles = ((a.g.W + kWtW - 1) / kWtW) * ((a.g.H + kWtH - 1) / kWtH);
  // few CTAs, many warp tiles each: the per-CTA census flush (capacity
  // global atomics on shared addresses) and the completion ticket are
  // serialised in L2, so they must not scale with the grid
#ifndef EVO_K2_GRID_FACTOR
#define EVO_K2_GRID_FACTOR 4
#endif
  int grid = num_sms() * EVO_K2_GRID_FACTOR;
  const int need = (tiles + kWarps2 - 1) / kWarps2;
  if (grid > need) grid = need;
  size_t smem = ((sizeof(WarpTile) * kWarps2 + 15) & ~(size_t)15) + (size_t)a.capacity * sizeof(int);
  if (a.tex_out) smem = ((smem + 15) & ~(size_t)15) + sizeof(float4) * kWtCells * kWarps2;
#define EVO_LAUNCH_K2(REC, MID)                                          \
  {                                                                      \
    static SmemOptIn cfg;                                                \
    cudaError_t e = set_smem(k_resolve<REC, MID>, smem, cfg);            \
    if (e != cudaSuccess) return e;                                      \
    k_resolve<REC, MID><<<grid, kThreads2, smem, st>>>(a);               \
  }
  if (a.tex_out && !a.mid_rec) return cudaErrorInvalidValue;
  if (a.ev.src) {
    if (a.tex_out) EVO_LAUNCH_K2(true, 2) else if (a.mid_rec) EVO_LAUNCH_K2(true, 1) else EVO_LAUNCH_K2(true, 0)
  } else {
    if (a.tex_out) EVO_LAUNCH_K2(false, 2) else if (a.mid_rec) EVO_LAUNCH_K2(false, 1) else EVO_LAUNCH_K2(false, 0)
  }
#undef EVO_LAUNCH_K2
#ifdef EVO_K2_SPLIT_CENSUS
  if (finish) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_census_finish(a.census, a.capacity, a.t, st, nullptr);
  }
#endif
  return cudaGetLastError();
}

// rcp_rn_ge1 against __frcp_rn over every float in [1, 2^125) (evo_debug_rcp_check)
__global__ void k_rcp_check(unsigned long long* mismatches) {
  unsigned long long bad = 0;
  for (unsigned long long b = 0x3f800000ull + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       b < 0x7e000000ull; b += (unsigned long long)gridDim.x * blockDim.x) {
    const float d = __uint_as_float((unsigned)b);
    bad += __float_as_uint(rcp_rn_ge1(d)) != __float_as_uint(__frcp_rn(d)) ? 1 : 0;
  }
  if (bad) atomicAdd(mismatches, bad);
}

cudaError_t debug_rcp_check(unsigned long long* host_out) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  cudaMemset(d, 0, sizeof(unsigned long long));
  k_rcp_check<<<num_sms() * 16, 256>>>(d);
  e = cudaMemcpy(host_out, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

cudaError_t debug_phase_cycles(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8);
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return e;
}

cudaError_t launch_census_finish(const Census& c, int capacity, long long t, cudaStream_t st, const int* skip) {
  const int blocks = (capacity + 255) / 256;
  k_census_finish<<<blocks, 256, 0, st>>>(c, capacity, t, skip);
  return cudaGetLastError();
}

cudaError_t launch_refresh_ghosts(const Planes& p, const StepGeom& g, cudaStream_t st) {
  const int blocks = (g.W + 255) / 256;
  k_refresh_ghosts<<<blocks, 256, 0, st>>>(p, g);
  return cudaGetLastError();
}

cudaError_t launch_wrap_mid(const Mid& m, const StepGeom& g, cudaStream_t st) {
  const int blocks = (g.W + 255) / 256;
  k_wrap_mid<<<blocks, 256, 0, st>>>(m, g);
  return cudaGetLastError();
}

cudaError_t launch_render_rgb(const Planes& f, const StepGeom& g, double norm_e, double norm_i, uint32_t* out,
                              cudaStream_t st) {
  const long long n = (long long)g.W * g.H;
  const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 16);
  k_render_rgb<<<blocks, 256, 0, st>>>(f, g, norm_e, norm_i, out);
  return cudaGetLastError();
}

cudaError_t launch_check_cells(int32_t* gi, uint8_t* rot, long long n, int capacity, int* bad, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 1023) / 1024;
  if (blocks > 1184) blocks = 1184;
  k_check_cells<<<(int)blocks, 256, 0, st>>>(gi, rot, n, capacity, bad);
  return cudaGetLastError();
}

cudaError_t launch_halo(const Planes& f, const Mid& m, const StepGeom& g, int which, bool pack, void* buf,
                        cudaStream_t st) {
  const int n = 2 * (which == 0 ? 5 : 3) * g.W;
  const int blocks = (n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256;
  if (pack)
    k_halo_pack<<<blocks, 256, 0, st>>>(f, m, g, which, static_cast<uint32_t*>(buf));
  else
    k_halo_unpack<<<blocks, 256, 0, st>>>(f, m, g, which, static_cast<const uint32_t*>(buf));
  return cudaGetLastError();
}

cudaError_t launch_halo_rec(float* tex, float* rec, const StepGeom& g, int which, bool pack, void* buf,
                            cudaStream_t st) {
  const int n = 2 * (which == 0 ? 5 : 3) * g.W;
  const int blocks = (n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256;
  if (pack)
    k_halo_pack_rec<<<blocks, 256, 0, st>>>(tex, rec, g, which, static_cast<uint32_t*>(buf));
  else
    k_halo_unpack_rec<<<blocks, 256, 0, st>>>(tex, rec, g, which, static_cast<const uint32_t*>(buf));
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
