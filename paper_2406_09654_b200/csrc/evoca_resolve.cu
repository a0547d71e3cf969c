// Pass 2, streaming form (physics.py:286-343 resolve + adoption,
// 395-404 census): exploration resolved by each target pulling the shipments
// aimed at it, with the 3x3 neighbourhood held in REGISTERS instead of a
// shared-memory halo tile.  A measured alternative to k_resolve (built in
// with -DEVO_K2_STREAM): bit-identical, but 9.0 warp instructions per cell
// against 9.6 - every warp row runs the 19-comparator sort because some
// lane almost always has three or more arrivals - so 0.24 ms against
// 0.22 ms on config 3.
//
// A warp owns a strip of 30 columns (lanes 1..30; lanes 0 and 31 carry the
// wrapped halo columns) and walks down R rows.  Each lane keeps its column's
// proposal byte, shipped quantity and post-death genome for rows y-1, y, y+1
// in registers (one new row loaded per step, two rows ahead in flight); a
// cell's eight neighbours come from its own registers and from lanes x-1 and
// x+1 through warp shuffles (the three proposal bytes of a column travel as
// one packed word).  The arrival mask is bit d of the source's byte at
// (x - dx_d, y - dy_d); arrivals are summed in (quantity desc, global source
// asc) order - the reference's lexsort (physics.py:294) - via a 19-comparator
// sort of the eight quantity bit patterns (q >= +0, so bits order like
// values), the maximal quantity wins (exact ties: lowest global source
// index) and adopts iff q > infrastructure before (physics.py:325).  No
// shared-memory staging, no block barriers in the cell loop; the census
// histogram and the last-CTA epilogue are those of k_resolve.

#include "evoca_net.cuh"

namespace evo {

namespace {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsCols = 30;  // interior columns per warp strip
constexpr int kRsRows = 32;  // rows per warp task

__device__ __forceinline__ float canon(float q) { return __fadd_rn(q, 0.0f); }  // -0 -> +0

#define EVO_CE2(a, b)                   \
  {                                     \
    const unsigned hi_ = max(a, b);     \
    b = min(a, b);                      \
    a = hi_;                            \
  }

}  // namespace

template <bool kRecord>
__global__ void __launch_bounds__(kRsThreads, 4) k_resolve_rows(const Pass2Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* hist = reinterpret_cast<int*>(smem_raw);
  __shared__ int s_adopt;
  __shared__ bool s_last;
  const StepGeom& g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < a.capacity; b += kRsThreads) hist[b] = 0;
  if (tid == 0) s_adopt = 0;
  __syncthreads();
  const int strips = (g.W + kRsCols - 1) / kRsCols;
  const int blocks_y = (g.H + kRsRows - 1) / kRsRows;
  const int ntasks = strips * blocks_y;
  int my_adopt = 0;
  const unsigned full = 0xffffffffu;
  for (int task = blockIdx.x * kRsWarps + warp; task < ntasks; task += gridDim.x * kRsWarps) {
    const int xs = (task % strips) * kRsCols;
    const int y0 = (task / strips) * kRsRows;
    const int y1 = min(y0 + kRsRows, g.H);
    int x = xs - 1 + lane;  // this lane's column, wrapped (any width)
    x %= g.W;
    if (x < 0) x += g.W;
    const bool interior = lane >= 1 && lane <= kRsCols && xs + lane - 1 < g.W;
    auto load = [&](int y, unsigned& rp, float& q, int& gi) {  // y in -1..H (ghost rows)
      const unsigned o = (unsigned)((y + 1) * g.W + x);
      rp = __ldg(a.mid.rp + o);
      q = canon(__ldg(a.mid.q + o));
      gi = __ldg(a.mid.gi + o);
    };
    unsigned rpm, rp0, rpp, rpn;
    float qm, q0, qp, qn;
    int gm, g0, gp, gn;
    load(y0 - 1, rpm, qm, gm);
    load(y0, rp0, q0, g0);
    load(y0 + 1 <= g.H ? y0 + 1 : g.H, rpp, qp, gp);
    if (y0 + 2 <= g.H) load(y0 + 2, rpn, qn, gn);
#pragma unroll 1
    for (int y = y0; y < y1; ++y) {
      // own cell's infrastructure before arrivals and its rotation
      const unsigned oc = (unsigned)((y + 1) * g.W + x);
      const float before = __ldg(a.mid.I + oc);
      const int rot = __ldg(a.rot_front + oc);
      const unsigned P = rpm | (rp0 << 8) | (rpp << 16);
      const unsigned L = __shfl_up_sync(full, P, 1), R = __shfl_down_sync(full, P, 1);
      // bit d: the neighbour at (x - dx_d, y - dy_d) ships in direction d
      // (offsets physics.py:40-43: (1,0) (1,1) (0,1) (-1,1) (-1,0) (-1,-1) (0,-1) (1,-1))
      unsigned m = ((L >> 8) & 1u) | (L & 2u) | (P & 4u) | (R & 8u) | ((R >> 8) & 16u) | ((R >> 16) & 32u) |
                   ((P >> 16) & 64u) | ((L >> 16) & 128u);
      if (!interior) m = 0;
      const float qL0 = __shfl_up_sync(full, q0, 1), qLm = __shfl_up_sync(full, qm, 1),
                  qLp = __shfl_up_sync(full, qp, 1);
      const float qR0 = __shfl_down_sync(full, q0, 1), qRm = __shfl_down_sync(full, qm, 1),
                  qRp = __shfl_down_sync(full, qp, 1);
      const int gL0 = __shfl_up_sync(full, g0, 1), gLm = __shfl_up_sync(full, gm, 1), gLp = __shfl_up_sync(full, gp, 1);
      const int gR0 = __shfl_down_sync(full, g0, 1), gRm = __shfl_down_sync(full, gm, 1),
                gRp = __shfl_down_sync(full, gp, 1);
      const float qd[8] = {qL0, qLm, qm, qRm, qR0, qRp, qp, qLp};
      const int n = __popc(m);
      float acc = before;
      int gnew = g0, rnew = rot, wd = -1;
      float qw = 0.0f;
      if (__any_sync(full, n >= 2)) {
        // general: the present quantities sorted descending (absent: 0, last),
        // added in that order; exact ties only decide the winner
        unsigned qb[8];
        unsigned qmax = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          qb[d] = ((m >> d) & 1u) ? __float_as_uint(qd[d]) : 0u;
          qmax = max(qmax, qb[d]);
        }
        unsigned tie = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) tie |= (((m >> d) & 1u) && qb[d] == qmax) ? (1u << d) : 0u;
        wd = n ? __ffs(tie) - 1 : -1;
        if (tie & (tie - 1)) {  // exact tie on the maximum: lowest global source index wins
          unsigned best = 0xFFFFFFFFu;
          for (unsigned rest = tie; rest; rest &= rest - 1) {
            const int d = __ffs(rest) - 1;
            int sx = x - dir_dx(d);
            sx = sx < 0 ? sx + g.W : (sx >= g.W ? sx - g.W : sx);
            int grow = (int)g.row0 + y - dir_dy(d);
            grow = grow < 0 ? grow + g.Hg : (grow >= g.Hg ? grow - g.Hg : grow);
            const unsigned src = (unsigned)grow * (unsigned)g.W + (unsigned)sx;
            if (src < best) {
              best = src;
              wd = d;
            }
          }
        }
        EVO_CE2(qb[0], qb[1]) EVO_CE2(qb[2], qb[3]) EVO_CE2(qb[4], qb[5]) EVO_CE2(qb[6], qb[7])
        EVO_CE2(qb[0], qb[2]) EVO_CE2(qb[1], qb[3]) EVO_CE2(qb[4], qb[6]) EVO_CE2(qb[5], qb[7])
        EVO_CE2(qb[1], qb[2]) EVO_CE2(qb[5], qb[6])
        EVO_CE2(qb[0], qb[4]) EVO_CE2(qb[1], qb[5]) EVO_CE2(qb[2], qb[6]) EVO_CE2(qb[3], qb[7])
        EVO_CE2(qb[2], qb[4]) EVO_CE2(qb[3], qb[5])
        EVO_CE2(qb[1], qb[2]) EVO_CE2(qb[3], qb[4]) EVO_CE2(qb[5], qb[6])
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < n) acc = __fadd_rn(acc, __uint_as_float(qb[i]));
        qw = __uint_as_float(qmax);
      } else if (n == 1) {
        wd = __ffs(m) - 1;
        qw = qd[0];
#pragma unroll
        for (int d = 1; d < 8; ++d)
          if (wd == d) qw = qd[d];
        acc = __fadd_rn(acc, qw);
      }
      bool adopt = false;
      if (wd >= 0 && qw > before) {  // physics.py:325
        adopt = true;
        const int gd[8] = {gL0, gLm, gm, gRm, gR0, gRp, gp, gLp};
        gnew = gd[0];
#pragma unroll
        for (int d = 1; d < 8; ++d)
          if (wd == d) gnew = gd[d];
        rnew = wd;
      }
      if (interior) {
        const long long cell = (long long)y * g.W + x;
        if (kRecord) {
          if (adopt) {
            int sx = x - dir_dx(wd);
            sx = sx < 0 ? sx + g.W : (sx >= g.W ? sx - g.W : sx);
            int grow = (int)g.row0 + y - dir_dy(wd);
            grow = grow < 0 ? grow + g.Hg : (grow >= g.Hg ? grow - g.Hg : grow);
            a.ev.src[cell] = (long long)grow * g.W + sx;
            a.ev.q[cell] = qw;
            a.ev.def[cell] = g0;
          } else {
            a.ev.src[cell] = -1;
          }
        }
        my_adopt += adopt ? 1 : 0;
        a.back.I[oc] = acc;
        a.back.gi[oc] = gnew;
        a.back.rot[oc] = (uint8_t)rnew;
        if (g.own_ghosts && y == 0) {  // wrapped ghost copies of a single strip
          const unsigned og = (unsigned)((g.H + 1) * g.W + x);
          a.back.I[og] = acc;
          a.back.gi[og] = gnew;
          a.back.rot[og] = (uint8_t)rnew;
        }
        if (g.own_ghosts && y == g.H - 1) {
          a.back.I[x] = acc;
          a.back.gi[x] = gnew;
          a.back.rot[x] = (uint8_t)rnew;
        }
        if (gnew >= 0 && gnew < a.capacity) atomicAdd(&hist[gnew], 1);
      }
      // slide the window one row down (row y + 3 in flight)
      rpm = rp0, qm = q0, gm = g0;
      rp0 = rpp, q0 = qp, g0 = gp;
      rpp = rpn, qp = qn, gp = gn;
      if (y + 3 <= g.H) load(y + 3, rpn, qn, gn);
    }
  }
  for (int off = 16; off > 0; off >>= 1) my_adopt += __shfl_xor_sync(full, my_adopt, off);
  if (lane == 0 && my_adopt) atomicAdd(&s_adopt, my_adopt);
  __syncthreads();
  if (tid == 0 && s_adopt) atomicAdd((unsigned long long*)&a.census.stats[0], (unsigned long long)s_adopt);
  for (int b = tid; b < a.capacity; b += kRsThreads)
    if (hist[b]) atomicAdd(&a.census.counts[b], hist[b]);
  if (!a.run_census) return;
  // last CTA: census epilogue (physics.py:395-404, neuroevo.py:521-542)
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
  for (int b = tid; b < a.capacity; b += kRsThreads) {
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
  for (int off = 16; off > 0; off >>= 1) dead += __shfl_xor_sync(full, dead, off);
  if ((tid & 31) == 0 && dead) atomicAdd((unsigned long long*)&a.census.stats[1], (unsigned long long)dead);
  if (tid == 0) *a.census.done = 0u;
}

cudaError_t launch_resolve_rows(const Pass2Args& a, int num_sms, cudaStream_t st) {
  const int strips = (a.g.W + kRsCols - 1) / kRsCols;
  const int tasks = strips * ((a.g.H + kRsRows - 1) / kRsRows);
  int grid = num_sms * 4;
  const int need = (tasks + kRsWarps - 1) / kRsWarps;
  if (grid > need) grid = need;
  const size_t smem = (size_t)a.capacity * sizeof(int);
  static int configured[2][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  const int r = a.ev.src ? 1 : 0;
  if (smem > 48 * 1024 && configured[r][dev] < (int)smem) {
    cudaError_t e = cudaFuncSetAttribute(r ? k_resolve_rows<true> : k_resolve_rows<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[r][dev] = (int)smem;
  }
  if (r)
    k_resolve_rows<true><<<grid, kRsThreads, smem, st>>>(a);
  else
    k_resolve_rows<false><<<grid, kRsThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace evo
