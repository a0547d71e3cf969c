// Controller evaluation helpers for pass 1 (direct FFMA2 net, hidden-layer net, action epilogue).
#pragma once

#include "evoca_device.cuh"

namespace evo {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(u64 v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
// acc.{lo,hi} = fma(x, w.{lo,hi}, acc.{lo,hi}), each lane a correctly rounded fmaf
__device__ __forceinline__ void ffma2(u64& acc, float x, u64 w) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pk2(x, x)), "l"(w));
}

__device__ __forceinline__ float ld_na(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}

// Direct 45->13 controller over one unit of U same-genome cells (compact
// weights: W12 [45][12] + W1 [45] for actuator 12, bias [16]).  Per sensor k
// and cell: 6 FFMA2 + 1 FFMA, summation order k = 0..44 then + bias, per
// output exactly fmaf-chained (the FFMA2 lanes are independent fmaf).
template <bool kSmemW>
__device__ __forceinline__ float4 wload4(const float4* p) {
  if (kSmemW) {  // shared-memory weight table (explicit 32-bit shared address)
    float4 r;
    asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
        : "r"((unsigned)__cvta_generic_to_shared(p)));
    return r;
  }
  return __ldg(p);
}
// Two packed weights.  From shared memory one volatile 64-bit load (kept
// apart so ptxas does not fuse neighbours into an LDS.128): measured on
// B200, an LDS.64 whose lanes read a few genome rows is served in ONE
// wavefront iff every even/odd lane pair reads the same row - hence the
// bucketing pads genome groups to an even number of units - while an
// LDS.128 never takes fewer than two (tools/microbench/lds_sizes.cu).
template <bool kSmemW>
__device__ __forceinline__ u64 wload2(const float* p) {
  u64 r;
  if (kSmemW) {
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(r) : "r"((unsigned)__cvta_generic_to_shared(p)));
  } else {
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(r) : "l"(p));
  }
  return r;
}
template <bool kSmemW>
__device__ __forceinline__ float wload1(const float* p) {
  if (kSmemW) {
    float r;
    asm("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return r;
  }
  return __ldg(p);
}

template <int U, bool kSmemW = false, typename SM>
__device__ __forceinline__ void net_direct_unit(const SM& sm, const float* __restrict__ W12,
                                                const float* __restrict__ W1, const float* __restrict__ B,
                                                const int hb[U], const int rot[U], float out[U][kActuators]) {
  u64 acc[U][6];
  float acc12[U];
#pragma unroll
  for (int c = 0; c < U; ++c) {
#pragma unroll
    for (int p = 0; p < 6; ++p) acc[c][p] = 0ull;
    acc12[c] = 0.0f;
  }
  // software pipeline: the next slot's sensors are in flight while this
  // slot's FMAs run (shared-memory latency dominates otherwise)
  float xn[U][5];
#pragma unroll
  for (int c = 0; c < U; ++c) {
    const float4 v = sm.eic[hb[c]];
    xn[c][0] = v.x;
    xn[c][1] = v.y;
    xn[c][2] = v.z;
    xn[c][3] = v.w;
    xn[c][4] = sm.c2[hb[c]];
  }
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    float x[U][5];
#pragma unroll
    for (int c = 0; c < U; ++c)
#pragma unroll
      for (int ch = 0; ch < 5; ++ch) x[c][ch] = xn[c][ch];
    if (s < 8) {
#pragma unroll
      for (int c = 0; c < U; ++c) {
        const int nb = hb[c] + sm.slot_off[rot[c] * 9 + s + 1];
        const float4 v = sm.eic[nb];
        xn[c][0] = v.x;
        xn[c][1] = v.y;
        xn[c][2] = v.z;
        xn[c][3] = v.w;
        xn[c][4] = sm.c2[nb];
      }
    }
    const float* wrow = W12 + (size_t)s * 5 * 12;
    const float* w1row = W1 + s * 5;
#pragma unroll
    for (int ch = 0; ch < 5; ++ch) {
#ifdef EVO_DIAG_NO_WEIGHTS  // diagnostics builds only: results are wrong
      const u64 wq = pk2(s * 1e-3f, ch * 1e-3f);
      const u64 wp[6] = {wq, wq, wq, wq, wq, wq};
      const float w12 = 1e-3f;
#else
      u64 wp[6];
#pragma unroll
      for (int p = 0; p < 6; ++p) wp[p] = wload2<kSmemW>(wrow + ch * 12 + 2 * p);
      const float w12 = wload1<kSmemW>(w1row + ch);
#endif
#ifndef EVO_DIAG_NO_FMA
#pragma unroll
      for (int c = 0; c < U; ++c) {
#pragma unroll
        for (int p = 0; p < 6; ++p) ffma2(acc[c][p], x[c][ch], wp[p]);
        acc12[c] = fmaf(x[c][ch], w12, acc12[c]);
      }
#else
#pragma unroll
      for (int c = 0; c < U; ++c) acc12[c] += x[c][ch] + __uint_as_float((unsigned)wp[ch % 6]) + w12;
#endif
    }
  }
  const float4* b4 = reinterpret_cast<const float4*>(B);
  const float4 b0 = wload4<kSmemW>(b4), b1 = wload4<kSmemW>(b4 + 1), b2 = wload4<kSmemW>(b4 + 2),
               b3 = wload4<kSmemW>(b4 + 3);
  const float b[13] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w, b3.x};
#pragma unroll
  for (int c = 0; c < U; ++c) {
#pragma unroll
    for (int p = 0; p < 6; ++p) {
      float lo, hi;
      up2(acc[c][p], lo, hi);
      out[c][2 * p] = __fadd_rn(lo, b[2 * p]);
      out[c][2 * p + 1] = __fadd_rn(hi, b[2 * p + 1]);
    }
    out[c][12] = __fadd_rn(acc12[c], b[12]);
  }
}

// Hidden-layer controller 45->H(tanh)->13 for one cell (reference DenseParams):
// z1 = s.W1^T (k order) + b1, tanh, z2 = h.W2^T (h order) + b2.  Returns logits.
template <typename SM>
__device__ __forceinline__ void net_hidden_cell(const SM& sm, const Params& P, int g, int hb, int rot,
                                                float out[kActuators]) {
  float x[kSensors];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int nb = hb + sm.slot_off[rot * 9 + s];
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
  for (int j = 0; j < kActuators; ++j) out[j] = __fadd_rn(acc[j], b[j]);
}

struct ActSmem {
  float inv[kTileCells], liq[kTileCells], c0[kTileCells], c1[kTileCells], c2[kTileCells], xmax[kTileCells];
  uint8_t kstar[kTileCells];
};

// logits -> squashed actions in smem (spatial index p) and optional export
template <bool kExport>
__device__ __forceinline__ void finish_actions(ActSmem& act, const Pass1Args& a, int p, int x0, int y0,
                                               const float* z) {
  if (!kExport) {
    act.inv[p] = squash(z[0]);
    act.liq[p] = squash(z[1]);
    act.c0[p] = squash(z[2]);
    act.c1[p] = squash(z[3]);
    act.c2[p] = squash(z[4]);
    int ks;
    float xm;
    explore_pick(z + 5, ks, xm);
    act.xmax[p] = xm;
    act.kstar[p] = (uint8_t)ks;
  } else {
    float v[kActuators];
#pragma unroll
    for (int j = 0; j < kActuators; ++j) v[j] = squash(z[j]);
    act.inv[p] = v[0];
    act.liq[p] = v[1];
    act.c0[p] = v[2];
    act.c1[p] = v[3];
    act.c2[p] = v[4];
    int ks;
    float xm;
    explore_argmax(v + 5, ks, xm);
    act.xmax[p] = xm;
    act.kstar[p] = (uint8_t)ks;
    const int ty = p / kTileW, tx = p - ty * kTileW;
    const long long cell = (long long)(y0 + ty) * a.g.W + (x0 + tx);
    float* dst = a.act_out + cell * kActuators;
#pragma unroll
    for (int j = 0; j < kActuators; ++j) dst[j] = v[j];
    a.act_out_flag[cell] = 1;
  }
}

}  // namespace evo
