// Gather-path helpers shared by the direct (evoca_gather.cu) and hidden-layer
// (evoca_hidden_tc.cu) nets: the 32-byte sense-texture record of a cell
// {E, I, C0, C1, C2, 0, 0, 0} (k_gs_count) and the sorted-list entry
// (rot << 29) | (y << 15) | x (k_gs_scatter).
#pragma once

#include "evoca_device.cuh"

namespace evo {
namespace gs {

struct f8r {
  float v[8];
};
// Sense texture record {E, C0, C1, C2 | I, 0, 0, 0}: sensor channel ch (E, I,
// C0, C1, C2: engine.py:164-190) sits at index tex_ch(ch).  The first half
// equals the first half of a pass-1 record (FusedPhysics), so pass 2 of a
// fused step can write the next step's texture from what it holds.
__host__ __device__ constexpr int tex_ch(int ch) { return ch == 0 ? 0 : (ch == 1 ? 4 : ch - 1); }
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
  int rot;
};
__device__ __forceinline__ GCell gcell(uint32_t e, int W) {
  GCell c;
  const int y = (int)((e >> 15) & 0x3FFFu), x = (int)(e & 0x7FFFu);
  c.rot = (int)(e >> 29);
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

}  // namespace gs
}  // namespace evo
