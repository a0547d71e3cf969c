// Observables of the device front buffer (metrics.py), bit-identical to the
// reference's numpy / math.fsum results:
//
//  * multi-scale complexity (metrics.py:57-103): the 2x2 block-mean pyramid
//    of a power-of-two crop in f64 (members sorted, ((q0+q1)+(q2+q3))*0.25),
//    and the overlaps math.fsum(fa*fb)/side^2 of the upsampled scales.  An
//    upsampled overlap repeats every distinct product 4^k times, so its fsum
//    is 4^k times the correctly rounded EXACT sum of the distinct products;
//    that sum is accumulated exactly in a fixed-point superaccumulator
//    (every double is an integer multiple of 2^-1074: 68 signed 32-bit
//    digits held in 64-bit slots absorb 2^31 additions without carries) and
//    rounded half-to-even once at the end, which is what fsum returns.
//  * float64 totals of the energy / infrastructure planes (metrics.py:200-213,
//    numpy sum(dtype=float64)): numpy casts through 8192-element buffers and
//    adds each buffer's pairwise sum (blocks of <= 128 with eight
//    accumulators, halving above) to the running total in order; restated
//    here chunk by chunk.

#include <cuda_runtime.h>

#include <cstdint>

#include "evoca_internal.h"

namespace evo {
namespace {

constexpr int kDigits = 68;  // 32-bit digits of X = sum * 2^1074 (2176 bits)

// Add p (exactly) into a digit accumulator.
__device__ __forceinline__ void acc_add(long long* acc, double p) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(p);
  const int e = (int)((bits >> 52) & 0x7FF);
  unsigned long long m = bits & 0xFFFFFFFFFFFFFull;
  if (e == 0x7FF) return;  // inf / nan: not produced by finite planes
  int s;
  if (e == 0) {
    s = 0;  // subnormal: m * 2^-1074
  } else {
    m |= 1ull << 52;
    s = e - 1;  // (2^52 + f) * 2^(e-1075) = m * 2^(e-1) * 2^-1074
  }
  if (m == 0) return;
  const bool neg = bits >> 63;
  const int j = s >> 5, off = s & 31;
  const unsigned long long lo = m << off;                       // bits [0, 64)
  const unsigned long long hi = off ? (m >> (64 - off)) : 0ull;  // bits [64, 85)
  const long long d0 = (long long)(lo & 0xFFFFFFFFull), d1 = (long long)(lo >> 32), d2 = (long long)hi;
  unsigned long long* a = reinterpret_cast<unsigned long long*>(acc);
  if (d0) atomicAdd(a + j, (unsigned long long)(neg ? -d0 : d0));
  if (d1) atomicAdd(a + j + 1, (unsigned long long)(neg ? -d1 : d1));
  if (d2) atomicAdd(a + j + 2, (unsigned long long)(neg ? -d2 : d2));
}

// value of level L at (y, x): level 0 is the f32 plane crop, higher levels f64
struct Level {
  const float* plane;  // level 0: row y at plane + (y0 + y + 1) * W + x0
  const double* f;     // levels >= 1: side_l x side_l
  int W, x0, y0, side;
  __device__ __forceinline__ double at(int y, int x) const {
    return plane ? (double)plane[(long long)(y0 + y + 1) * W + x0 + x] : f[(long long)y * side + x];
  }
};

__device__ __forceinline__ void sort2(double& a, double& b) {
  const double lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}

__global__ void k_block_means(const Level src, double* dst) {
  const int s = src.side >> 1;
  const long long n = (long long)s * s;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / s), x = (int)(i - (long long)y * s);
    double q0 = src.at(2 * y, 2 * x), q1 = src.at(2 * y, 2 * x + 1), q2 = src.at(2 * y + 1, 2 * x),
           q3 = src.at(2 * y + 1, 2 * x + 1);
    // ascending order (np.sort over the four members)
    sort2(q0, q1);
    sort2(q2, q3);
    sort2(q0, q2);
    sort2(q1, q3);
    sort2(q1, q2);
    dst[i] = __dmul_rn(__dadd_rn(__dadd_rn(q0, q1), __dadd_rn(q2, q3)), 0.25);
  }
}

// exact sum of a_i * b_parent(i) over level a (b = a: squares; b one level
// coarser: the cross overlap)
__global__ void k_overlap_sum(const Level a, const Level b, int coarser, long long* acc_out) {
  __shared__ long long acc[kDigits];
  for (int i = threadIdx.x; i < kDigits; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const int s = a.side;
  const long long n = (long long)s * s;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / s), x = (int)(i - (long long)y * s);
    const double va = a.at(y, x);
    const double vb = coarser ? b.at(y >> 1, x >> 1) : va;
    acc_add(acc, __dmul_rn(va, vb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kDigits; i += blockDim.x)
    if (acc[i]) atomicAdd(reinterpret_cast<unsigned long long*>(acc_out) + i, (unsigned long long)acc[i]);
}

// bits [pos, pos + 64) of the non-negative big integer held in 32-bit digits
__device__ unsigned long long big_bits(const unsigned* d, int pos) {
  unsigned long long r = 0;
  for (int k = 0; k < 3; ++k) {
    const int j = (pos >> 5) + k;
    if (j < 0 || j >= kDigits + 2) continue;
    const unsigned long long v = d[j];
    const int sh = j * 32 - pos;  // position of digit j relative to pos
    if (sh >= 64 || sh <= -32) continue;
    r |= sh >= 0 ? (v << sh) : (v >> -sh);
  }
  return r;
}

// correctly rounded (half to even) value of each accumulated sum
__global__ void k_exact_finalize(const long long* accs, int nsum, double* out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsum) return;
  const long long* a = accs + (long long)q * kDigits;
  unsigned d[kDigits + 2];
  long long carry = 0;
  for (int j = 0; j < kDigits; ++j) {
    const long long v = a[j] + carry;  // |a[j]| < 2^63 - 2^33: no overflow
    d[j] = (unsigned)(v & 0xFFFFFFFFll);
    carry = v >> 32;  // arithmetic
  }
  d[kDigits] = (unsigned)(carry & 0xFFFFFFFFll);
  d[kDigits + 1] = (unsigned)((carry >> 32) & 0xFFFFFFFFll);
  const bool neg = carry < 0;
  if (neg) {  // two's complement negate
    unsigned long long c = 1;
    for (int j = 0; j < kDigits + 2; ++j) {
      const unsigned long long v = (unsigned long long)(~d[j]) + c;
      d[j] = (unsigned)v;
      c = v >> 32;
    }
  }
  int top = -1;
  for (int j = kDigits + 1; j >= 0; --j)
    if (d[j]) {
      top = j * 32 + 31 - __clz(d[j]);
      break;
    }
  double r;
  if (top < 0) {
    r = 0.0;
  } else if (top < 53) {
    r = (double)big_bits(d, 0) * 0x1p-1074;  // exact: below 2^53 * 2^-1074 (subnormal range)
  } else {
    const int shift = top - 52;
    unsigned long long t = big_bits(d, shift) & ((1ull << 53) - 1);
    const bool half = (big_bits(d, shift - 1) & 1ull) != 0;
    bool sticky = false;
    for (int j = 0; j <= (shift - 2) >> 5 && !sticky; ++j) {
      unsigned v = d[j];
      const int hi_bit = shift - 2 - j * 32;  // keep bits [j*32, shift-1)
      if (hi_bit < 31) v &= (hi_bit >= 0) ? ((2u << hi_bit) - 1u) : 0u;
      sticky = v != 0;
    }
    int sh = shift;
    if (half && (sticky || (t & 1ull))) {
      ++t;
      if (t >> 53) {
        t >>= 1;
        ++sh;
      }
    }
    r = ldexp((double)t, sh - 1074);
  }
  out[q] = neg ? -r : r;
}

// numpy pairwise sum (loops_utils.h.src pairwise_sum) of n f64-cast floats
__device__ double np_pairwise(const float* a, long long n) {
  // explicit stack of (offset, count) segments, left before right
  long long st_off[32], st_n[32];
  double st_val[32];
  int st_state[32];  // 0: not expanded, 1: left done
  int sp = 0;
  st_off[0] = 0;
  st_n[0] = n;
  st_state[0] = 0;
  double ret = 0.0;
  bool have_ret = false;
  while (sp >= 0) {
    const long long o = st_off[sp], m = st_n[sp];
    if (st_state[sp] == 0 && m > 128) {
      long long n2 = m / 2;
      n2 -= n2 % 8;
      st_state[sp] = 1;
      ++sp;
      st_off[sp] = o;
      st_n[sp] = n2;
      st_state[sp] = 0;
      continue;
    }
    double v;
    if (st_state[sp] == 0) {  // leaf
      if (m < 8) {
        v = 0.0;
        for (long long i = 0; i < m; ++i) v = __dadd_rn(v, (double)a[o + i]);
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = (double)a[o + j];
        long long i = 8;
        for (; i < m - (m % 8); i += 8)
          for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], (double)a[o + i + j]);
        v = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < m; ++i) v = __dadd_rn(v, (double)a[o + i]);
      }
    } else if (st_state[sp] == 1) {  // left child finished: expand the right one
      long long n2 = m / 2;
      n2 -= n2 % 8;
      st_val[sp] = ret;
      st_state[sp] = 2;
      ++sp;
      st_off[sp] = o + n2;
      st_n[sp] = m - n2;
      st_state[sp] = 0;
      continue;
    } else {  // both children finished
      v = __dadd_rn(st_val[sp], ret);
    }
    ret = v;
    have_ret = true;
    --sp;
  }
  (void)have_ret;
  return ret;
}

constexpr long long kNpBuf = 8192;  // numpy's default ufunc buffer size

__global__ void k_plane_chunks(const float* plane, long long n, double* chunk_sums) {
  const long long nch = (n + kNpBuf - 1) / kNpBuf;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nch; c += (long long)gridDim.x * blockDim.x) {
    const long long o = c * kNpBuf;
    chunk_sums[c] = np_pairwise(plane + o, n - o < kNpBuf ? n - o : kNpBuf);
  }
}

__global__ void k_chunks_total(const double* chunk_sums, long long nch, double* out) {
  if (blockIdx.x || threadIdx.x) return;
  double r = 0.0;
  for (long long c = 0; c < nch; ++c) r = __dadd_rn(r, chunk_sums[c]);
  *out = r;
}

}  // namespace

int msc_side(int W, int H) {
  int s = 1;
  while (2 * s <= W && 2 * s <= H) s *= 2;
  return s;
}

long long msc_workspace_doubles(int side) {
  long long n = 0;
  for (int s = side / 2; s >= 1; s /= 2) n += (long long)s * s;
  return n;
}

cudaError_t launch_msc(const float* plane, int W, int H, int n_scales, double* work, long long* accs, double* out,
                       int* k_max_out, cudaStream_t st) {
  const int side = msc_side(W, H);
  int max_scales = 0;
  while ((1 << (max_scales + 1)) <= side) ++max_scales;
  const int k_max = n_scales > 0 && n_scales < max_scales ? n_scales : max_scales;
  *k_max_out = k_max;
  if (k_max < 1) return cudaSuccess;
  Level lv[32];
  lv[0].plane = plane;
  lv[0].f = nullptr;
  lv[0].W = W;
  lv[0].x0 = (W - side) / 2;
  lv[0].y0 = (H - side) / 2;
  lv[0].side = side;
  double* w = work;
  for (int k = 1; k <= k_max; ++k) {
    const int s = side >> k;
    lv[k].plane = nullptr;
    lv[k].f = w;
    lv[k].W = 0;
    lv[k].x0 = lv[k].y0 = 0;
    lv[k].side = s;
    const long long n = (long long)s * s;
    const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    k_block_means<<<blocks, 256, 0, st>>>(lv[k - 1], w);
    w += n;
  }
  const int nsum = 2 * k_max + 1;
  cudaError_t e = cudaMemsetAsync(accs, 0, sizeof(long long) * kDigits * nsum, st);
  if (e != cudaSuccess) return e;
  for (int k = 0; k <= k_max; ++k) {
    const long long n = (long long)lv[k].side * lv[k].side;
    const int blocks = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
    k_overlap_sum<<<blocks, 256, 0, st>>>(lv[k], lv[k], 0, accs + (long long)k * kDigits);
    if (k < k_max) k_overlap_sum<<<blocks, 256, 0, st>>>(lv[k], lv[k + 1], 1, accs + (long long)(k_max + 1 + k) * kDigits);
  }
  k_exact_finalize<<<1, 64, 0, st>>>(accs, nsum, out);
  return cudaGetLastError();
}

long long plane_sum_chunks(long long n) { return (n + kNpBuf - 1) / kNpBuf; }

cudaError_t launch_plane_sum(const float* plane, long long n, double* chunks, double* out, cudaStream_t st) {
  const long long nch = plane_sum_chunks(n);
  const int blocks = (int)((nch + 63) / 64);
  k_plane_chunks<<<blocks > 0 ? blocks : 1, 64, 0, st>>>(plane, n, chunks);
  k_chunks_total<<<1, 32, 0, st>>>(chunks, nch, out);
  return cudaGetLastError();
}

int msc_digits() { return kDigits; }

}  // namespace evo
