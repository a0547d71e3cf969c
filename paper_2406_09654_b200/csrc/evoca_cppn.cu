// Batched CPPN expression: the reference's
// generate_network (/root/reference/pkg/src/evoca/hypernet.py:183-220) for
// many admitted genomes in one launch, writing the dense controller tables
// of their pool slots in place.
//
// The host linearises each genome (paper_2406_09654_b200/neat.py:
// compile_programs): nodes in the reference's Kahn order (hypernet.py:
// 100-125), each compute node with its ENABLED incoming edges in
// connection-list order.  One thread evaluates one weight query: node values
// live in shared memory ([node][thread], conflict-free), every incoming sum
// is total = total + w * v in float64 with separately rounded multiply and
// add (no FMA contraction, hypernet.py:150-153), activations in float64
// (hypernet.py:90-97), then the threshold-and-rescale expression
// (hypernet.py:168-180) and the float32 cast.
//
// Query blocks (hypernet.py:203-217), per genome, dst-major:
//   direct 45->13 (hidden == 0): 13 x 45 (input -> actuator, weight signal),
//                                13 bias queries ((0,0) -> actuator, bias signal)
//   hidden H:  H x 45 (input -> hidden), 13 x H (hidden -> actuator),
//              H + 13 bias queries.

#include "evoca_internal.h"

namespace evo {

__device__ __forceinline__ double cppn_act(int code, double x) {
  switch (code) {
    case 0: return sin(x);                                          // sine
    case 1: return exp(-__dmul_rn(x, x));                           // gaussian: exp(-square(x))
    case 2: return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));         // sigmoid
    case 3: return tanh(x);                                         // tanh
    case 4: return x;                                               // identity
    default: return fabs(x);                                        // abs
  }
}

// _express: |s| <= tau -> 0; else sign(s) * min((|s| - tau) / (1 - tau), 1) * w_max;
// non-finite -> 0; float32 cast.
__device__ __forceinline__ float cppn_express(double s, double tau, double w_max) {
  if (!isfinite(s)) return 0.0f;
  const double mag = fabs(s);
  if (!(mag > tau)) return 0.0f;
  const double sgn = s > 0.0 ? 1.0 : (s < 0.0 ? -1.0 : 0.0);
  const double r = fmin(__ddiv_rn(__dsub_rn(mag, tau), __dsub_rn(1.0, tau)), 1.0);
  return __double2float_rn(__dmul_rn(__dmul_rn(sgn, r), w_max));
}

__global__ void k_express_cppn(const CppnBatch b, Params net, float* wA, float* bA, float* wB, float* bB) {
  extern __shared__ double vals[];  // [max_nodes][blockDim.x]
  const int gidx = blockIdx.y;
  const int slot = b.slots[gidx];
  const int H = net.hidden, hp = net.hpad;
  const int n_in = kSensors;
  const double* cin = b.coords;                  // (45, 2)
  const double* chid = b.coords + 2 * n_in;      // (H, 2)
  const double* cout = chid + 2 * H;             // (13, 2)
  const int nw1 = H > 0 ? H * n_in : kActuators * n_in;
  const int nw2 = H > 0 ? kActuators * H : 0;
  const int nq = nw1 + nw2 + (H + kActuators);
  const int n0 = b.node_off[gidx], n1 = b.node_off[gidx + 1];
  const int out0 = b.outs[2 * gidx], out1 = b.outs[2 * gidx + 1];
  const int T = blockDim.x;
  for (int qi = blockIdx.x * T + threadIdx.x; qi < nq; qi += gridDim.x * T) {
    double q[5];
    int which, r = qi;
    const double *src, *dst;
    if (r < nw1) {
      const int d = r / n_in, s = r - d * n_in;
      src = cin + 2 * s;
      dst = H > 0 ? chid + 2 * d : cout + 2 * d;
      which = 0;
    } else if ((r -= nw1) < nw2) {
      const int d = r / H, s = r - d * H;
      src = chid + 2 * s;
      dst = cout + 2 * d;
      which = 0;
    } else {
      r -= nw2;
      src = nullptr;
      dst = r < H ? chid + 2 * r : cout + 2 * (r - H);
      which = 1;
    }
    q[0] = src ? src[0] : 0.0;
    q[1] = src ? src[1] : 0.0;
    q[2] = dst[0];
    q[3] = dst[1];
    q[4] = 1.0;
    for (int i = n0; i < n1; ++i) {
      const int4 nd = b.nodes[i];
      double v;
      if (nd.x < 0) {
        v = q[nd.y];
      } else {
        double total = 0.0;
        for (int e = nd.z; e < nd.w; ++e)
          total = __dadd_rn(total, __dmul_rn(b.edge_w[e], vals[b.edge_src[e] * T + threadIdx.x]));
        v = cppn_act(nd.x, total);
      }
      vals[(i - n0) * T + threadIdx.x] = v;
    }
    const float w = cppn_express(vals[(which ? out1 : out0) * T + threadIdx.x], b.tau, b.w_max);
    // scatter into the slot's device tables (layouts of evo_set_params)
    r = qi;
    if (H == 0) {
      if (r < nw1) {
        const int j = r / n_in, k = r - j * n_in;
        if (j < 12)
          wA[((size_t)slot * n_in + k) * 12 + j] = w;
        else
          wB[(size_t)slot * n_in + k] = w;
      } else {
        bA[(size_t)slot * kOutPad + (r - nw1)] = w;
      }
    } else {
      if (r < nw1) {
        const int h = r / n_in, k = r - h * n_in;
        wA[((size_t)slot * n_in + k) * hp + h] = w;
      } else if ((r -= nw1) < nw2) {
        const int j = r / H, h = r - j * H;
        wB[((size_t)slot * hp + h) * kOutPad + j] = w;
      } else if ((r -= nw2) < H) {
        bA[(size_t)slot * hp + r] = w;
      } else {
        bB[(size_t)slot * kOutPad + (r - H)] = w;
      }
    }
  }
  // zero padding (hidden rows H..hpad-1, actuator columns 13..15) once per genome
  if (blockIdx.x == 0) {
    if (H == 0) {
      for (int j = kActuators + threadIdx.x; j < kOutPad; j += T) bA[(size_t)slot * kOutPad + j] = 0.0f;
    } else {
      const int ph = hp - H;
      for (int i = threadIdx.x; i < ph * (n_in + 1 + kOutPad); i += T) {
        const int h = H + i % ph, part = i / ph;
        if (part < n_in)
          wA[((size_t)slot * n_in + part) * hp + h] = 0.0f;
        else if (part == n_in)
          bA[(size_t)slot * hp + h] = 0.0f;
        else
          wB[((size_t)slot * hp + h) * kOutPad + (part - n_in - 1)] = 0.0f;
      }
      for (int i = threadIdx.x; i < hp * (kOutPad - kActuators); i += T) {
        const int h = i / (kOutPad - kActuators), j = kActuators + i % (kOutPad - kActuators);
        wB[((size_t)slot * hp + h) * kOutPad + j] = 0.0f;
      }
      for (int j = kActuators + threadIdx.x; j < kOutPad; j += T) bB[(size_t)slot * kOutPad + j] = 0.0f;
    }
  }
}

int cppn_threads(int max_nodes) {
  // node values in shared memory: max_nodes * threads * 8 B <= 96 KB
  int t = 256;
  while (t > 32 && (size_t)max_nodes * t * 8 > 96 * 1024) t >>= 1;
  return (size_t)max_nodes * t * 8 > 96 * 1024 ? 0 : t;
}

cudaError_t launch_express_cppn(const CppnBatch& b, const Params& net, float* wA, float* bA, float* wB, float* bB,
                                cudaStream_t st) {
  if (b.n == 0) return cudaSuccess;
  const int T = cppn_threads(b.max_nodes);
  const size_t smem = (size_t)(b.max_nodes > 0 ? b.max_nodes : 1) * T * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_express_cppn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int H = net.hidden;
  const int nq = H > 0 ? H * kSensors + kActuators * H + H + kActuators : kActuators * kSensors + kActuators;
  dim3 grid((nq + T - 1) / T, b.n);
  k_express_cppn<<<grid, T, smem, st>>>(b, net, wA, bA, wB, bB);
  return cudaGetLastError();
}

}  // namespace evo
