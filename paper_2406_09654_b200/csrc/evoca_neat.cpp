// Host NEAT for the radiation feed (north_star (6): topology mutation and
// crossover stay on the host) as native code: batched mutation of pattern
// networks (reference neuroevo.py:233-299 `mutate`) and their linearisation
// into evo_express_cppn programs (hypernet.py:100-155 topological order and
// connection-list summation order).  Replaces the per-genome Python loops
// whose NumPy calls (~0.5 us each, ~150 per genome) made one config-3
// radiation event with 256 parents cost ~45 ms.
//
// Random draws reproduce NumPy's Generator(Philox(key)) bit for bit:
//   * Philox4x64-10, counter incremented before each 4-word block, words
//     handed out in order (numpy/random/src/philox);
//   * next_uint32 hands out the low half of a fresh word and keeps the high
//     half for the next 32-bit request (Philox bit generator buffering);
//   * random() = (u64 >> 11) * 2^-53, uniform(a, b) = a + (b - a) * random();
//   * normal(loc, scale) = loc + scale * z with NumPy's 256-layer ziggurat
//     (tables extracted from NumPy, evoca_ziggurat.h);
//   * integers(n) = Lemire's bounded method on 32-bit draws (n <= 2^32).
// tools/ + tests/test_neat_native.py pin every distribution and whole
// mutations against NumPy and this package's Python mutate.

#include <stdint.h>

#include <algorithm>
#include <cstdint>
#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "evoca_b200.h"
#include "evoca_ziggurat.h"

namespace {

struct Philox {
  uint64_t ctr[4] = {0, 0, 0, 0};
  uint64_t key[2];
  uint64_t buf[4];
  int pos = 4;
  bool has32 = false;
  uint32_t half = 0;

  Philox(uint64_t k0, uint64_t k1) { key[0] = k0, key[1] = k1; }

  static inline void mulhilo(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
    const unsigned __int128 p = (unsigned __int128)a * b;
    hi = (uint64_t)(p >> 64);
    lo = (uint64_t)p;
  }
  void block() {
    if (++ctr[0] == 0 && ++ctr[1] == 0 && ++ctr[2] == 0) ++ctr[3];
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
      uint64_t hi0, lo0, hi1, lo1;
      mulhilo(0xD2E7470EE14C6C93ull, c0, hi0, lo0);
      mulhilo(0xCA5A826395121157ull, c2, hi1, lo1);
      const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
      c0 = n0, c1 = lo1, c2 = n2, c3 = lo0;
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    buf[0] = c0, buf[1] = c1, buf[2] = c2, buf[3] = c3;
    pos = 0;
  }
  uint64_t u64() {
    if (pos >= 4) block();
    return buf[pos++];
  }
  uint32_t u32() {
    if (has32) {
      has32 = false;
      return half;
    }
    const uint64_t v = u64();
    has32 = true;
    half = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  double random() { return (double)(u64() >> 11) * (1.0 / 9007199254740992.0); }
  double uniform(double a, double b) { return a + (b - a) * random(); }
  double standard_normal() {
    const double kR = 3.6541528853610087963519472518, kInvR = 1.0 / kR;
    for (;;) {
      uint64_t r = u64();
      const int idx = (int)(r & 0xff);
      r >>= 8;
      const int sign = (int)(r & 1);
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
      double x = (double)rabs * evo::kZigWi[idx];
      if (sign) x = -x;
      if (rabs < evo::kZigKi[idx]) return x;
      if (idx == 0) {
        for (;;) {
          const double xx = -kInvR * std::log1p(-random());
          const double yy = -std::log1p(-random());
          if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(kR + xx) : kR + xx;
        }
      }
      if ((evo::kZigFi[idx - 1] - evo::kZigFi[idx]) * random() + evo::kZigFi[idx] < std::exp(-0.5 * x * x)) return x;
    }
  }
  double normal(double loc, double scale) { return loc + scale * standard_normal(); }
  int64_t integers(int64_t n) {  // [0, n), 1 <= n <= 2^32
    const uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    const uint64_t excl = (uint64_t)rng + 1;
    uint64_t m = (uint64_t)u32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
      while (left < thr) {
        m = (uint64_t)u32() * excl;
        left = (uint32_t)m;
      }
    }
    return (int64_t)(m >> 32);
  }
};

struct Conn {
  int64_t innov, src, dst;
  double w;
  uint8_t en;
};
struct Node {
  int64_t id;
  int8_t role, act;  // role 0 input, 1 hidden, 2 output
};

// is `src` reachable from `dst` over every gene (disabled ones included)
bool creates_cycle(const std::vector<Conn>& cs, int64_t src, int64_t dst) {
  if (src == dst) return true;
  std::vector<int64_t> stack{dst}, seen{dst};
  while (!stack.empty()) {
    const int64_t n = stack.back();
    stack.pop_back();
    if (n == src) return true;
    for (const Conn& c : cs)
      if (c.src == n && std::find(seen.begin(), seen.end(), c.dst) == seen.end()) {
        seen.push_back(c.dst);
        stack.push_back(c.dst);
      }
  }
  return false;
}

thread_local std::string g_neat_err;

constexpr int64_t kDeferredNode = INT64_MAX;  // = EVO_NEAT_DEFERRED_NODE

}  // namespace

extern "C" {

EVO_API const char* evo_neat_last_error(void) { return g_neat_err.c_str(); }

}  // extern "C"

namespace {

// deferred: new genes keep placeholder numbers instead of drawing from the
// shared counter - the k-th new connection of a genome gets innovation
// -1 - k, its new node id kDeferredNode (larger than every existing id, as
// the real one will be) - so the draws of a batch can run before it is known
// which genomes will be admitted (the numbering is done afterwards, in the
// admitted genomes' order: neat.number_deferred)
int mutate_impl(bool deferred, int n, const uint64_t* keys, const double* rates, int64_t* counter,
                const int32_t* node_off, const int64_t* node_id, const int8_t* node_role, const int8_t* node_act,
                const int32_t* conn_off, const int64_t* c_innov, const int64_t* c_src, const int64_t* c_dst,
                const double* c_w, const uint8_t* c_en, int32_t* o_node_off, int64_t* o_node_id, int8_t* o_node_role,
                int8_t* o_node_act, int32_t* o_conn_off, int64_t* o_innov, int64_t* o_src, int64_t* o_dst,
                double* o_w, uint8_t* o_en) {
  if (n < 0 || (n > 0 && (!keys || !rates || (!deferred && !counter) || !node_off || !conn_off))) {
    g_neat_err = "evo_neat_mutate: bad arguments";
    return EVO_EINVAL;
  }
  const double p_reset = rates[0], p_perturb = rates[1], sigma = rates[2], p_conn = rates[3], p_node = rates[4],
               p_toggle = rates[5];
  int64_t next_innov = deferred ? 0 : counter[0], next_node = deferred ? 0 : counter[1];
  std::vector<Conn> cs;
  std::vector<Node> ns;
  int32_t on = 0, oc = 0;
  o_node_off[0] = 0;
  o_conn_off[0] = 0;
  for (int g = 0; g < n; ++g) {
    Philox rng(keys[2 * g], keys[2 * g + 1]);
    int64_t k_new = 0;  // deferred: placeholders restart per genome
    auto new_innov = [&]() { return deferred ? -1 - k_new++ : next_innov++; };
    cs.clear();
    ns.clear();
    for (int32_t i = conn_off[g]; i < conn_off[g + 1]; ++i)
      cs.push_back({c_innov[i], c_src[i], c_dst[i], c_w[i], c_en[i]});
    for (int32_t i = node_off[g]; i < node_off[g + 1]; ++i) ns.push_back({node_id[i], node_role[i], node_act[i]});
    // weights: reset, else perturb (neuroevo.py mutate, first loop)
    for (Conn& c : cs) {
      if (rng.random() < p_reset)
        c.w = rng.uniform(-1.0, 1.0);
      else if (rng.random() < p_perturb)
        c.w = c.w + rng.normal(0.0, sigma);
    }
    for (Conn& c : cs)
      if (rng.random() < p_toggle) c.en = !c.en;
    if (rng.random() < p_conn) {
      std::vector<Node> ord(ns);
      std::sort(ord.begin(), ord.end(), [](const Node& a, const Node& b) { return a.id < b.id; });
      std::vector<std::pair<int64_t, int64_t>> cands;
      for (const Node& s : ord) {
        if (s.role == 2) continue;
        for (const Node& d : ord) {
          if (d.role == 0) continue;
          bool taken = false;
          for (const Conn& c : cs)
            if (c.src == s.id && c.dst == d.id) {
              taken = true;
              break;
            }
          if (!taken && !creates_cycle(cs, s.id, d.id)) cands.emplace_back(s.id, d.id);
        }
      }
      if (!cands.empty()) {
        const auto pick = cands[(size_t)rng.integers((int64_t)cands.size())];
        const double w = rng.uniform(-1.0, 1.0);
        cs.push_back({new_innov(), pick.first, pick.second, w, 1});
      }
    }
    if (rng.random() < p_node) {
      std::vector<int> enabled;
      for (int i = 0; i < (int)cs.size(); ++i)
        if (cs[i].en) enabled.push_back(i);
      if (!enabled.empty()) {
        const int pick = enabled[(size_t)rng.integers((int64_t)enabled.size())];
        const Conn old = cs[pick];
        const int64_t nid = deferred ? kDeferredNode : next_node++;
        const int8_t act = (int8_t)rng.integers(6);
        cs[pick].en = 0;
        ns.push_back({nid, 1, act});
        const int64_t i0 = new_innov();
        cs.push_back({i0, old.src, nid, 1.0, 1});
        cs.push_back({new_innov(), nid, old.dst, old.w, 1});
      }
    }
    for (const Node& v : ns) {
      o_node_id[on] = v.id;
      o_node_role[on] = v.role;
      o_node_act[on] = v.act;
      ++on;
    }
    for (const Conn& c : cs) {
      o_innov[oc] = c.innov;
      o_src[oc] = c.src;
      o_dst[oc] = c.dst;
      o_w[oc] = c.w;
      o_en[oc] = c.en;
      ++oc;
    }
    o_node_off[g + 1] = on;
    o_conn_off[g + 1] = oc;
  }
  if (!deferred) {
    counter[0] = next_innov;
    counter[1] = next_node;
  }
  return 0;
}

}  // namespace

extern "C" {

EVO_API int evo_neat_mutate(int n, const uint64_t* keys, const double* rates, int64_t* counter,
                            const int32_t* node_off, const int64_t* node_id, const int8_t* node_role,
                            const int8_t* node_act, const int32_t* conn_off, const int64_t* c_innov,
                            const int64_t* c_src, const int64_t* c_dst, const double* c_w, const uint8_t* c_en,
                            int32_t* o_node_off, int64_t* o_node_id, int8_t* o_node_role, int8_t* o_node_act,
                            int32_t* o_conn_off, int64_t* o_innov, int64_t* o_src, int64_t* o_dst, double* o_w,
                            uint8_t* o_en) {
  return mutate_impl(false, n, keys, rates, counter, node_off, node_id, node_role, node_act, conn_off, c_innov, c_src,
                     c_dst, c_w, c_en, o_node_off, o_node_id, o_node_role, o_node_act, o_conn_off, o_innov, o_src,
                     o_dst, o_w, o_en);
}

EVO_API int evo_neat_mutate_deferred(int n, const uint64_t* keys, const double* rates, const int32_t* node_off,
                                     const int64_t* node_id, const int8_t* node_role, const int8_t* node_act,
                                     const int32_t* conn_off, const int64_t* c_innov, const int64_t* c_src,
                                     const int64_t* c_dst, const double* c_w, const uint8_t* c_en,
                                     int32_t* o_node_off, int64_t* o_node_id, int8_t* o_node_role,
                                     int8_t* o_node_act, int32_t* o_conn_off, int64_t* o_innov, int64_t* o_src,
                                     int64_t* o_dst, double* o_w, uint8_t* o_en) {
  return mutate_impl(true, n, keys, rates, nullptr, node_off, node_id, node_role, node_act, conn_off, c_innov, c_src,
                     c_dst, c_w, c_en, o_node_off, o_node_id, o_node_role, o_node_act, o_conn_off, o_innov, o_src,
                     o_dst, o_w, o_en);
}

// Linearised pattern networks for evo_express_cppn (the layout of
// paper_2406_09654_b200.neat.compile_programs): per genome, nodes in Kahn
// order over the full gene graph with an id-sorted frontier
// (hypernet.py:100-125); node record {act | -1 for inputs, input position |
// -1, edge begin, edge end}; incoming edges = ENABLED connections in
// connection-list order (hypernet.py:140-153), edge source = the source's
// position in the order; outs = positions of the two output nodes in
// ascending id order.  Capacities: nodes_out >= total nodes, edges >= total
// connections.
EVO_API int evo_neat_compile(int n, const int32_t* node_off, const int64_t* node_id, const int8_t* node_role,
                             const int8_t* node_act, const int32_t* conn_off, const int64_t* c_src,
                             const int64_t* c_dst, const double* c_w, const uint8_t* c_en, int32_t* prog_off,
                             int32_t* nodes_out, int32_t* edge_src, double* edge_w, int32_t* outs) {
  int32_t np_ = 0, ne = 0;
  prog_off[0] = 0;
  // scratch reused across genomes (no per-genome allocations once grown);
  // out-edges in CSR form, each node's list in connection order
  std::vector<int> indeg, order, pos_of, frontier, csrc, cdst, adj_off, adj, inputs, outputs;
  std::vector<int64_t> ids;
  for (int g = 0; g < n; ++g) {
    const int n0 = node_off[g], nn = node_off[g + 1] - n0;
    const int c0 = conn_off[g], nc = conn_off[g + 1] - c0;
    ids.assign(node_id + n0, node_id + n0 + nn);
    auto local = [&](int64_t id) -> int {
      for (int i = 0; i < nn; ++i)
        if (ids[i] == id) return i;
      return -1;
    };
    indeg.assign(nn, 0);
    adj_off.assign(nn + 1, 0);
    csrc.resize(nc);
    cdst.resize(nc);
    for (int k = 0; k < nc; ++k) {
      csrc[k] = local(c_src[c0 + k]);
      cdst[k] = local(c_dst[c0 + k]);
      if (csrc[k] < 0 || cdst[k] < 0) {
        g_neat_err = "evo_neat_compile: connection to an unknown node";
        return EVO_EINVAL;
      }
      indeg[cdst[k]]++;
      adj_off[csrc[k] + 1]++;
    }
    for (int i = 0; i < nn; ++i) adj_off[i + 1] += adj_off[i];
    adj.resize(nc);
    for (int k = 0, i; k < nc; ++k) {
      i = csrc[k];
      adj[adj_off[i]++] = cdst[k];
    }
    for (int i = nn; i > 0; --i) adj_off[i] = adj_off[i - 1];
    adj_off[0] = 0;
    frontier.clear();
    for (int i = 0; i < nn; ++i)
      if (indeg[i] == 0) frontier.push_back(i);
    auto by_id = [&](int a, int b) { return ids[a] > ids[b]; };  // min-heap on id
    std::make_heap(frontier.begin(), frontier.end(), by_id);
    order.clear();
    while (!frontier.empty()) {
      std::pop_heap(frontier.begin(), frontier.end(), by_id);
      const int v = frontier.back();
      frontier.pop_back();
      order.push_back(v);
      for (int e = adj_off[v]; e < adj_off[v + 1]; ++e)
        if (const int m = adj[e]; --indeg[m] == 0) {
          frontier.push_back(m);
          std::push_heap(frontier.begin(), frontier.end(), by_id);
        }
    }
    if ((int)order.size() != nn) {
      g_neat_err = "evo_neat_compile: gene graph contains a cycle";
      return EVO_EINVAL;
    }
    pos_of.assign(nn, 0);
    for (int p = 0; p < nn; ++p) pos_of[order[p]] = p;
    // input positions: inputs ranked by id
    inputs.clear();
    for (int i = 0; i < nn; ++i)
      if (node_role[n0 + i] == 0) inputs.push_back(i);
    std::sort(inputs.begin(), inputs.end(), [&](int a, int b) { return ids[a] < ids[b]; });
    outputs.clear();
    for (int i = 0; i < nn; ++i)
      if (node_role[n0 + i] == 2) outputs.push_back(i);
    std::sort(outputs.begin(), outputs.end(), [&](int a, int b) { return ids[a] < ids[b]; });
    if (inputs.size() != 5 || outputs.size() != 2) {
      g_neat_err = "evo_neat_compile: a pattern network needs five inputs and two outputs";
      return EVO_EINVAL;
    }
    for (int p = 0; p < nn; ++p) {
      const int v = order[p];
      int32_t* rec = nodes_out + 4 * (size_t)(np_ + p);
      if (node_role[n0 + v] == 0) {
        const int ip = (int)(std::find(inputs.begin(), inputs.end(), v) - inputs.begin());
        rec[0] = -1, rec[1] = ip, rec[2] = ne, rec[3] = ne;
        continue;
      }
      const int b = ne;
      for (int k = 0; k < nc; ++k)
        if (c_en[c0 + k] && cdst[k] == v) {
          edge_src[ne] = pos_of[csrc[k]];
          edge_w[ne] = c_w[c0 + k];
          ++ne;
        }
      rec[0] = node_act[n0 + v], rec[1] = -1, rec[2] = b, rec[3] = ne;
    }
    outs[2 * g] = pos_of[outputs[0]];
    outs[2 * g + 1] = pos_of[outputs[1]];
    np_ += nn;
    prog_off[g + 1] = np_;
  }
  return 0;
}

}  // extern "C"
