// C ABI of the B200 substrate step (include/evoca_b200.h).
//
// Owns every device allocation of one strip: double-buffered SoA planes with
// a ghost row above and below, the pass-1 intermediate planes, the per-slot
// controller tables in the kernel layout, the device census and the optional
// parity buffers (injected / exported ActionField, adoption events).

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "evoca_b200.h"
#include "evoca_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                                     \
  do {                                                                                               \
    cudaError_t _e = (expr);                                                                         \
    if (_e != cudaSuccess) return fail((int)_e, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

}  // namespace

struct evo_ctx {
  int device = 0;
  int W = 0, H = 0, Hg = 0;
  long long row0 = 0;
  int cap = 0, hidden = 0, hpad = 0;
  bool strip = false;
  long long stride = 0;  // (H + 2) * W
  evo::Planes buf[2] = {};
  int front = 0;
  evo::Mid mid = {};
  float *wA = nullptr, *bA = nullptr, *wB = nullptr, *bB = nullptr;
  // direct nets of pools <= kMmaSlots: fragment-order copy for the mma.sync
  // tile kernel (EVO_F_MMA_NET), rebuilt on the stream before the next such
  // pass 1 after any weight write
  float* wF = nullptr;
  bool frag_stale = true;
  // hidden nets, gather form: per-slot pre-split tables (k_hid_tables),
  // rebuilt on the stream before the next such pass 1 after any weight write
  unsigned char* htab = nullptr;
  bool htab_stale = true;
  // cluster-sharded pass 1 (evoca_shard.cu): slot -> (shard, local) map and
  // per-shard weight tables, rebuilt on the stream when the pool changed
  int* shard_map = nullptr;
  int* shard_res = nullptr;
  float* shard_tables = nullptr;
  bool shard_stale = true;
  int shard_q = 0;
  int live = 0;  // live slots at the last evo_set_slots
  evo::Census census = {};
  float* act_in = nullptr;
  uint8_t* act_in_flag = nullptr;
  float* act_out = nullptr;
  uint8_t* act_out_flag = nullptr;
  int64_t* ev_src = nullptr;
  float* ev_q = nullptr;
  int32_t* ev_def = nullptr;
  float* src_map = nullptr;
  // field-radiation selection (allocated on first use)
  int32_t* sel_list = nullptr;
  int32_t* sel_chunk_cnt = nullptr;
  long long* sel_chunk_off = nullptr;
  unsigned long long* sel_n = nullptr;
  int32_t* sel_parent = nullptr;
  int32_t* sel_map = nullptr;
  bool have_select = false;
  // tensor-core hidden-layer controller buffers (allocated on first use)
  evo::HidBuffers hid = {};
  evo::GatherBuffers gat = {};  // large-pool direct nets by gather (allocated on first use)
  // TMA maps of the texture build for each plane buffer (whole-strip steps;
  // built with the gather buffers, 0 = not available -> the LSU kernel)
  evo::GatherMaps* gmaps = nullptr;  // [2], 64-byte aligned host memory
  bool have_gmaps = false;
  const float* mid_rec = nullptr;  // pass-1 records of a fused evo_step (consumed by its pass 2), else null
  // Lazy fused steps (evo_step / evo_run on the gather path): pass 2 writes
  // E', C' and the final I into the sense texture instead of the planes, and
  // the next such step builds no texture.  tex_state: the texture holds the
  // FRONT buffer's E, I, C and that buffer's planes are stale (materialize()
  // unpacks them before anything else touches them); tex_pending: pass 2 of
  // the running evo_step wrote the texture for the buffer the swap makes front.
  bool tex_state = false, tex_pending = false, lazy_step = false;
  // evo_profile: per-step events (start, between the passes, end) of evo_step
  // evo_run's instantiated step graphs, destroyed once their stream has drained
  std::vector<cudaGraphExec_t> run_execs;
  cudaStream_t run_stream = nullptr;
  bool profile = false;
  std::vector<cudaEvent_t> prof_ev;
  size_t prof_used = 0;
  int num_sms = 0;
  // rows / flags evo_get_actions reads (act_out, or hid.act after a tensor-core step)
  const float* exp_rows = nullptr;
  const uint8_t* exp_flag = nullptr;
  const int32_t* exp_rank = nullptr;  // rank-indexed rows (genome-sorted paths)
  bool have_export = false, have_events = false, have_src_map = false;
  cudaStream_t stream = nullptr;
  // host-pipelined step (evo_step_host; created on first use)
  static constexpr int kMaxBands = 64;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_out = nullptr, ev_in[kMaxBands] = {}, ev_p2[kMaxBands + 2] = {};
  static constexpr size_t kTraceEvents = 512;
  cudaEvent_t tev[kTraceEvents] = {};
  uint32_t* rgba = nullptr;  // render target (evo_render_rgb; allocated on first use)
  double* msc_work = nullptr;  // block-mean pyramid + results (evo_msc / evo_plane_sums)
  long long* msc_acc = nullptr;
  int* bad = nullptr;
  unsigned char* h_stage = nullptr;  // pinned: bad flag, stats, census counts
  std::vector<void*> allocs;

  long long ncell() const { return (long long)W * H; }
  evo::Params params() const {
    evo::Params p;
    p.hidden = hidden;
    p.hpad = hpad;
    p.wA = wA;
    p.bA = bA;
    p.wB = wB;
    p.bB = bB;
    p.wF = nullptr;
    return p;
  }
  evo::StepGeom geom() const {
    evo::StepGeom g;
    g.W = W;
    g.H = H;
    g.row0 = row0;
    g.Hg = Hg;
    g.stride = stride;
    g.own_ghosts = strip ? 0 : 1;
    return g;
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, count * sizeof(T) > 0 ? count * sizeof(T) : 16);
    if (e != cudaSuccess) return e;
    allocs.push_back(v);
    *p = static_cast<T*>(v);
    // the legacy default stream does not order against the context's
    // non-blocking streams: zero synchronously before anything can use it
    e = cudaMemset(v, 0, count * sizeof(T) > 0 ? count * sizeof(T) : 16);
    return e == cudaSuccess ? cudaDeviceSynchronize() : e;
  }
};

namespace {

cudaStream_t pick(evo_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->stream; }

// Host <-> device copies of the ABI's small tables, ordered on the context's
// stream and complete on return.  (The legacy default stream does not order
// against the context's non-blocking streams, and a pageable host->device
// cudaMemcpy may return before its DMA has landed: a copy into the census
// table raced the next step's kernels.)
cudaError_t copy_sync(evo_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c->stream);
  return e == cudaSuccess ? cudaStreamSynchronize(c->stream) : e;
}
cudaError_t zero_sync(evo_ctx* c, void* dst, int value, size_t bytes) {
  cudaError_t e = cudaMemsetAsync(dst, value, bytes, c->stream);
  return e == cudaSuccess ? cudaStreamSynchronize(c->stream) : e;
}

int check_ctx(evo_ctx* c) {
  if (!c) return fail(EVO_EINVAL, "null context");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail((int)e, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return 0;
}

evo::Scalars to_scalars(const evo_scalars& s) {
  evo::Scalars o;
  o.mode = s.rho_mode;
  o.rho = s.rho_f32;
  o.drain = s.drain_f32;
  o.kinv = s.invest_rate;
  o.kliq = s.liquidate_rate;
  o.einv = s.invest_efficiency;
  o.eliq = s.liquidate_efficiency;
  o.alpha = s.explore_fraction;
  o.upkeep = s.upkeep;
  o.dstarve = s.decay_on_starvation;
  o.imin = s.death_threshold;
  return o;
}

int create_impl(evo_ctx** out, int width, int height, long long row0, int hg, int capacity, int hidden, int device,
                bool strip) {
  if (!out) return fail(EVO_EINVAL, "out is null");
  *out = nullptr;
  if (width < 1 || height < 1) return fail(EVO_EINVAL, "substrate dimensions must be positive");
  if (capacity < 1 || capacity > evo::kMaxCapacity)
    return fail(EVO_EINVAL, "capacity must be in [1, " + std::to_string(evo::kMaxCapacity) + "]");
  if (hidden < 0 || hidden > 1024) return fail(EVO_EINVAL, "hidden size must be in [0, 1024]");
  if (hg < height || row0 < 0 || row0 + height > hg) return fail(EVO_EINVAL, "strip outside the global torus");
  if ((long long)width * hg >= 0xFFFFFFFFLL) return fail(EVO_EINVAL, "grid exceeds 2^32-1 cells");
  if ((long long)(height + 2) * width >= 0x7F800000LL)
    return fail(EVO_EINVAL, "strip exceeds 2^31 - 2^23 cells per plane: split it over more strips");
  if (strip && height < 1) return fail(EVO_EINVAL, "strip needs at least one row");
  evo_ctx* c = new evo_ctx();
  c->device = device;
  c->W = width;
  c->H = height;
  c->row0 = row0;
  c->Hg = hg;
  c->cap = capacity;
  c->hidden = hidden;
  c->hpad = hidden > 0 ? ((hidden + 7) / 8) * 8 : 0;
  c->strip = strip;
  c->stride = (long long)(height + 2) * width;
  auto bail = [&](cudaError_t e, const char* what) {
    for (void* p : c->allocs) cudaFree(p);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return fail((int)e, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(e, "cudaSetDevice");
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(e, "cudaStreamCreate");
  const size_t n = (size_t)c->stride;
  // E, I, C0..C2 and the genome plane of a buffer are one block of six
  // equally spaced 4-byte planes, so a row band of all six moves between host
  // and device in one 2-D copy when the host planes are laid out alike
  for (int b = 0; b < 2; ++b) {
    float* blk = nullptr;
    if ((e = c->alloc(&blk, 6 * n)) != cudaSuccess) return bail(e, "alloc planes");
    c->buf[b].E = blk;
    c->buf[b].I = blk + n;
    c->buf[b].C = blk + 2 * n;
    c->buf[b].gi = reinterpret_cast<int32_t*>(blk + 5 * n);
    if ((e = c->alloc(&c->buf[b].rot, n)) != cudaSuccess) return bail(e, "alloc rot");
  }
  if ((e = cudaMemset(c->buf[0].gi, 0xFF, n * sizeof(int32_t))) != cudaSuccess) return bail(e, "memset gi");
  if ((e = cudaMemset(c->buf[1].gi, 0xFF, n * sizeof(int32_t))) != cudaSuccess) return bail(e, "memset gi");
  if ((e = c->alloc(&c->mid.I, n)) != cudaSuccess) return bail(e, "alloc mid");
  if ((e = c->alloc(&c->mid.gi, n)) != cudaSuccess) return bail(e, "alloc mid");
  if ((e = c->alloc(&c->mid.rp, n)) != cudaSuccess) return bail(e, "alloc mid");
  if ((e = c->alloc(&c->mid.q, n)) != cudaSuccess) return bail(e, "alloc mid");
  const size_t cap = (size_t)capacity;
  if (hidden == 0) {
    // compact direct layout: W12 [cap][45][12] (actuators 0..11), W1 [cap][45] (actuator 12)
    if ((e = c->alloc(&c->wA, cap * evo::kSensors * 12)) != cudaSuccess) return bail(e, "alloc w");
    if ((e = c->alloc(&c->wB, (cap * evo::kSensors + 3) / 4 * 4)) != cudaSuccess) return bail(e, "alloc w");
    if ((e = c->alloc(&c->bA, cap * evo::kOutPad)) != cudaSuccess) return bail(e, "alloc b");
    if (capacity <= evo::kMmaSlots && (e = c->alloc(&c->wF, cap * evo::kFragGenome)) != cudaSuccess)
      return bail(e, "alloc wF");
  } else {
    if ((e = c->alloc(&c->wA, cap * evo::kSensors * c->hpad)) != cudaSuccess) return bail(e, "alloc w1");
    if ((e = c->alloc(&c->bA, cap * c->hpad)) != cudaSuccess) return bail(e, "alloc b1");
    if ((e = c->alloc(&c->wB, cap * c->hpad * evo::kOutPad)) != cudaSuccess) return bail(e, "alloc w2");
    if ((e = c->alloc(&c->bB, cap * evo::kOutPad)) != cudaSuccess) return bail(e, "alloc b2");
  }
  if ((e = c->alloc(&c->census.counts, cap)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.counts_last, cap)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.state, cap)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.death_step, cap)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.peak, cap)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.done, 1)) != cudaSuccess) return bail(e, "alloc census");
  if ((e = c->alloc(&c->census.stats, 2)) != cudaSuccess) return bail(e, "alloc stats");
  if ((e = cudaMemset(c->census.death_step, 0xFF, cap * sizeof(int64_t))) != cudaSuccess) return bail(e, "memset");
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "sync");
  *out = c;
  return 0;
}

int ensure_actions_in(evo_ctx* c) {
  if (c->act_in) return 0;
  CK(c->alloc(&c->act_in, (size_t)c->ncell() * evo::kActuators));
  CK(c->alloc(&c->act_in_flag, (size_t)c->ncell()));
  return 0;
}

int ensure_actions_out(evo_ctx* c) {
  if (c->act_out) return 0;
  CK(c->alloc(&c->act_out, (size_t)c->ncell() * evo::kActuators));
  CK(c->alloc(&c->act_out_flag, (size_t)c->ncell()));
  return 0;
}

// actuator rows / decided records and the cell -> row map shared by every
// genome-sorted path
int ensure_sorted_out(evo_ctx* c) {
  if (c->hid.act) return 0;
  const size_t n = (size_t)c->ncell();
  CK(c->alloc(&c->hid.act, n * 16 + (size_t)c->W * 16));  // + two ghost rows of 8-float pass-1 records (strips)
  CK(c->alloc(&c->hid.rank, n));
  if (!c->num_sms) CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  return 0;
}

int ensure_gather(evo_ctx* c) {
  if (int r = ensure_sorted_out(c)) return r;
  if (c->gat.tex) return 0;
  CK(c->alloc(&c->gat.tex, ((size_t)c->H + 2) * c->W * 8));
  if (!c->gmaps) {
    void* m = nullptr;
    if (posix_memalign(&m, 128, 2 * sizeof(evo::GatherMaps)) != 0) return fail(EVO_EINVAL, "out of host memory");
    c->gmaps = static_cast<evo::GatherMaps*>(m);
  }
  c->have_gmaps = !std::getenv("EVO_NO_TMA") && evo::make_gather_maps(c->buf[0], c->geom(), c->gat.tex, &c->gmaps[0]) &&
                  evo::make_gather_maps(c->buf[1], c->geom(), c->gat.tex, &c->gmaps[1]);
  const evo::GatherSizes z = evo::gather_sizes(c->W, c->H, c->cap, c->num_sms);
  const size_t n = (size_t)c->ncell(), nb = (size_t)z.nbands, bins = (size_t)z.bins;
  CK(c->alloc(&c->gat.cta_hist, (size_t)z.nctas * bins));
  CK(c->alloc(&c->gat.lrank, n));
  CK(c->alloc(&c->gat.band_hist, nb * bins));
  CK(c->alloc(&c->gat.goff, nb * (bins + 1)));
  CK(c->alloc(&c->gat.ght, nb * (bins + 1)));
  CK(c->alloc(&c->gat.band_tot, nb * 2));
  CK(c->alloc(&c->gat.band_base, nb * 2 + 2));
  CK(c->alloc(&c->gat.n_ht, 2));
  CK(c->alloc(&c->gat.sorted, n));
  CK(c->alloc(&c->gat.info, (size_t)z.max_ht));
  return 0;
}

int ensure_hidden_tc(evo_ctx* c) {
  if (int r = ensure_sorted_out(c)) return r;
  if (c->hid.sens) return 0;
  const size_t n = (size_t)c->ncell(), cap = (size_t)c->cap;
  CK(c->alloc(&c->hid.counts, cap));
  CK(c->alloc(&c->hid.offs, cap + 1));
  CK(c->alloc(&c->hid.tiles, cap + 1));
  CK(c->alloc(&c->hid.cursor, cap));
  CK(c->alloc(&c->hid.n_tiles, 1));
  CK(c->alloc(&c->hid.cta_hist, (size_t)evo::hidden_sort_ctas(c->W, c->H) * cap));
  CK(c->alloc(&c->hid.tile_info, n / 128 + cap + 1));
  CK(c->alloc(&c->hid.sens, n * 48));
  return 0;
}

int ensure_events(evo_ctx* c) {
  if (c->ev_src) return 0;
  CK(c->alloc(&c->ev_src, (size_t)c->ncell()));
  CK(c->alloc(&c->ev_q, (size_t)c->ncell()));
  CK(c->alloc(&c->ev_def, (size_t)c->ncell()));
  return 0;
}

int ensure_pipe(evo_ctx* c) {
  if (c->s_in) return 0;
  CK(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  for (cudaEvent_t& e : c->ev_in) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (cudaEvent_t& e : c->ev_p2) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (std::getenv("EVO_PIPE_TRACE"))
    for (size_t i = 0; i < evo_ctx::kTraceEvents; ++i) CK(cudaEventCreate(&c->tev[i]));
  CK(c->alloc(&c->bad, 1));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_stage), 32 + (size_t)c->cap * 4, cudaHostAllocDefault));
  return 0;
}

// A run of rows of the strip viewed as a strip of its own: plane pointers
// shifted by `off` = first row * W so that the view's ghost rows are the
// neighbouring real rows (row-band pipelining of evo_step_host).
struct View {
  evo::StepGeom g;
  evo::Planes front, back;
  evo::Mid mid;
  long long off;
};

evo::Planes shifted(const evo::Planes& p, long long o) {
  evo::Planes q;
  q.E = p.E + o;
  q.I = p.I + o;
  q.C = p.C + o;
  q.gi = p.gi + o;
  q.rot = p.rot + o;
  return q;
}

View full_view(const evo_ctx* c) {
  View v;
  v.g = c->geom();
  v.front = c->buf[c->front];
  v.back = c->buf[c->front ^ 1];
  v.mid = c->mid;
  v.off = 0;
  return v;
}

View band_view(const evo_ctx* c, int r0, int rows) {
  View v = full_view(c);
  const long long o = (long long)r0 * c->W;
  v.g.H = rows;
  v.g.row0 = c->row0 + r0;
  v.g.own_ghosts = 0;
  v.front = shifted(v.front, o);
  v.back = shifted(v.back, o);
  v.mid.I += o;
  v.mid.gi += o;
  v.mid.rp += o;
  v.mid.q += o;
  v.off = o;
  return v;
}

// The front E, I, C planes from the texture after lazy fused steps: called by
// every entry point that reads or writes those planes (not by evo_step itself).
int materialize(evo_ctx* c, cudaStream_t st) {
  if (!c->tex_state) return 0;
  c->tex_state = false;
  if (!c->num_sms) CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  CK(evo::launch_tex_to_planes(c->gat.tex, c->geom(), c->buf[c->front], c->num_sms, st));
  return 0;
}

int pass1_view(evo_ctx* c, const View& v, const evo_scalars* s, int phases, int flags, long long* stats,
               cudaStream_t st) {
  if (!s) return fail(EVO_EINVAL, "null scalars");
  const bool inject = flags & EVO_F_INJECT_ACTIONS;
  bool exp = (flags & EVO_F_EXPORT_ACTIONS) && !inject;
  c->mid_rec = nullptr;
  if (inject && !c->act_in) return fail(EVO_EINVAL, "EVO_F_INJECT_ACTIONS without evo_set_actions");
  if ((inject || exp) && v.off != 0) return fail(EVO_EINVAL, "action injection/export needs a whole-strip pass");
  // wide hidden layers run on the tensor cores (sense -> genome buckets ->
  // tcgen05 3xTF32 MLP -> actuator rows), the physics as pass 1 with those
  // rows; narrow ones (the reference's default 16) stay on the CUDA cores in
  // fixed-order FP32 - 3xTF32 is ~2^-21 relative per product, which exceeds
  // the 1e-5 action tolerance when CPPN weights reach w_max = 3
  // (tests/test_radiation.py), and a 45x16 layer is not dense enough to pay
  const bool tc_net = !inject && c->hidden > 0 && evo::hidden_tc_supported(c->hidden) &&
                      !(flags & EVO_F_CUDA_CORE_NET) &&
                      (c->hidden >= evo::kTcMinHidden || (flags & EVO_F_TC_NET));
  // direct nets of large pools (weights do not fit next to the tile in shared
  // memory): cells sorted by (row band, slot, rotation), each warp gathering
  // its cells' Moore neighbourhoods from an L2-resident sense texture
  // (evoca_gather.cu); EVO_F_ROWS_NET selects the earlier genome-sorted
  // sensor rows written to HBM (evoca_hidden_tc.cu); EVO_F_SHARD_NET the measured
  // alternative that shards the weight table over a thread-block cluster
  // working on one tile (evoca_shard.cu: 4.7 ms against 2.4 ms per config-3
  // step - each CTA sees ~256 cells of a tile, too few to hide its latency)
  const bool big_pool = !inject && c->hidden == 0 &&
                        (c->cap > evo::kSmemWeightSlotsAbi || (flags & EVO_F_GATHER_NET)) &&
                        !(flags & EVO_F_TILE_NET);
  const bool shard_net = big_pool && !exp && (flags & EVO_F_SHARD_NET) && c->live <= evo::kShardMaxLive;
  const bool gather_net = big_pool && !shard_net && !(flags & EVO_F_ROWS_NET) &&
                          evo::gather_supported(c->W, c->H, c->cap);
  const bool rows_net = big_pool && !shard_net && !gather_net;
  if (exp && !tc_net && !rows_net && !gather_net) {
    if (int r = ensure_actions_out(c)) return r;
  }
  // hidden-layer nets on the tensor cores: genome-sorted sensor rows; with
  // EVO_F_GATHER_NET over the gather sort instead (cells by (band, slot),
  // Moore records from the sense texture, actuator rows at the cell index) -
  // measured slower on config 5 (9.8 ms against 3.7 ms per net): with 4096
  // genomes a (band, slot) group is two tiles, so the 64 KB of split
  // weights are restaged every other tile
  const bool hid_gather = tc_net && (flags & EVO_F_GATHER_NET) && !(flags & (EVO_F_ROWS_NET | EVO_F_L2_CUDA_CORE)) &&
                          evo::hidden_gather_supported(c->hidden) && evo::gather_supported(c->W, c->H, c->cap);
  if ((tc_net && !hid_gather) || rows_net) {
    if (int r = ensure_hidden_tc(c)) return r;
    CK(evo::launch_hidden_tc(c->hid, v.g, v.front, c->params(), c->cap, c->num_sms, /*decided=*/!exp,
                             (flags & EVO_F_L2_CUDA_CORE) != 0, st));
  }
  if (hid_gather) {
    if (int r = ensure_gather(c)) return r;
    CK(evo::launch_gather_sort(c->gat, v.g, v.front, c->cap, c->num_sms, 128, /*one_band=*/false, c->hid.rank, st));
    if (!c->htab) CK(c->alloc(&c->htab, (size_t)c->cap * evo::hidden_table_bytes(c->hidden)));
    if (c->htab_stale) {
      CK(evo::launch_hidden_tables(c->params(), c->cap, c->htab, st));
      c->htab_stale = false;
    }
    CK(evo::launch_hidden_gather(c->gat, v.g, c->params(), c->cap, c->num_sms, c->htab, c->hid.act, st));
  }
  if (!gather_net || !(flags & EVO_F_LAZY)) {
    if (int r = materialize(c, st)) return r;
  }
  c->lazy_step = false;
  if (gather_net) {  // rows (export) or decided records at the cell index; rank = identity for occupied cells
    const int variant = (flags & EVO_F_TC_DIRECT) ? evo::kGatherTc : evo::kGatherFfma2;
    if (int r = ensure_gather(c)) return r;
    // TMA texture build for whole-strip steps (band views of evo_step_host
    // shift the planes: the LSU kernel)
    const evo::GatherMaps* maps = (c->have_gmaps && v.off == 0) ? &c->gmaps[c->front] : nullptr;
    // evo_step / evo_run on a whole torus (or evo_pass1 with
    // EVO_F_FUSE_MID): the physics runs in the net's epilogue and pass 2
    // reads 32-byte pass-1 records (no k_physics_rows, no mid planes); a bare
    // evo_pass1 keeps the mid planes it documents
    if ((flags & EVO_F_FUSE_MID) && !(flags & EVO_F_UNFUSED) && maps && !exp &&
        variant == evo::kGatherFfma2) {
      evo::FusedPhysics fp;
      fp.s = to_scalars(*s);
      fp.phases = phases;
      fp.src_map = c->have_src_map ? c->src_map : nullptr;
      fp.stats = stats;
      CK(evo::launch_direct_gather(c->gat, v.g, v.front, c->params(), c->cap, c->num_sms, variant, false, c->hid.act,
                                   c->hid.rank, st, maps, &fp, c->tex_state));
      c->mid_rec = c->hid.act;
      c->lazy_step = (flags & EVO_F_LAZY) && !std::getenv("EVO_NO_LAZY");
      c->have_export = false;
      return 0;
    }
    if (int r = materialize(c, st)) return r;  // a lazy evo_step that cannot fuse (export, tcgen05 variant, no TMA maps)
    CK(evo::launch_direct_gather(c->gat, v.g, v.front, c->params(), c->cap, c->num_sms, variant, exp, c->hid.act,
                                 c->hid.rank, st, maps));
  }
  const bool via_rows = tc_net || rows_net || gather_net;
  // 8-float decided records at the cell index: direct nets, and hidden nets through k_hid_net2
  const bool decided = via_rows && !exp &&
                       (c->hidden == 0 || (tc_net && !hid_gather &&
                                           evo::hidden_net2_used(c->hidden, (flags & EVO_F_L2_CUDA_CORE) != 0)));
  c->have_export = exp || (via_rows && !decided);
  c->exp_rows = via_rows ? c->hid.act : c->act_out;
  c->exp_flag = via_rows ? nullptr : c->act_out_flag;
  c->exp_rank = via_rows ? c->hid.rank : nullptr;
  evo::Pass1Args a;
  a.g = v.g;
  a.front = v.front;
  a.back = v.back;
  a.mid = v.mid;
  a.net.hidden = c->hidden;
  a.net.hpad = c->hpad;
  a.net.wA = c->wA;
  a.net.bA = c->bA;
  a.net.wB = c->wB;
  a.net.bB = c->bB;
  a.net.wF = nullptr;
  if (c->wF && !inject && !via_rows && (flags & EVO_F_MMA_NET)) {
    if (c->frag_stale) {
      CK(evo::launch_frag_relayout(c->params(), c->cap, c->wF, st));
      c->frag_stale = false;
    }
    a.net.wF = c->wF;
  }
  a.s = to_scalars(*s);
  a.phases = phases;
  a.src_map = c->have_src_map ? c->src_map + v.off : nullptr;
  a.act_in = via_rows ? c->hid.act : c->act_in;
  a.act_flag = via_rows ? nullptr : c->act_in_flag;
  a.act_rank = via_rows ? c->hid.rank : nullptr;
  a.act_decided = decided ? 1 : 0;
  a.act_out = c->act_out;
  a.act_out_flag = c->act_out_flag;
  a.capacity = c->cap;
  a.stats = stats;
  if (shard_net) {
    const int Q = std::min(evo::kShardMaxQ, std::max(2, (std::min(c->live, evo::kShardMaxQ * evo::kShardSlots) +
                                                         evo::kShardSlots - 1) / evo::kShardSlots));
    if (!c->num_sms) CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    if (!c->shard_map) {
      CK(c->alloc(&c->shard_map, (size_t)c->cap));
      CK(c->alloc(&c->shard_res, (size_t)evo::kShardMaxQ * evo::kShardSlots));
      CK(c->alloc(&c->shard_tables, (size_t)evo::kShardMaxQ * evo::kShardFloats));
    }
    if (c->shard_stale || Q != c->shard_q) {
      CK(evo::launch_shard_plan(c->census.state, c->cap, Q, c->shard_map, c->shard_res, c->params(),
                                c->shard_tables, st));
      c->shard_stale = false;
      c->shard_q = Q;
    }
    CK(evo::launch_pass1_shard(a, c->shard_map, c->shard_tables, Q, c->num_sms, st));
    return 0;
  }
  CK(evo::launch_pass1(a, inject || via_rows, exp && !via_rows, st));
  return 0;
}

int pass2_view(evo_ctx* c, const View& v, int64_t t, int flags, int run_census, cudaStream_t st) {
  const bool rec = flags & EVO_F_RECORD_EVENTS;
  if (rec) {
    if (int r = ensure_events(c)) return r;
  }
  c->have_events = rec;
  evo::Pass2Args a;
  a.g = v.g;
  a.back = v.back;
  a.rot_front = v.front.rot;
  a.mid = v.mid;
  a.mid_rec = v.off == 0 ? c->mid_rec : nullptr;
  a.tex_out = (a.mid_rec && c->lazy_step) ? c->gat.tex : nullptr;
  if (a.mid_rec && !a.tex_out && c->tex_state) {
    // the fused pass 1 read the state from the texture, this pass 2 writes
    // whole planes again: the front planes stay stale, the back ones are complete
    c->tex_state = false;
  }
  c->tex_pending = a.tex_out != nullptr;
  if (a.tex_out) c->tex_state = false;  // the texture now belongs to the buffer the swap makes front
  a.census = c->census;
  a.ev.src = rec ? c->ev_src + v.off : nullptr;
  a.ev.q = rec ? c->ev_q + v.off : nullptr;
  a.ev.def = rec ? c->ev_def + v.off : nullptr;
  a.capacity = c->cap;
  a.run_census = run_census;
  a.t = t;
  CK(evo::launch_pass2(a, st));
  return 0;
}

}  // namespace

void drop_run_graphs(evo_ctx* c, bool force) {
  if (c->run_execs.empty()) return;
  if (!force && cudaStreamQuery(c->run_stream) != cudaSuccess) {
    cudaGetLastError();
    return;  // still running: keep them for the next call
  }
  if (force) cudaStreamSynchronize(c->run_stream);
  for (cudaGraphExec_t e : c->run_execs) cudaGraphExecDestroy(e);
  c->run_execs.clear();
}


extern "C" {

EVO_API const char* evo_last_error(void) { return g_err.c_str(); }

EVO_API int evo_version(void) { return 1; }

EVO_API int evo_create(evo_ctx** out, int width, int height, int capacity, int hidden, int device) {
  return create_impl(out, width, height, 0, height, capacity, hidden, device, false);
}

EVO_API int evo_create_strip(evo_ctx** out, int width, int height, int64_t row0, int height_global, int capacity,
                             int hidden, int device) {
  return create_impl(out, width, height, row0, height_global, capacity, hidden, device, true);
}

EVO_API int evo_destroy(evo_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  drop_run_graphs(c, true);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  c->prof_ev.clear();
  if (c->s_in) {
    cudaStreamSynchronize(c->s_in);
    cudaStreamSynchronize(c->s_out);
    cudaStreamDestroy(c->s_in);
    cudaStreamDestroy(c->s_out);
    cudaEventDestroy(c->ev_start);
    cudaEventDestroy(c->ev_out);
    for (cudaEvent_t e : c->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_p2) cudaEventDestroy(e);
    cudaFreeHost(c->h_stage);
    for (size_t i = 0; i < evo_ctx::kTraceEvents; ++i)
      if (c->tev[i]) cudaEventDestroy(c->tev[i]);
  }
  for (void* p : c->allocs) cudaFree(p);
  free(c->gmaps);
  cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

EVO_API int evo_upload_planes(evo_ctx* c, const float* E, const float* I, const float* C, const int32_t* gi,
                              const uint8_t* rot, void* stream) {
  if (int r = check_ctx(c)) return r;
  if (!E || !I || !C || !gi || !rot) return fail(EVO_EINVAL, "null plane pointer");
  c->tex_state = false;  // every plane is overwritten
  cudaStream_t st = pick(c, stream);
  const evo::Planes& p = c->buf[c->front];
  const size_t n = (size_t)c->ncell();
  const size_t W = (size_t)c->W;
  CK(cudaMemcpyAsync(p.E + W, E, n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(p.I + W, I, n * 4, cudaMemcpyHostToDevice, st));
  for (int k = 0; k < 3; ++k)
    CK(cudaMemcpyAsync(p.C + k * c->stride + W, C + k * n, n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(p.gi + W, gi, n * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(p.rot + W, rot, n, cudaMemcpyHostToDevice, st));
  if (!c->strip) CK(evo::launch_refresh_ghosts(p, c->geom(), st));
  if (!stream) CK(cudaStreamSynchronize(st));
  return 0;
}

EVO_API int evo_download_planes(evo_ctx* c, float* E, float* I, float* C, int32_t* gi, uint8_t* rot, void* stream) {
  if (int r = check_ctx(c)) return r;
  cudaStream_t st = pick(c, stream);
  if (int r = materialize(c, st)) return r;
  const evo::Planes& p = c->buf[c->front];
  const size_t n = (size_t)c->ncell();
  const size_t W = (size_t)c->W;
  if (E) CK(cudaMemcpyAsync(E, p.E + W, n * 4, cudaMemcpyDeviceToHost, st));
  if (I) CK(cudaMemcpyAsync(I, p.I + W, n * 4, cudaMemcpyDeviceToHost, st));
  if (C)
    for (int k = 0; k < 3; ++k)
      CK(cudaMemcpyAsync(C + k * n, p.C + k * c->stride + W, n * 4, cudaMemcpyDeviceToHost, st));
  if (gi) CK(cudaMemcpyAsync(gi, p.gi + W, n * 4, cudaMemcpyDeviceToHost, st));
  if (rot) CK(cudaMemcpyAsync(rot, p.rot + W, n, cudaMemcpyDeviceToHost, st));
  if (!stream) CK(cudaStreamSynchronize(st));
  return 0;
}

EVO_API int evo_set_params(evo_ctx* c, int slot0, int n, const float* w1, const float* b1, const float* w2,
                           const float* b2) {
  if (int r = check_ctx(c)) return r;
  if (slot0 < 0 || n < 0 || slot0 + n > c->cap) return fail(EVO_EINVAL, "slot range outside the pool capacity");
  if (n == 0) return 0;
  if (!w2 || !b2) return fail(EVO_EINVAL, "w2/b2 are required");
  const int H = c->hidden;
  if (H > 0 && (!w1 || !b1)) return fail(EVO_EINVAL, "w1/b1 are required for a hidden layer");
  CK(cudaStreamSynchronize(c->stream));
  if (H == 0) {
    std::vector<float> w12((size_t)n * evo::kSensors * 12, 0.0f), w1((size_t)n * evo::kSensors, 0.0f);
    std::vector<float> bt((size_t)n * evo::kOutPad, 0.0f);
    for (int s = 0; s < n; ++s)
      for (int j = 0; j < evo::kActuators; ++j) {
        for (int k = 0; k < evo::kSensors; ++k) {
          const float v = w2[((size_t)s * evo::kActuators + j) * evo::kSensors + k];
          if (j < 12)
            w12[((size_t)s * evo::kSensors + k) * 12 + j] = v;
          else
            w1[(size_t)s * evo::kSensors + k] = v;
        }
        bt[(size_t)s * evo::kOutPad + j] = b2[(size_t)s * evo::kActuators + j];
      }
    CK(copy_sync(c, c->wA + (size_t)slot0 * evo::kSensors * 12, w12.data(), w12.size() * 4, cudaMemcpyHostToDevice));
    CK(copy_sync(c, c->wB + (size_t)slot0 * evo::kSensors, w1.data(), w1.size() * 4, cudaMemcpyHostToDevice));
    CK(copy_sync(c, c->bA + (size_t)slot0 * evo::kOutPad, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice));
    c->frag_stale = true;
    c->shard_stale = true;
    c->htab_stale = true;
    return 0;
  }
  const int hp = c->hpad;
  std::vector<float> W1((size_t)n * evo::kSensors * hp, 0.0f), B1((size_t)n * hp, 0.0f);
  std::vector<float> W2((size_t)n * hp * evo::kOutPad, 0.0f), B2((size_t)n * evo::kOutPad, 0.0f);
  for (int s = 0; s < n; ++s) {
    for (int h = 0; h < H; ++h) {
      for (int k = 0; k < evo::kSensors; ++k)
        W1[((size_t)s * evo::kSensors + k) * hp + h] = w1[((size_t)s * H + h) * evo::kSensors + k];
      B1[(size_t)s * hp + h] = b1[(size_t)s * H + h];
      for (int j = 0; j < evo::kActuators; ++j)
        W2[((size_t)s * hp + h) * evo::kOutPad + j] = w2[((size_t)s * evo::kActuators + j) * H + h];
    }
    for (int j = 0; j < evo::kActuators; ++j) B2[(size_t)s * evo::kOutPad + j] = b2[(size_t)s * evo::kActuators + j];
  }
  CK(copy_sync(c, c->wA + (size_t)slot0 * evo::kSensors * hp, W1.data(), W1.size() * 4, cudaMemcpyHostToDevice));
  CK(copy_sync(c, c->bA + (size_t)slot0 * hp, B1.data(), B1.size() * 4, cudaMemcpyHostToDevice));
  CK(copy_sync(c, c->wB + (size_t)slot0 * hp * evo::kOutPad, W2.data(), W2.size() * 4, cudaMemcpyHostToDevice));
  CK(copy_sync(c, c->bB + (size_t)slot0 * evo::kOutPad, B2.data(), B2.size() * 4, cudaMemcpyHostToDevice));
  c->htab_stale = true;
  return 0;
}

EVO_API int evo_get_params(evo_ctx* c, int slot0, int n, float* w1, float* b1, float* w2, float* b2) {
  if (int r = check_ctx(c)) return r;
  if (slot0 < 0 || n < 0 || slot0 + n > c->cap) return fail(EVO_EINVAL, "slot range outside the pool capacity");
  if (n == 0) return 0;
  if (!w2 || !b2) return fail(EVO_EINVAL, "w2/b2 are required");
  const int H = c->hidden;
  if (H > 0 && (!w1 || !b1)) return fail(EVO_EINVAL, "w1/b1 are required for a hidden layer");
  CK(cudaStreamSynchronize(c->stream));
  if (H == 0) {
    std::vector<float> w12((size_t)n * evo::kSensors * 12), wl((size_t)n * evo::kSensors), bt((size_t)n * evo::kOutPad);
    CK(copy_sync(c, w12.data(), c->wA + (size_t)slot0 * evo::kSensors * 12, w12.size() * 4, cudaMemcpyDeviceToHost));
    CK(copy_sync(c, wl.data(), c->wB + (size_t)slot0 * evo::kSensors, wl.size() * 4, cudaMemcpyDeviceToHost));
    CK(copy_sync(c, bt.data(), c->bA + (size_t)slot0 * evo::kOutPad, bt.size() * 4, cudaMemcpyDeviceToHost));
    for (int s = 0; s < n; ++s)
      for (int j = 0; j < evo::kActuators; ++j) {
        for (int k = 0; k < evo::kSensors; ++k)
          w2[((size_t)s * evo::kActuators + j) * evo::kSensors + k] =
              j < 12 ? w12[((size_t)s * evo::kSensors + k) * 12 + j] : wl[(size_t)s * evo::kSensors + k];
        b2[(size_t)s * evo::kActuators + j] = bt[(size_t)s * evo::kOutPad + j];
      }
    return 0;
  }
  const int hp = c->hpad;
  std::vector<float> W1((size_t)n * evo::kSensors * hp), B1((size_t)n * hp);
  std::vector<float> W2((size_t)n * hp * evo::kOutPad), B2((size_t)n * evo::kOutPad);
  CK(copy_sync(c, W1.data(), c->wA + (size_t)slot0 * evo::kSensors * hp, W1.size() * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, B1.data(), c->bA + (size_t)slot0 * hp, B1.size() * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, W2.data(), c->wB + (size_t)slot0 * hp * evo::kOutPad, W2.size() * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, B2.data(), c->bB + (size_t)slot0 * evo::kOutPad, B2.size() * 4, cudaMemcpyDeviceToHost));
  for (int s = 0; s < n; ++s) {
    for (int h = 0; h < H; ++h) {
      for (int k = 0; k < evo::kSensors; ++k)
        w1[((size_t)s * H + h) * evo::kSensors + k] = W1[((size_t)s * evo::kSensors + k) * hp + h];
      b1[(size_t)s * H + h] = B1[(size_t)s * hp + h];
      for (int j = 0; j < evo::kActuators; ++j)
        w2[((size_t)s * evo::kActuators + j) * H + h] = W2[((size_t)s * hp + h) * evo::kOutPad + j];
    }
    for (int j = 0; j < evo::kActuators; ++j) b2[(size_t)s * evo::kActuators + j] = B2[(size_t)s * evo::kOutPad + j];
  }
  return 0;
}

EVO_API int evo_set_slots(evo_ctx* c, const int8_t* state, const int32_t* peak) {
  if (int r = check_ctx(c)) return r;
  CK(cudaStreamSynchronize(c->stream));
  if (state) {
    CK(copy_sync(c, c->census.state, state, (size_t)c->cap, cudaMemcpyHostToDevice));
    c->live = (int)std::count(state, state + c->cap, (int8_t)1);
    c->shard_stale = true;
    std::vector<int64_t> ds((size_t)c->cap, -1);
    CK(copy_sync(c, c->census.death_step, ds.data(), ds.size() * 8, cudaMemcpyHostToDevice));
  }
  if (peak) CK(copy_sync(c, c->census.peak, peak, (size_t)c->cap * 4, cudaMemcpyHostToDevice));
  return 0;
}

EVO_API int evo_set_source_map(evo_ctx* c, const float* map) {
  if (int r = check_ctx(c)) return r;
  CK(cudaStreamSynchronize(c->stream));
  if (!map) {
    c->have_src_map = false;
    return 0;
  }
  if (!c->src_map) CK(c->alloc(&c->src_map, (size_t)c->ncell()));
  CK(copy_sync(c, c->src_map, map, (size_t)c->ncell() * 4, cudaMemcpyHostToDevice));
  c->have_src_map = true;
  return 0;
}

EVO_API int evo_pass1(evo_ctx* c, const evo_scalars* s, int64_t t, int phases, int flags, void* stream) {
  if (int r = check_ctx(c)) return r;
  (void)t;
  return pass1_view(c, full_view(c), s, phases, flags, c->census.stats, pick(c, stream));
}

EVO_API int evo_pass2(evo_ctx* c, int64_t t, int flags, void* stream) {
  if (int r = check_ctx(c)) return r;
  return pass2_view(c, full_view(c), t, flags, (flags & EVO_F_NO_CENSUS) ? 0 : 1, pick(c, stream));
}

EVO_API int evo_census_finish(evo_ctx* c, int64_t t, void* stream) {
  if (int r = check_ctx(c)) return r;
  CK(evo::launch_census_finish(c->census, c->cap, t, pick(c, stream)));
  return 0;
}

EVO_API int evo_swap(evo_ctx* c) {
  if (!c) return fail(EVO_EINVAL, "null context");
  if (c->tex_pending) {  // evo_step's own swap after a lazy pass 2
    c->tex_pending = false;
    c->front ^= 1;
    c->tex_state = true;
    return 0;
  }
  if (int r = materialize(c, c->stream)) return r;
  c->front ^= 1;
  return 0;
}

EVO_API int evo_step(evo_ctx* c, const evo_scalars* s, int64_t t, int phases, int flags, void* stream) {
  if (c && c->strip) return fail(EVO_EINVAL, "strip contexts step through evo_pass1/evo_pass2 with a halo exchange");
  if (int r = check_ctx(c)) return r;
  cudaStream_t st = pick(c, stream);
  cudaEvent_t* pe = nullptr;
  if (c->profile) {
    if (c->prof_used + 3 > c->prof_ev.size()) {
      const size_t old_n = c->prof_ev.size();
      c->prof_ev.resize(old_n + 192);
      for (size_t i = old_n; i < c->prof_ev.size(); ++i) CK(cudaEventCreate(&c->prof_ev[i]));
    }
    pe = &c->prof_ev[c->prof_used];
    c->prof_used += 3;
    CK(cudaEventRecord(pe[0], st));
  }
  if (int r = pass1_view(c, full_view(c), s, phases, flags | EVO_F_FUSE_MID | EVO_F_LAZY,
                         c->census.stats, st))
    return r;
  if (pe) CK(cudaEventRecord(pe[1], st));
  if (int r = pass2_view(c, full_view(c), t, flags, (flags & EVO_F_NO_CENSUS) ? 0 : 1, st)) return r;
  if (pe) CK(cudaEventRecord(pe[2], st));
  return evo_swap(c);
}

EVO_API int evo_step_host(evo_ctx* c, const evo_scalars* s, int64_t t, int flags, const float* E, const float* I,
                          const float* C, const int32_t* gi, const uint8_t* rot, float* E_out, float* I_out,
                          float* C_out, int32_t* gi_out, uint8_t* rot_out, int32_t* counts, int64_t* stats,
                          int bands, void* stream) {
  if (int r = check_ctx(c)) return r;
  if (c->strip) return fail(EVO_EINVAL, "evo_step_host steps a single-strip context");
  if (!s) return fail(EVO_EINVAL, "null scalars");
  if (!E || !I || !C || !gi || !rot || !E_out || !I_out || !C_out || !gi_out || !rot_out)
    return fail(EVO_EINVAL, "null plane pointer");
  c->tex_state = false;  // the host planes replace the device state
  if (flags & (EVO_F_INJECT_ACTIONS | EVO_F_EXPORT_ACTIONS))
    return fail(EVO_EINVAL, "action injection/export is not available in the host-pipelined step");
  if (int r = ensure_pipe(c)) return r;
  if (c->hidden > 0 || c->cap > evo::kSmemWeightSlotsAbi) {
    const bool gather = !(flags & (EVO_F_ROWS_NET | EVO_F_TILE_NET | EVO_F_SHARD_NET)) &&
                        evo::gather_supported(c->W, c->H, c->cap) &&
                        (c->hidden == 0 || ((flags & EVO_F_GATHER_NET) && evo::hidden_gather_supported(c->hidden)));
    if (int r = gather ? ensure_gather(c) : ensure_hidden_tc(c)) return r;
  }
  if ((flags & EVO_F_RECORD_EVENTS)) {
    if (int r = ensure_events(c)) return r;
  }
  const int W = c->W, H = c->H;
  const long long n = c->ncell();
  // Row bands.  Band nb-1 is the last 32 rows and is uploaded first (it holds
  // the torus row above row 0); bands 0..nb-2 split the rest in whole 32-row
  // tiles.  Pass 1 chunk b = rows [R_b - 32, R_{b+1} - 32) needs only bands
  // <= b; pass 2 chunk b = rows [R_b - 33, R_{b+1} - 33) needs only pass-1
  // chunks <= b; row 0 and the last chunk close the seam at the end.
  // default: ~1.4 M cells per band, 4..12 bands (config 3 measured 12.9 /
  // 11.7 / 11.2 / 11.6 ms per step at 4 / 8 / 12 / 16 bands, tools/e2e_bands.py;
  // config 2 keeps 4)
  int nb = bands > 0 ? bands : (int)std::max(4LL, std::min(12LL, n / 1400000));
  nb = std::min(nb, evo_ctx::kMaxBands);
  if (H - 32 < 64) nb = 1;
  std::vector<int> R;  // band starts, R[nb] = H
  if (nb == 1) {
    R = {0, H};
  } else {
    const int main_rows = H - 32;
    int per = (main_rows + (nb - 1) - 1) / (nb - 1);
    per = std::max(64, (per + 31) / 32 * 32);
    for (int r0 = 0; r0 < main_rows; r0 += per) R.push_back(r0);
    R.push_back(H - 32);
    R.push_back(H);
    nb = (int)R.size() - 1;
  }
  const cudaStream_t st = pick(c, stream);
  // EVO_PIPE_TRACE=1: per-band timeline on stderr (diagnostics)
  static const bool trace = std::getenv("EVO_PIPE_TRACE") != nullptr;
  std::vector<std::string> tname;
  auto markn = [&](cudaStream_t q, const std::string& nm) {
    if (!trace || tname.size() >= evo_ctx::kTraceEvents) return;
    cudaEventRecord(c->tev[tname.size()], q);
    tname.push_back(nm);
  };
  const evo::Planes F = c->buf[c->front], B = c->buf[c->front ^ 1];
  const size_t pitch = (size_t)c->stride * 4, hpitch = (size_t)n * 4;
  // host planes E, I, C0..C2, genome equally spaced (this package's PlaneSet
  // allocates them as one block): one 2-D copy per band instead of five
  auto block6 = [&](const void* e, const void* i, const void* cc, const void* g) {
    const char* b0 = static_cast<const char*>(e);
    return static_cast<const char*>(i) == b0 + hpitch && static_cast<const char*>(cc) == b0 + 2 * hpitch &&
           static_cast<const char*>(g) == b0 + 5 * hpitch;
  };
  const bool in6 = block6(E, I, C, gi), out6 = block6(E_out, I_out, C_out, gi_out);
  auto h2d = [&](int b) -> int {
    const size_t o = (size_t)(R[b] + 1) * W, h = (size_t)R[b] * W, m = (size_t)(R[b + 1] - R[b]) * W;
    if (in6) {
      CK(cudaMemcpy2DAsync(F.E + o, pitch, E + h, hpitch, m * 4, 6, cudaMemcpyHostToDevice, c->s_in));
    } else {
      CK(cudaMemcpyAsync(F.E + o, E + h, m * 4, cudaMemcpyHostToDevice, c->s_in));
      CK(cudaMemcpyAsync(F.I + o, I + h, m * 4, cudaMemcpyHostToDevice, c->s_in));
      CK(cudaMemcpy2DAsync(F.C + o, pitch, C + h, hpitch, m * 4, 3, cudaMemcpyHostToDevice, c->s_in));
      CK(cudaMemcpyAsync(F.gi + o, gi + h, m * 4, cudaMemcpyHostToDevice, c->s_in));
    }
    CK(cudaMemcpyAsync(F.rot + o, rot + h, m, cudaMemcpyHostToDevice, c->s_in));
    CK(cudaEventRecord(c->ev_in[b], c->s_in));
    markn(c->s_in, "h2d " + std::to_string(b));
    return 0;
  };
  auto check = [&](int b) -> int {
    const size_t o = (size_t)(R[b] + 1) * W, m = (size_t)(R[b + 1] - R[b]) * W;
    CK(evo::launch_check_cells(F.gi + o, F.rot + o, (long long)m, c->cap, c->bad, st));
    return 0;
  };
  int n_out = 0;
  auto d2h = [&](int r0, int r1) -> int {
    if (r1 <= r0) return 0;
    const size_t o = (size_t)(r0 + 1) * W, h = (size_t)r0 * W, m = (size_t)(r1 - r0) * W;
    const int k = n_out++;
    CK(cudaEventRecord(c->ev_p2[k], st));
    CK(cudaStreamWaitEvent(c->s_out, c->ev_p2[k], 0));
    if (out6) {
      CK(cudaMemcpy2DAsync(E_out + h, hpitch, B.E + o, pitch, m * 4, 6, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaMemcpyAsync(rot_out + h, B.rot + o, m, cudaMemcpyDeviceToHost, c->s_out));
    } else {
      CK(cudaMemcpyAsync(E_out + h, B.E + o, m * 4, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaMemcpyAsync(I_out + h, B.I + o, m * 4, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaMemcpy2DAsync(C_out + h, hpitch, B.C + o, pitch, m * 4, 3, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaMemcpyAsync(gi_out + h, B.gi + o, m * 4, cudaMemcpyDeviceToHost, c->s_out));
      CK(cudaMemcpyAsync(rot_out + h, B.rot + o, m, cudaMemcpyDeviceToHost, c->s_out));
    }
    markn(c->s_out, "d2h " + std::to_string(r0) + "-" + std::to_string(r1));
    return 0;
  };
  auto p1 = [&](int r0, int r1) -> int {
    if (r1 <= r0) return 0;
    if (int r = pass1_view(c, band_view(c, r0, r1 - r0), s, EVO_PH_ALL, flags, r0 == 0 ? c->census.stats : nullptr,
                           st))
      return r;
    markn(st, "pass1 " + std::to_string(r0) + "-" + std::to_string(r1));
    return 0;
  };
  auto p2 = [&](int r0, int r1) -> int {
    if (r1 <= r0) return 0;
    if (int r = pass2_view(c, band_view(c, r0, r1 - r0), t, flags, 0, st)) return r;
    markn(st, "pass2 " + std::to_string(r0) + "-" + std::to_string(r1));
    return d2h(r0, r1);
  };
  const bool census = !(flags & EVO_F_NO_CENSUS);
  const auto host_t0 = std::chrono::steady_clock::now();
  markn(st, "start");
  CK(cudaEventRecord(c->ev_start, st));
  CK(cudaStreamWaitEvent(c->s_in, c->ev_start, 0));
  CK(cudaStreamWaitEvent(c->s_out, c->ev_start, 0));
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), st));
  // uploads: the seam band first, then bands 0..nb-2
  if (nb > 1) {
    if (int r = h2d(nb - 1)) return r;
  }
  for (int b = 0; b < std::max(1, nb - 1); ++b)
    if (int r = h2d(b)) return r;
  if (nb == 1) {
    CK(cudaStreamWaitEvent(st, c->ev_in[0], 0));
    if (int r = check(0)) return r;
    CK(evo::launch_refresh_ghosts(F, c->geom(), st));
    if (int r = p1(0, H)) return r;
    CK(evo::launch_wrap_mid(c->mid, c->geom(), st));
    if (int r = p2(0, H)) return r;
  } else {
    for (int b = 0; b < nb - 1; ++b) {
      CK(cudaStreamWaitEvent(st, c->ev_in[b], 0));
      if (b == 0) {
        if (int r = check(nb - 1)) return r;
      }
      if (int r = check(b)) return r;
      if (b == 0) CK(evo::launch_refresh_ghosts(F, c->geom(), st));  // rows -1 and H from rows H-1 and 0
      if (int r = p1(b == 0 ? 0 : R[b] - 32, R[b + 1] - 32)) return r;
      if (int r = p2(b == 0 ? 1 : R[b] - 33, R[b + 1] - 33)) return r;
    }
    if (int r = p1(R[nb - 1] - 32, H)) return r;
    CK(evo::launch_wrap_mid(c->mid, c->geom(), st));
    if (int r = p2(R[nb - 1] - 33, H)) return r;
    if (int r = p2(0, 1)) return r;
  }
  // the census epilogue (slot deaths) only runs on accepted planes: with
  // *bad set it just clears the counts, so a rejected step leaves the
  // slot table as it was
  if (census) CK(evo::launch_census_finish(c->census, c->cap, t, st, c->bad));
  CK(evo::launch_refresh_ghosts(B, c->geom(), st));  // device-resident steps may follow
  CK(cudaMemcpyAsync(c->h_stage, c->bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (stats) CK(cudaMemcpyAsync(c->h_stage + 8, c->census.stats, 16, cudaMemcpyDeviceToHost, st));
  if (counts && census)
    CK(cudaMemcpyAsync(c->h_stage + 32, c->census.counts_last, (size_t)c->cap * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(c->ev_out, c->s_out));
  CK(cudaStreamWaitEvent(st, c->ev_out, 0));
  const auto host_t1 = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(st));
  if (trace) {
    std::fprintf(stderr, "[pipe] host enqueue %.3f ms\n",
                 std::chrono::duration<double, std::milli>(host_t1 - host_t0).count());
    for (size_t i = 0; i < tname.size(); ++i) {
      float ms = 0;
      const cudaError_t e = cudaEventElapsedTime(&ms, c->tev[0], c->tev[i]);
      std::fprintf(stderr, "%s%s %.3f%s", i ? ", " : "[pipe] ", tname[i].c_str(), ms, e ? "(err)" : "");
    }
    std::fprintf(stderr, " in6=%d out6=%d\n", (int)in6, (int)out6);
  }
  c->have_export = false;
  int bad_flag;
  std::memcpy(&bad_flag, c->h_stage, sizeof(int));
  if (bad_flag)
    return fail(EVO_EINVAL, "genome_index outside [-1, capacity) or rotation > 7 in the uploaded planes");
  if (stats) std::memcpy(stats, c->h_stage + 8, 16);
  if (counts && census) std::memcpy(counts, c->h_stage + 32, (size_t)c->cap * 4);
  c->front ^= 1;
  return 0;
}

EVO_API int evo_render_rgb(evo_ctx* c, double norm_energy, double norm_infrastructure, uint8_t* rgba, void* stream) {
  if (int r = check_ctx(c)) return r;
  if (!rgba) return fail(EVO_EINVAL, "null frame pointer");
  if (!(norm_energy != 0.0) || !(norm_infrastructure != 0.0)) return fail(EVO_EINVAL, "display norms must be non-zero");
  if (!c->rgba) CK(c->alloc(&c->rgba, (size_t)c->ncell()));
  cudaStream_t st = pick(c, stream);
  if (int r = materialize(c, st)) return r;
  CK(evo::launch_render_rgb(c->buf[c->front], c->geom(), norm_energy, norm_infrastructure, c->rgba, st));
  CK(cudaMemcpyAsync(rgba, c->rgba, (size_t)c->ncell() * 4, cudaMemcpyDeviceToHost, st));
  if (!stream) CK(cudaStreamSynchronize(st));
  return 0;
}

int ensure_metrics(evo_ctx* c) {
  if (c->msc_work) return 0;
  const int side = evo::msc_side(c->W, c->H);
  const long long chunks = evo::plane_sum_chunks(c->ncell());
  CK(c->alloc(&c->msc_work, (size_t)(evo::msc_workspace_doubles(side) + 64 + chunks + 2)));
  CK(c->alloc(&c->msc_acc, (size_t)evo::msc_digits() * 64));
  return 0;
}

EVO_API int evo_msc(evo_ctx* c, int plane, int n_scales, double* squares, double* cross, int* side, int* k_max) {
  if (int r = check_ctx(c)) return r;
  if (c->strip) return fail(EVO_EINVAL, "evo_msc needs a single-strip context");
  if (plane < 0 || plane > 4) return fail(EVO_EINVAL, "plane must be 0 (energy), 1 (infrastructure) or 2..4 (communication)");
  if (!squares || !cross || !side || !k_max) return fail(EVO_EINVAL, "null output pointer");
  const int sd = evo::msc_side(c->W, c->H);
  if (sd < 2) return fail(EVO_EINVAL, "field side must be a power of two >= 2");
  if (int r = ensure_metrics(c)) return r;
  if (int r = materialize(c, c->stream)) return r;
  const evo::Planes& f = c->buf[c->front];
  const float* p = plane == 0 ? f.E : (plane == 1 ? f.I : f.C + (plane - 2) * c->stride);
  double* out = c->msc_work + evo::msc_workspace_doubles(sd);
  int km = 0;
  CK(evo::launch_msc(p, c->W, c->H, n_scales, c->msc_work, c->msc_acc, out, &km, c->stream));
  double host[64];
  CK(cudaMemcpyAsync(host, out, sizeof(double) * (2 * km + 1), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k <= km; ++k) squares[k] = host[k];
  for (int k = 0; k < km; ++k) cross[k] = host[km + 1 + k];
  *side = sd;
  *k_max = km;
  return 0;
}

EVO_API int evo_plane_sums(evo_ctx* c, double* energy, double* infrastructure) {
  if (int r = check_ctx(c)) return r;
  if (c->strip) return fail(EVO_EINVAL, "evo_plane_sums needs a single-strip context");
  if (int r = ensure_metrics(c)) return r;
  if (int r = materialize(c, c->stream)) return r;
  const int sd = evo::msc_side(c->W, c->H);
  double* res = c->msc_work + evo::msc_workspace_doubles(sd) + 64;
  double* chunks = res + 2;
  const evo::Planes& f = c->buf[c->front];
  CK(evo::launch_plane_sum(f.E + c->W, c->ncell(), chunks, res, c->stream));
  CK(evo::launch_plane_sum(f.I + c->W, c->ncell(), chunks, res + 1, c->stream));
  double host[2];
  CK(cudaMemcpyAsync(host, res, sizeof(host), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (energy) *energy = host[0];
  if (infrastructure) *infrastructure = host[1];
  return 0;
}

EVO_API int evo_profile(evo_ctx* c, int enable) {
  if (int r = check_ctx(c)) return r;
  c->profile = enable != 0;
  c->prof_used = 0;
  return 0;
}

EVO_API int evo_profile_read(evo_ctx* c, double* pass1_ms, double* pass2_ms, int* steps) {
  if (int r = check_ctx(c)) return r;
  if (!pass1_ms || !pass2_ms || !steps) return fail(EVO_EINVAL, "null argument");
  *pass1_ms = *pass2_ms = 0.0;
  *steps = (int)(c->prof_used / 3);
  for (size_t i = 0; i + 2 < c->prof_used; i += 3) {
    CK(cudaEventSynchronize(c->prof_ev[i + 2]));
    float a = 0.0f, b = 0.0f;
    CK(cudaEventElapsedTime(&a, c->prof_ev[i], c->prof_ev[i + 1]));
    CK(cudaEventElapsedTime(&b, c->prof_ev[i + 1], c->prof_ev[i + 2]));
    *pass1_ms += a;
    *pass2_ms += b;
  }
  c->prof_used = 0;
  return 0;
}

// evo_run (engine.py:251-271's loop): the first step runs eagerly (it makes
// the lazy allocations and shared-memory opt-ins), the others are captured
// into CUDA graphs of up to kRunGraphSteps steps and launched as one unit -
// small worlds are launch-bound (config 1: two ~5 us kernels per step).  The
// host-side step state (front buffer, lazy-texture flags) advances while
// capturing exactly as it does eagerly.  EVO_NO_GRAPH=1 keeps the eager loop.
constexpr int kRunGraphSteps = 128;

EVO_API int evo_run(evo_ctx* c, const evo_scalars* s, int64_t t0, int k, void* stream) {
  if (!s && k > 0) return fail(EVO_EINVAL, "null scalars");
  if (k <= 0) return 0;
  if (int r = check_ctx(c)) return r;
  static const bool no_graph = std::getenv("EVO_NO_GRAPH") != nullptr;
  const bool graphs = k >= 4 && !c->strip && !c->profile && !no_graph;
  if (!graphs) {
    for (int i = 0; i < k; ++i)
      if (int r = evo_step(c, s + i, t0 + i, EVO_PH_ALL, 0, stream)) return r;
    return 0;
  }
  cudaStream_t st = pick(c, stream);
  if (st != c->run_stream) drop_run_graphs(c, true);
  c->run_stream = st;
  drop_run_graphs(c, false);
  if (int r = evo_step(c, s, t0, EVO_PH_ALL, 0, stream)) return r;
  for (int i = 1; i < k;) {
    const int n = std::min(k - i, kRunGraphSteps);
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();  // e.g. the legacy default stream: run the rest eagerly
      for (; i < k; ++i)
        if (int r = evo_step(c, s + i, t0 + i, EVO_PH_ALL, 0, stream)) return r;
      return 0;
    }
    int rc = 0;
    for (int j = 0; j < n && !rc; ++j) rc = evo_step(c, s + i + j, t0 + i + j, EVO_PH_ALL, 0, stream);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    if (rc || e != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      return rc ? rc : fail((int)e, std::string("evo_run: stream capture failed: ") + cudaGetErrorString(e));
    }
    cudaGraphExec_t ge = nullptr;
    cudaError_t ei = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    CK(ei);
    c->run_execs.push_back(ge);
    CK(cudaGraphLaunch(ge, st));
    i += n;
  }
  return 0;
}

EVO_API int evo_refresh_ghosts(evo_ctx* c, void* stream) {
  if (int r = check_ctx(c)) return r;
  if (c->strip) return 0;
  if (int r = materialize(c, pick(c, stream))) return r;
  CK(evo::launch_refresh_ghosts(c->buf[c->front], c->geom(), pick(c, stream)));
  return 0;
}

EVO_API int evo_sync(evo_ctx* c) {
  if (int r = check_ctx(c)) return r;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  return 0;
}

EVO_API int evo_set_actions(evo_ctx* c, const int64_t* cells, int64_t n, const float* acts) {
  if (int r = check_ctx(c)) return r;
  if (n < 0 || (n > 0 && (!cells || !acts))) return fail(EVO_EINVAL, "bad action arrays");
  if (int r = ensure_actions_in(c)) return r;
  const long long nc = c->ncell();
  for (int64_t i = 0; i < n; ++i)
    if (cells[i] < 0 || cells[i] >= nc) return fail(EVO_EINVAL, "action cell index out of range");
  CK(cudaStreamSynchronize(c->stream));
  CK(zero_sync(c, c->act_in_flag, 0, (size_t)nc));
  if (n == 0) return 0;
  int64_t* dcells = nullptr;
  float* drows = nullptr;
  CK(cudaMalloc(&dcells, (size_t)n * 8));
  cudaError_t e = cudaMalloc(&drows, (size_t)n * evo::kActuators * 4);
  if (e == cudaSuccess) e = copy_sync(c, dcells, cells, (size_t)n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = copy_sync(c, drows, acts, (size_t)n * evo::kActuators * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = evo::launch_scatter_actions(c->act_in, c->act_in_flag, dcells, drows, n, nc, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dcells);
  cudaFree(drows);
  CK(e);
  return 0;
}

EVO_API int evo_get_actions(evo_ctx* c, int64_t capacity, int64_t* cells, float* acts, int64_t* n) {
  if (int r = check_ctx(c)) return r;
  if (!n) return fail(EVO_EINVAL, "n is null");
  if (!c->have_export || !c->exp_rows) return fail(EVO_EINVAL, "no exported actions (step with EVO_F_EXPORT_ACTIONS)");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  const long long nc = c->ncell();
  std::vector<uint8_t> flag((size_t)nc);
  std::vector<float> rows((size_t)nc * evo::kActuators);
  int64_t m = 0;
  if (c->exp_rank) {  // genome-sorted rows of 16 floats, located through the cell -> row map
    std::vector<int32_t> rank((size_t)nc);
    std::vector<float> srows((size_t)nc * 16);
    CK(copy_sync(c, rank.data(), c->exp_rank, (size_t)nc * 4, cudaMemcpyDeviceToHost));
    CK(copy_sync(c, srows.data(), c->exp_rows, srows.size() * 4, cudaMemcpyDeviceToHost));
    for (long long i = 0; i < nc; ++i) {
      const int r = rank[(size_t)i];
      if (r < 0) continue;
      if (m < capacity) {
        if (cells) cells[m] = i;
        if (acts) std::memcpy(acts + m * evo::kActuators, srows.data() + (size_t)r * 16, evo::kActuators * 4);
      }
      ++m;
    }
    *n = m;
    return 0;
  }
  CK(copy_sync(c, flag.data(), c->exp_flag, (size_t)nc, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, rows.data(), c->exp_rows, rows.size() * 4, cudaMemcpyDeviceToHost));
  for (long long i = 0; i < nc; ++i) {
    if (!flag[(size_t)i]) continue;
    if (m < capacity) {
      if (cells) cells[m] = i;
      if (acts) std::memcpy(acts + m * evo::kActuators, rows.data() + i * evo::kActuators, evo::kActuators * 4);
    }
    ++m;
  }
  *n = m;
  return 0;
}

EVO_API int evo_read_census(evo_ctx* c, int32_t* counts, int8_t* state, int64_t* death_step, int32_t* peak) {
  if (int r = check_ctx(c)) return r;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  const size_t cap = (size_t)c->cap;
  if (counts) CK(copy_sync(c, counts, c->census.counts_last, cap * 4, cudaMemcpyDeviceToHost));
  if (state) CK(copy_sync(c, state, c->census.state, cap, cudaMemcpyDeviceToHost));
  if (death_step) CK(copy_sync(c, death_step, c->census.death_step, cap * 8, cudaMemcpyDeviceToHost));
  if (peak) CK(copy_sync(c, peak, c->census.peak, cap * 4, cudaMemcpyDeviceToHost));
  return 0;
}

EVO_API int evo_census_take(evo_ctx* c, int32_t* counts) {
  if (int r = check_ctx(c)) return r;
  if (!counts) return fail(EVO_EINVAL, "null counts");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  CK(copy_sync(c, counts, c->census.counts, (size_t)c->cap * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemsetAsync(c->census.counts, 0, (size_t)c->cap * 4, c->stream));  // ordered before the next step
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

EVO_API int evo_read_stats(evo_ctx* c, int64_t* adoptions, int64_t* extinctions) {
  if (int r = check_ctx(c)) return r;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  long long st[2];
  CK(copy_sync(c, st, c->census.stats, sizeof(st), cudaMemcpyDeviceToHost));
  if (adoptions) *adoptions = st[0];
  if (extinctions) *extinctions = st[1];
  return 0;
}

EVO_API int evo_read_events(evo_ctx* c, int64_t capacity, int64_t* target, int64_t* source, int32_t* winner,
                            int32_t* defender, int64_t* direction, float* quantity, int64_t* m) {
  if (int r = check_ctx(c)) return r;
  if (!m) return fail(EVO_EINVAL, "m is null");
  if (!c->have_events || !c->ev_src) return fail(EVO_EINVAL, "no recorded events (step with EVO_F_RECORD_EVENTS)");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaDeviceSynchronize());
  const long long nc = c->ncell();
  std::vector<int64_t> src((size_t)nc);
  std::vector<float> q((size_t)nc);
  std::vector<int32_t> def((size_t)nc), gi((size_t)nc);
  std::vector<uint8_t> rot((size_t)nc);
  // events belong to the step that produced the current front buffer
  const evo::Planes& p = c->buf[c->front];
  CK(copy_sync(c, src.data(), c->ev_src, (size_t)nc * 8, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, q.data(), c->ev_q, (size_t)nc * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, def.data(), c->ev_def, (size_t)nc * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, gi.data(), p.gi + c->W, (size_t)nc * 4, cudaMemcpyDeviceToHost));
  CK(copy_sync(c, rot.data(), p.rot + c->W, (size_t)nc, cudaMemcpyDeviceToHost));
  int64_t k = 0;
  for (long long i = 0; i < nc; ++i) {
    if (src[(size_t)i] < 0) continue;
    if (k < capacity) {
      if (target) target[k] = c->row0 * c->W + i;
      if (source) source[k] = src[(size_t)i];
      if (winner) winner[k] = gi[(size_t)i];
      if (defender) defender[k] = def[(size_t)i];
      if (direction) direction[k] = rot[(size_t)i];
      if (quantity) quantity[k] = q[(size_t)i];
    }
    ++k;
  }
  *m = k;
  return 0;
}

EVO_API int evo_patch_genomes(evo_ctx* c, const int64_t* cells, const int32_t* slots, int64_t n) {
  if (int r = check_ctx(c)) return r;
  if (n <= 0) return 0;
  if (!cells || !slots) return fail(EVO_EINVAL, "null arrays");
  const long long nc = c->ncell();
  for (int64_t i = 0; i < n; ++i) {
    if (cells[i] < 0 || cells[i] >= nc) return fail(EVO_EINVAL, "cell index out of range");
    if (slots[i] < -1 || slots[i] >= c->cap) return fail(EVO_EINVAL, "slot outside the pool capacity");
  }
  CK(cudaStreamSynchronize(c->stream));
  int64_t* dc = nullptr;
  int32_t* ds = nullptr;
  CK(cudaMalloc(&dc, (size_t)n * 8));
  cudaError_t e = cudaMalloc(&ds, (size_t)n * 4);
  if (e == cudaSuccess) e = copy_sync(c, dc, cells, (size_t)n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = copy_sync(c, ds, slots, (size_t)n * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = evo::launch_patch_genomes(c->buf[c->front].gi, c->W, dc, ds, n, c->stream);
  if (e == cudaSuccess && !c->strip) e = evo::launch_refresh_ghosts(c->buf[c->front], c->geom(), c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dc);
  cudaFree(ds);
  CK(e);
  return 0;
}

EVO_API int evo_express_cppn(evo_ctx* c, int n, const int32_t* slots, const int32_t* node_off,
                             const int32_t* nodes, const int32_t* edge_src, const double* edge_w,
                             const int32_t* outs, const double* coords, double tau, double w_max, void* stream) {
  if (int r = check_ctx(c)) return r;
  if (!(tau >= 0.0 && tau < 1.0)) return fail(EVO_EINVAL, "tau must be in [0, 1)");
  if (!(w_max > 0.0)) return fail(EVO_EINVAL, "w_max must be positive");
  if (n < 0) return fail(EVO_EINVAL, "negative genome count");
  if (n == 0) return 0;
  if (!slots || !node_off || !nodes || !outs || !coords) return fail(EVO_EINVAL, "null arrays");
  // validate the programs on the host: node ranges, topological edges, outputs
  if (node_off[0] != 0) return fail(EVO_EINVAL, "node_off[0] must be 0");
  int max_nodes = 0;
  int64_t n_edges = 0;
  for (int g = 0; g < n; ++g) {
    if (slots[g] < 0 || slots[g] >= c->cap) return fail(EVO_EINVAL, "slot outside the pool capacity");
    const int a = node_off[g], b = node_off[g + 1];
    if (b <= a) return fail(EVO_EINVAL, "empty or unordered program");
    max_nodes = std::max(max_nodes, b - a);
    for (int i = a; i < b; ++i) {
      const int32_t* nd = nodes + 4 * (size_t)i;
      if (nd[0] < -1 || nd[0] > 5) return fail(EVO_EINVAL, "unknown activation code");
      if (nd[0] < 0 && (nd[1] < 0 || nd[1] > 4)) return fail(EVO_EINVAL, "input position outside 0..4");
      if (nd[2] < 0 || nd[3] < nd[2]) return fail(EVO_EINVAL, "bad edge range");
      n_edges = std::max<int64_t>(n_edges, nd[3]);
      for (int e = nd[2]; e < nd[3]; ++e)
        if (!edge_src || !edge_w || edge_src[e] < 0 || edge_src[e] >= i - a)
          return fail(EVO_EINVAL, "edge source is not an earlier node of the same program");
    }
    if (outs[2 * g] < 0 || outs[2 * g] >= b - a || outs[2 * g + 1] < 0 || outs[2 * g + 1] >= b - a)
      return fail(EVO_EINVAL, "output node outside the program");
  }
  if (evo::cppn_threads(max_nodes) == 0) return fail(EVO_EINVAL, "pattern network too large (> 384 nodes)");
  const int ncoord = 2 * (evo::kSensors + c->hidden + evo::kActuators);
  const int total_nodes = node_off[n];
  // one staging allocation: ints | doubles
  const size_t bi = ((size_t)n + (n + 1) + 4 * (size_t)total_nodes + (size_t)n_edges + 2 * (size_t)n) * 4;
  const size_t bd = ((size_t)n_edges + ncoord) * 8;
  const size_t off_d = (bi + 15) & ~(size_t)15;
  cudaStream_t st = pick(c, stream);
  char* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, off_d + bd));
  std::vector<char> h(off_d + bd);
  size_t o = 0;
  auto put = [&](const void* src, size_t bytes) {
    if (bytes) std::memcpy(h.data() + o, src, bytes);
    o += bytes;
  };
  evo::CppnBatch b{};
  b.n = n;
  b.max_nodes = max_nodes;
  b.tau = tau;
  b.w_max = w_max;
  b.nodes = reinterpret_cast<const int4*>(dbuf + o);  // first: int4 needs 16-byte alignment
  put(nodes, (size_t)total_nodes * 16);
  b.slots = reinterpret_cast<const int32_t*>(dbuf + o);
  put(slots, (size_t)n * 4);
  b.node_off = reinterpret_cast<const int32_t*>(dbuf + o);
  put(node_off, (size_t)(n + 1) * 4);
  b.edge_src = reinterpret_cast<const int32_t*>(dbuf + o);
  put(edge_src, (size_t)n_edges * 4);
  b.outs = reinterpret_cast<const int32_t*>(dbuf + o);
  put(outs, (size_t)n * 8);
  o = off_d;
  b.edge_w = reinterpret_cast<const double*>(dbuf + o);
  put(edge_w, (size_t)n_edges * 8);
  b.coords = reinterpret_cast<const double*>(dbuf + o);
  put(coords, (size_t)ncoord * 8);
  cudaError_t e = cudaMemcpyAsync(dbuf, h.data(), h.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = evo::launch_express_cppn(b, c->params(), c->wA, c->bA, c->wB, c->bB, st);
  c->frag_stale = true;
  c->shard_stale = true;
  c->htab_stale = true;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dbuf);
  CK(e);
  return 0;
}

namespace {
int ensure_select(evo_ctx* c) {
  if (c->sel_list) return 0;
  const long long n = c->ncell();
  cudaError_t e;
  if ((e = c->alloc(&c->sel_list, (size_t)n)) != cudaSuccess ||
      (e = c->alloc(&c->sel_chunk_cnt, (size_t)evo::select_chunks(n) + 1)) != cudaSuccess ||
      (e = c->alloc(&c->sel_chunk_off, (size_t)evo::select_chunks(n) + 1)) != cudaSuccess ||
      (e = c->alloc(&c->sel_n, 1)) != cudaSuccess || (e = c->alloc(&c->sel_parent, (size_t)c->cap)) != cudaSuccess ||
      (e = c->alloc(&c->sel_map, (size_t)c->cap)) != cudaSuccess)
    return fail((int)e, std::string("selection buffers: ") + cudaGetErrorString(e));
  return 0;
}
}  // namespace

EVO_API int evo_count_occupied(evo_ctx* c, int64_t* n_occupied) {
  if (int r = check_ctx(c)) return r;
  if (!n_occupied) return fail(EVO_EINVAL, "n_occupied is null");
  if (int r = ensure_select(c)) return r;
  const long long n = c->ncell();
  CK(evo::launch_count_occupied(c->buf[c->front].gi + c->W, n, c->sel_chunk_cnt, c->sel_chunk_off, c->stream));
  long long tot = 0;
  CK(cudaMemcpyAsync(&tot, c->sel_chunk_off + evo::select_chunks(n), sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *n_occupied = tot;
  return 0;
}

EVO_API int evo_select_cells_at(evo_ctx* c, uint64_t key_lo, uint64_t key_hi, double p, int64_t first_draw,
                                int32_t* parent_counts, int64_t* n_selected) {
  if (int r = check_ctx(c)) return r;
  if (!(p >= 0.0 && p <= 1.0)) return fail(EVO_EINVAL, "selection probability must be in [0, 1]");
  if (first_draw < 0) return fail(EVO_EINVAL, "first_draw must be >= 0");
  if (int r = ensure_select(c)) return r;
  const long long n = c->ncell();
  CK(evo::launch_select_cells(c->buf[c->front].gi + c->W, n, key_lo, key_hi, p, c->sel_chunk_cnt, c->sel_chunk_off,
                              c->sel_list, c->sel_n, c->sel_parent, c->cap, (long long)first_draw, c->stream));
  c->have_select = true;
  unsigned long long ns = 0;
  CK(cudaMemcpyAsync(&ns, c->sel_n, sizeof(ns), cudaMemcpyDeviceToHost, c->stream));
  if (parent_counts)
    CK(cudaMemcpyAsync(parent_counts, c->sel_parent, (size_t)c->cap * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (n_selected) *n_selected = (int64_t)ns;
  return 0;
}

EVO_API int evo_select_cells(evo_ctx* c, uint64_t key_lo, uint64_t key_hi, double p, int32_t* parent_counts,
                             int64_t* n_selected) {
  if (int r = check_ctx(c)) return r;
  if (c->strip) return fail(EVO_EINVAL, "a strip context draws after the strips above it: use evo_select_cells_at");
  return evo_select_cells_at(c, key_lo, key_hi, p, 0, parent_counts, n_selected);
}

EVO_API int evo_read_selected(evo_ctx* c, int64_t capacity, int64_t* cells, int64_t* n) {
  if (int r = check_ctx(c)) return r;
  if (!c->have_select) return fail(EVO_EINVAL, "no selection: call evo_select_cells first");
  unsigned long long ns = 0;
  CK(copy_sync(c, &ns, c->sel_n, sizeof(ns), cudaMemcpyDeviceToHost));
  if (n) *n = (int64_t)ns;
  if (!cells) return 0;
  if ((long long)ns > capacity) return fail(EVO_EINVAL, "cells buffer too small");
  std::vector<int32_t> tmp(ns);
  CK(copy_sync(c, tmp.data(), c->sel_list, ns * 4, cudaMemcpyDeviceToHost));
  std::sort(tmp.begin(), tmp.end());
  for (size_t i = 0; i < tmp.size(); ++i) cells[i] = tmp[i];
  return 0;
}

EVO_API int evo_remap_selected(evo_ctx* c, const int32_t* slot_map) {
  if (int r = check_ctx(c)) return r;
  if (!c->have_select) return fail(EVO_EINVAL, "no selection: call evo_select_cells first");
  if (!slot_map) return fail(EVO_EINVAL, "null slot map");
  for (int i = 0; i < c->cap; ++i)
    if (slot_map[i] < -1 || slot_map[i] >= c->cap) return fail(EVO_EINVAL, "slot map entry outside the pool");
  CK(cudaMemcpyAsync(c->sel_map, slot_map, (size_t)c->cap * 4, cudaMemcpyHostToDevice, c->stream));
  CK(evo::launch_remap_selected(c->buf[c->front].gi + c->W, c->sel_list, c->sel_n, c->sel_map, c->ncell(), c->stream));
  CK(evo::launch_refresh_ghosts(c->buf[c->front], c->geom(), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->have_select = false;  // the selection is consumed
  return 0;
}

EVO_API int evo_host_register(void* p, int64_t bytes) {
  if (!p || bytes <= 0) return fail(EVO_EINVAL, "empty host range");
  cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return 0;
  }
  CK(e);
  return 0;
}

EVO_API int evo_host_unregister(void* p) {
  if (!p) return fail(EVO_EINVAL, "null pointer");
  cudaError_t e = cudaHostUnregister(p);
  if (e == cudaErrorHostMemoryNotRegistered) {
    cudaGetLastError();
    return 0;
  }
  CK(e);
  return 0;
}

EVO_API int evo_halo_row_words(evo_ctx* c, int which, int64_t* words) {
  if (int r = check_ctx(c)) return r;
  if ((which != 0 && which != 1) || !words) return fail(EVO_EINVAL, "which must be 0 (front) or 1 (pass-1 outputs)");
  *words = (int64_t)(which == 0 ? 5 : 3) * c->W;
  return 0;
}

EVO_API int evo_halo_pack(evo_ctx* c, int which, void* send, void* stream) {
  if (int r = check_ctx(c)) return r;
  if ((which != 0 && which != 1) || !send) return fail(EVO_EINVAL, "bad halo pack arguments");
  // fused / lazy strip steps: the same rows from the pass-1 records, or from
  // the sense texture while it holds the state
  if ((which == 0 && c->tex_state) || (which == 1 && c->mid_rec)) {
    CK(evo::launch_halo_rec(c->gat.tex, c->hid.act, c->geom(), which, true, send, pick(c, stream)));
    return 0;
  }
  CK(evo::launch_halo(c->buf[c->front], c->mid, c->geom(), which, true, send, pick(c, stream)));
  return 0;
}

EVO_API int evo_halo_unpack(evo_ctx* c, int which, const void* recv, void* stream) {
  if (int r = check_ctx(c)) return r;
  if ((which != 0 && which != 1) || !recv) return fail(EVO_EINVAL, "bad halo unpack arguments");
  if ((which == 0 && c->tex_state) || (which == 1 && c->mid_rec)) {
    CK(evo::launch_halo_rec(c->gat.tex, c->hid.act, c->geom(), which, false, const_cast<void*>(recv),
                            pick(c, stream)));
    return 0;
  }
  CK(evo::launch_halo(c->buf[c->front], c->mid, c->geom(), which, false, const_cast<void*>(recv), pick(c, stream)));
  return 0;
}

EVO_API int evo_plane_ptr(evo_ctx* c, int which, int buffer, void** ptr, int64_t* plane_stride) {
  if (!c || !ptr) return fail(EVO_EINVAL, "null argument");
  if (which <= 2) {  // the caller may read or write E, I, C behind the library's back
    if (int r = materialize(c, c->stream)) return r;
    CK(cudaStreamSynchronize(c->stream));
  }
  const evo::Planes& p = c->buf[(c->front ^ (buffer ? 1 : 0)) & 1];
  switch (which) {
    case 0: *ptr = p.E; break;
    case 1: *ptr = p.I; break;
    case 2: *ptr = p.C; break;
    case 3: *ptr = p.gi; break;
    case 4: *ptr = p.rot; break;
    case 5: *ptr = c->mid.I; break;
    case 6: *ptr = c->mid.gi; break;
    case 7: *ptr = c->mid.rp; break;
    case 8: *ptr = c->mid.q; break;
    case 9: *ptr = c->census.counts; break;      /* int32 [capacity] accumulated counts */
    case 10: *ptr = c->census.stats; break;      /* int64 [2] adoptions, extinctions */
    default: return fail(EVO_EINVAL, "unknown plane");
  }
  if (plane_stride) *plane_stride = c->stride;
  return 0;
}

EVO_API int evo_debug_rcp_check(uint64_t* mismatches) {
  if (!mismatches) return fail(EVO_EINVAL, "null argument");
  unsigned long long n = 0;
  CK(evo::debug_rcp_check(&n));
  *mismatches = n;
  return 0;
}

EVO_API int evo_debug_phase_cycles(uint64_t* out8, int reset) {
  if (!out8) return fail(EVO_EINVAL, "null argument");
  CK(cudaDeviceSynchronize());
  CK(evo::debug_phase_cycles(reinterpret_cast<unsigned long long*>(out8), reset != 0));
  return 0;
}

EVO_API int evo_debug_hidden_cycles(uint64_t* out8, int reset) {
  if (!out8) return fail(EVO_EINVAL, "null argument");
  CK(cudaDeviceSynchronize());
  CK(evo::debug_hidden_cycles(reinterpret_cast<unsigned long long*>(out8), reset != 0));
  return 0;
}

EVO_API int evo_fnv1a64(uint64_t h, const uint8_t* data, int64_t n, uint64_t* out) {
  if (!out || (n > 0 && !data)) return fail(EVO_EINVAL, "null argument");
  const uint64_t prime = 0x100000001B3ULL;
  for (int64_t k = 0; k < n; ++k) h = (h ^ (uint64_t)data[k]) * prime;
  *out = h;
  return 0;
}

}  // extern "C"
