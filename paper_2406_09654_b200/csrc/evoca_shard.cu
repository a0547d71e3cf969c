// Pass 1 for direct nets of pools larger than one shared-memory weight table
// (BASELINE config 3: 256 genomes + radiation children), fused per tile with
// the genome weight table SHARDED over a thread-block cluster.  A measured
// alternative to the genome-sorted rows path, selected with EVO_F_SHARD_NET:
// bit-identical results, and it removes the 384 bytes per cell of sensor-row
// traffic, but on config 3 it runs the step in 4.7 ms against 2.4 ms - each
// CTA evaluates only ~256 of a tile's cells (~140 same-genome pairs for 256
// threads), so its per-tile latency chain (halo wait, 45-step FFMA2 chains,
// DSMEM records, cluster barrier) is exposed with ~4 active warps per SM
// (DESIGN.md section 3).
//
// One 32x32 tile's cells carry ~all of the pool's genomes, and 64 genomes'
// weights (154 KB) are what one SM's shared memory holds next to the tile.
// So a cluster of Q CTAs (Q SMs) works on the same tile at the same time:
// CTA r keeps the weights of shard r (64 "resident" slots) in shared memory
// for the whole launch, stages the tile's halo itself (the Q CTAs read the
// same lines, deduplicated in L2), buckets only the cells whose genome is in
// its shard (pairs of same-genome cells, the tile kernel's FFMA2 net and k
// order: results bit-identical to k_pass1_direct and the genome-sorted rows
// path), and ships each decided action record (32 bytes: invest, liquidate,
// comm x3, explore max, argmax) through distributed shared memory to the CTA
// that owns the cell's row band of the tile.  After one cluster barrier
// every CTA runs the fused physics tail (physics.py:178-290) for its band in
// spatial order with coalesced stores.  Records are double-buffered, so one
// cluster barrier per tile orders everything.
//
// Slots that are live but not resident (beyond 64 Q, e.g. freshly irradiated
// children with a few hundred cells each) are "stragglers": the CTA whose
// rank is the tile index mod Q evaluates them one cell per thread with the
// weights read from global memory (L2-resident tables).
//
// HBM traffic per cell: the 25-byte state read once (+ halo rows), the
// pass-1 outputs written once - no sensor rows (the genome-sorted path
// writes and reads 192 bytes of rows per cell).
//
// k_shard_map / k_shard_tables build the residency map and the per-shard
// weight tables on the device whenever the pool changed (evo_set_params,
// evo_express_cppn, evo_set_slots mark the context's plan dirty).

#include <algorithm>

#include "evoca_tile.cuh"

namespace evo {

namespace {

constexpr int kShardThreads = 256;
constexpr int kShardPre = (kTileCells + kShardThreads - 1) / kShardThreads;

__host__ __device__ constexpr int region_row0(int p, int Q) { return (p * kTileH) / Q; }
__device__ __forceinline__ int region_owner(int ty, int Q) { return ((ty + 1) * Q - 1) / kTileH; }

struct ShardSmem {
  float4 eic[kHaloCells];
  float c2[kHaloCells];
  int gi[kTileCells];
  uint8_t rot[kTileCells];
  uint8_t key[kTileCells];  // local genome index within this shard, or 0xFF
  unsigned short order[2 * kTileCells];
  unsigned short strag[kTileCells];
  int n_strag;
  int slot_off[72];
  int scratch[kShardThreads / 32];
  int n_units;
  int bins[kShardSlots];
  unsigned long long bar[2];  // per record buffer: this CTA's band records delivered
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_remote(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
// 16 bytes into a peer CTA's shared memory; the write completes 16 bytes of
// the transaction count of the peer's mbarrier (no fence, no polling)
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// progress barrier without a memory fence (record data is ordered by the
// mbarriers); keeps every CTA within one tile of its peers
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// shard key of a cell's genome slot: (rank << 8) | local for resident slots,
// 0xFFFF for a live straggler, -1 for an empty cell
__device__ __forceinline__ int shard_key(const int* map, int slot) {
  return slot < 0 ? -1 : __ldg(map + slot);
}

}  // namespace

// Residency: the first 64 Q live slots in slot order, dealt round-robin to
// the Q shards (rank = i mod Q, local index = i / Q); one CTA.
__global__ void __launch_bounds__(1024) k_shard_map(const int8_t* state, int cap, int Q, int* map, int* resident) {
  __shared__ int scratch[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  for (int i = threadIdx.x; i < Q * kShardSlots; i += blockDim.x) resident[i] = -1;
  __syncthreads();
  for (int b0 = 0; b0 < cap; b0 += 1024) {
    const int s = b0 + threadIdx.x;
    const int live = (s < cap && state[s] == 1) ? 1 : 0;
    int total;
    const int before = block_exclusive_sum<1024>(live, scratch, total);
    if (s < cap) {
      const int i = carry + before;
      if (live && i < Q * kShardSlots) {
        const int r = i % Q, l = i / Q;
        map[s] = (r << 8) | l;
        resident[r * kShardSlots + l] = s;
      } else {
        map[s] = 0xFFFF;  // not resident: a live straggler (free / dead slots own no cells)
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

// Per-shard weight tables in the layout k_pass1_direct stages: W12 [64][45][12]
// | W1 [64][45] (padded to 4) | bias [64][16]; empty entries zero.
__global__ void k_shard_tables(const Params net, const int* resident, int Q, float* tables) {
  constexpr int w1off = kShardSlots * kSensors * 12;
  constexpr int boff = w1off + ((kShardSlots * kSensors + 3) & ~3);
  const long long n = (long long)Q * kShardFloats;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / kShardFloats), e = (int)(i - (long long)r * kShardFloats);
    float v = 0.0f;
    if (e < w1off) {
      const int l = e / (kSensors * 12), k = e - l * kSensors * 12;
      const int s = resident[r * kShardSlots + l];
      if (s >= 0) v = net.wA[(size_t)s * kSensors * 12 + k];
    } else if (e < boff) {
      const int j = e - w1off, l = j / kSensors, k = j - l * kSensors;
      const int s = l < kShardSlots ? resident[r * kShardSlots + l] : -1;
      if (s >= 0) v = net.wB[(size_t)s * kSensors + k];
    } else {
      const int j = e - boff, l = j / kOutPad, k = j - l * kOutPad;
      const int s = resident[r * kShardSlots + l];
      if (s >= 0) v = net.bA[(size_t)s * kOutPad + k];
    }
    tables[i] = v;
  }
}

namespace {

// decided action record of one cell: {inv, liq, m0, m1}, {m2, xmax, kstar, 0},
// sent to the CTA owning the cell's row band (32 bytes of its mbarrier tx)
__device__ __forceinline__ void send_record(uint32_t rec_base, uint32_t bar, int pos, int Q, const float* z) {
  const int ty = pos / kTileW, tx = pos - ty * kTileW;
  const int p = region_owner(ty, Q);
  const int li = (ty - region_row0(p, Q)) * kTileW + tx;
  int ks;
  float xm;
  explore_pick(z + 5, ks, xm);
  const uint32_t dst = map_remote(rec_base + (uint32_t)li * 32u, (uint32_t)p);
  const uint32_t rbar = map_remote(bar, (uint32_t)p);
  st_async_v4(dst, make_float4(squash(z[0]), squash(z[1]), squash(z[2]), squash(z[3])), rbar);
  st_async_v4(dst + 16u, make_float4(squash(z[4]), xm, __int_as_float(ks), 0.0f), rbar);
}

}  // namespace

__global__ void __launch_bounds__(kShardThreads, 1) k_pass1_shard(const Pass1Args a, const int* map,
                                                                   const float* tables, int Q) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ShardSmem& sm = *reinterpret_cast<ShardSmem*>(smem_raw);
  const StepGeom& g = a.g;
  const int rank = (int)cta_rank();
  const int cluster = blockIdx.x / Q, nclusters = gridDim.x / Q;
  const int tiles_x = (g.W + kTileW - 1) / kTileW;
  const int ntiles = tiles_x * ((g.H + kTileH - 1) / kTileH);
  const int region_cells = (region_row0(rank + 1, Q) - region_row0(rank, Q)) * kTileW;
  const int max_region = ((kTileH + Q - 1) / Q) * kTileW;
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.stats) {
    a.stats[0] = 0;
    a.stats[1] = 0;
  }
  // this shard's weights, resident for the whole launch
  const size_t off = (sizeof(ShardSmem) + 15) & ~(size_t)15;
  float* sW12 = reinterpret_cast<float*>(smem_raw + off);
  float* sW1 = sW12 + kShardSlots * kSensors * 12;
  float* sB = sW1 + ((kShardSlots * kSensors + 3) & ~3);
  float4* rec = reinterpret_cast<float4*>(sW12 + kShardFloats);  // [2][max_region][2] records
  const uint32_t rec_addr = (uint32_t)__cvta_generic_to_shared(rec);
  stage_weights<kShardThreads>(sW12, tables + (size_t)rank * kShardFloats, kShardFloats);
  asm volatile("cp.async.commit_group;" ::: "memory");
  fill_slot_offsets(sm.slot_off);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sm.bar[0]);
  if (threadIdx.x == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8u, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();  // peers' barriers initialised before any record is sent

  int tile = cluster;
  int rank_in[kShardPre];
  int key_pf[kShardPre];
  auto count = [&](const PrefetchT<kShardThreads>& pf, int t) {
    // keys of the prefetched tile for this shard, stragglers listed
    const bool mine_strag = (t % Q) == rank;
#pragma unroll
    for (int j = 0; j < kShardPre; ++j) {
      const int k = shard_key(map, pf.gi[j]);
      const bool mine = k >= 0 && k != 0xFFFF && (k >> 8) == rank;
      key_pf[j] = mine ? (k & 0xFF) : -1;
      const int pos = threadIdx.x + j * kShardThreads;
      if (mine_strag && k == 0xFFFF && pos < kTileCells) sm.strag[atomicAdd(&sm.n_strag, 1)] = (unsigned short)pos;
    }
    bucket_count<kShardThreads, kShardPre>(sm.bins, key_pf, rank_in);
  };
  auto commit = [&](const PrefetchT<kShardThreads>& pf) {
    commit_tile(sm, pf);
#pragma unroll
    for (int j = 0; j < kShardPre; ++j) {
      const int pos = threadIdx.x + j * kShardThreads;
      if (pos < kTileCells) sm.key[pos] = key_pf[j] >= 0 ? (uint8_t)key_pf[j] : (uint8_t)0xFF;
    }
  };
  if (tile < ntiles) {
    PrefetchT<kShardThreads> pf;
    prefetch_tile(a, tile, tiles_x, pf);
    for (int b = threadIdx.x; b < kShardSlots; b += kShardThreads) sm.bins[b] = 0;
    if (threadIdx.x == 0) sm.n_strag = 0;
    __syncthreads();
    count(pf, tile);
    __syncthreads();
    bucket_offsets<kShardThreads, 2, 2>(sm.bins, sm.scratch, sm.order, &sm.n_units, kShardSlots);
    __syncthreads();
    bucket_scatter<kShardThreads, kShardPre>(sm.bins, key_pf, rank_in, sm.order);
    commit(pf);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  int buf = 0;
  uint32_t phase = 0u;  // bit b: parity of record buffer b's mbarrier
  const int r0 = region_row0(rank, Q);
  for (; tile < ntiles; tile += nclusters) {
    const int x0 = (tile % tiles_x) * kTileW;
    const int y0 = (tile / tiles_x) * kTileH;
    const int next = tile + nclusters;
    if (next < ntiles) prefetch_tile_l2<kShardThreads>(a, next, tiles_x);
    const uint32_t rbase = rec_addr + (uint32_t)(buf * max_region * 32);
    const uint32_t mybar = bar0 + 8u * (uint32_t)buf;
    {  // records expected in this CTA's band: one per occupied cell
      int n_occ = 0;
      for (int i0 = 0; i0 < region_cells; i0 += kShardThreads) {
        const int i = i0 + threadIdx.x;
        bool occ = false;
        if (i < region_cells) {
          const int ty = r0 + i / kTileW, tx = i % kTileW;
          occ = y0 + ty < g.H && x0 + tx < g.W && sm.gi[ty * kTileW + tx] >= 0;
        }
        n_occ += __syncthreads_count(occ);
      }
      if (threadIdx.x == 0) mbar_expect(mybar, (uint32_t)n_occ * 32u);
    }
    // controller: this shard's cells in same-genome pairs (weights in smem)
    const int nu = sm.n_units;
    for (int q = threadIdx.x; q < nu; q += kShardThreads) {
      const unsigned w = reinterpret_cast<const unsigned*>(sm.order)[q];
      const int o0 = (int)(w & 0xFFFFu), o1 = (int)(w >> 16);
      if (o0 == 0xFFFF) continue;
      const bool v1 = o1 != 0xFFFF;
      const int pos[2] = {o0, v1 ? o1 : o0};
      int hb[2], rot[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int ty = pos[c] / kTileW, tx = pos[c] - ty * kTileW;
        hb[c] = (ty + 1) * kHaloW + tx + 1;
        rot[c] = sm.rot[pos[c]];
      }
      const int l = sm.key[o0];
      float out[2][kActuators];
      net_direct_unit<2, true>(sm, sW12 + (size_t)l * kSensors * 12, sW1 + (size_t)l * kSensors,
                               sB + (size_t)l * kOutPad, hb, rot, out);
      send_record(rbase, mybar, o0, Q, out[0]);
      if (v1) send_record(rbase, mybar, o1, Q, out[1]);
    }
    // stragglers (live slots without resident weights): one cell per thread,
    // weights from global memory
    const int ns = sm.n_strag;
    for (int i = threadIdx.x; i < ns; i += kShardThreads) {
      const int p0 = sm.strag[i];
      const int ty = p0 / kTileW, tx = p0 - ty * kTileW;
      const int hb[1] = {(ty + 1) * kHaloW + tx + 1};
      const int rot[1] = {sm.rot[p0]};
      const int slot = sm.gi[p0];
      float out[1][kActuators];
      net_direct_unit<1, false>(sm, a.net.wA + (size_t)slot * kSensors * 12, a.net.wB + (size_t)slot * kSensors,
                                a.net.bA + (size_t)slot * kOutPad, hb, rot, out);
      send_record(rbase, mybar, p0, Q, out[0]);
    }
    mbar_wait(mybar, (phase >> buf) & 1u);  // every record of this CTA's band delivered
    phase ^= 1u << buf;
    PrefetchT<kShardThreads> pf;
    if (next < ntiles) prefetch_tile(a, next, tiles_x, pf);
    // physics tail of this CTA's row band, spatial order, coalesced stores
    const float4* rb = rec + buf * max_region * 2;
    for (int i = threadIdx.x; i < region_cells; i += kShardThreads) {
      const int ty = r0 + i / kTileW, tx = i % kTileW;
      const int y = y0 + ty, x = x0 + tx;
      if (y >= g.H || x >= g.W) continue;
      const int p = ty * kTileW + tx, hp = (ty + 1) * kHaloW + tx + 1;
      const float4 f = sm.eic[hp];
      const CellState st{f.x, f.y, f.z, f.w, sm.c2[hp], sm.gi[p], sm.rot[p]};
      CellAct ac{};
      ac.acted = st.slot >= 0;
      if (ac.acted) {
        const float4 ra = rb[2 * i], rc = rb[2 * i + 1];
        ac.inv = ra.x;
        ac.liq = ra.y;
        ac.m0 = ra.z;
        ac.m1 = ra.w;
        ac.m2 = rc.x;
        ac.xmax = rc.y;
        ac.kstar = __float_as_int(rc.z);
      }
      store_pass1(a, y, x, cell_physics(a.s, a.phases, a.src_map, (long long)y * g.W + x, st, ac));
    }
    for (int b = threadIdx.x; b < kShardSlots; b += kShardThreads) sm.bins[b] = 0;
    if (threadIdx.x == 0) sm.n_strag = 0;
    __syncthreads();
    if (next < ntiles) {
      count(pf, next);
      __syncthreads();
      bucket_offsets<kShardThreads, 2, 2>(sm.bins, sm.scratch, sm.order, &sm.n_units, kShardSlots);
      __syncthreads();
      bucket_scatter<kShardThreads, kShardPre>(sm.bins, key_pf, rank_in, sm.order);
      commit(pf);
    }
    // every CTA of the cluster is done with this tile's records before any
    // peer can run two tiles ahead into the same buffer (also a CTA barrier)
    cluster_sync_relaxed();
    buf ^= 1;
  }
  cluster_sync();  // no CTA leaves while a peer can still address its shared memory
}

size_t shard_smem_bytes(int Q) {
  const int max_region = ((kTileH + Q - 1) / Q) * kTileW;
  return ((sizeof(ShardSmem) + 15) & ~(size_t)15) + (size_t)kShardFloats * 4 + (size_t)2 * max_region * 32;
}

cudaError_t launch_shard_plan(const int8_t* state, int cap, int Q, int* map, int* resident, const Params& net,
                              float* tables, cudaStream_t st) {
  k_shard_map<<<1, 1024, 0, st>>>(state, cap, Q, map, resident);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long long n = (long long)Q * kShardFloats;
  k_shard_tables<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(net, resident, Q, tables);
  return cudaGetLastError();
}

cudaError_t launch_pass1_shard(const Pass1Args& a, const int* map, const float* tables, int Q, int num_sms,
                               cudaStream_t st) {
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem = shard_smem_bytes(Q);
  cudaError_t e = cudaSuccess;
  if (dev < 0 || dev >= 64) dev = 0;
  if (configured[dev] < (int)smem) {
    e = cudaFuncSetAttribute(k_pass1_shard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_pass1_shard, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured[dev] = (int)smem;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = Q;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kShardThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // as many clusters as can be co-resident (a persistent grid must not wait
  // for a second wave): clusters of 4 cannot use every SM of every GPC
  cfg.gridDim = dim3(Q * (num_sms / Q), 1, 1);
  int max_clusters = 0;
  e = cudaOccupancyMaxActiveClusters(&max_clusters, k_pass1_shard, &cfg);
  if (e != cudaSuccess) return e;
  if (max_clusters <= 0) return cudaErrorInvalidConfiguration;
  const int tiles = ((a.g.W + kTileW - 1) / kTileW) * ((a.g.H + kTileH - 1) / kTileH);
  int nclusters = std::min(max_clusters, num_sms / Q);
  nclusters = std::max(1, std::min(nclusters, tiles));
  cfg.gridDim = dim3(Q * nclusters, 1, 1);
  return cudaLaunchKernelEx(&cfg, k_pass1_shard, a, map, tables, Q);
}

}  // namespace evo
