// Internal declarations shared by the kernels and the C ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "evoca_b200.h"

namespace evo {

constexpr int kTileW = 32;               // pass-1 tile: 32 x 32 cells
constexpr int kTileH = 32;
constexpr int kTileCells = kTileW * kTileH;
constexpr int kHaloW = kTileW + 2;       // tile + 1-cell Moore halo
constexpr int kHaloH = kTileH + 2;
constexpr int kHaloCells = kHaloW * kHaloH;
constexpr int kThreads1 = 256;           // pass-1 CTA
constexpr int kThreads2 = 256;           // pass-2 CTA
constexpr int kSensors = 45;             // hypernet.py:35-38
constexpr int kActuators = 13;
constexpr int kOutPad = 16;              // 13 actuators padded to 4 float4
constexpr int kMaxCapacity = 8192;       // device census bins per CTA (smem)
constexpr int kSmemWeightSlotsAbi = 68;  // largest pool the tile kernel keeps in shared memory
constexpr int kTcMinHidden = 64;
// Cluster-sharded pass 1 (evoca_shard.cu): 64 resident genomes per CTA.
constexpr int kShardSlots = 64;
constexpr int kShardFloats = kShardSlots * kSensors * 12 + ((kShardSlots * kSensors + 3) & ~3) + kShardSlots * kOutPad;
constexpr int kShardMaxQ = 4;
constexpr int kShardMaxLive = 768;       // larger live pools take the genome-sorted rows path         // narrowest hidden layer run on the tensor cores by default
// Tensor-core direct net (k_pass1_mma): per-genome weights in mma.sync A-fragment
// order, 6 K-steps x (lanes 0-19: 4 floats, lanes 20-31: 2 floats) + bias[16].
constexpr int kMmaSlots = 64;            // largest pool k_pass1_mma keeps in shared memory
constexpr int kFragStep = 20 * 4 + 12 * 2;
constexpr int kFragGenome = 6 * kFragStep + 16;

// Proposal byte written by pass 1 (one per cell): one-hot shipment direction
// (bit d set: the cell ships in direction d this step), 0 = no shipment.
// Pass 2 finds the arrivals at a target by masking each neighbour's byte
// with the one direction that points back at the target.

struct Scalars {
  int mode;  // 0 none, 1 day, 2 night
  float rho, drain;
  float kinv, kliq, einv, eliq, alpha, upkeep, dstarve, imin;
};

// Device state of one strip.  Every plane pointer addresses ghost row -1;
// row y (-1..H) lives at ptr + (y + 1) * W.
struct Planes {
  float* E;
  float* I;
  float* C;  // 3 planes, stride = plane stride
  int32_t* gi;
  uint8_t* rot;
};

struct Mid {
  float* I;      // infrastructure after invest/liquidate/upkeep and withdrawal
  int32_t* gi;   // genome after starvation deaths
  uint8_t* rp;   // proposal byte
  float* q;      // shipped quantity
};

struct Params {
  int hidden;     // 0 = direct 45->13
  int hpad;       // hidden rounded up to 8
  const float* wA;  // direct: W12 [cap][45][12];  hidden: W1 [cap][45][hpad]
  const float* bA;  // direct: bias [cap][16];     hidden: b1 [cap][hpad]
  const float* wB;  // direct: W1 [cap][45] (actuator 12); hidden: W2^T [cap][hpad][16]
  const float* bB;  // hidden: b2 [cap][16]
  const float* wF;  // direct, pools <= kMmaSlots: fragment-order table [cap][kFragGenome] (or null)
};

struct Census {
  int32_t* counts;       // accumulated by pass 2 (cap)
  int32_t* counts_last;  // published by the epilogue (cap)
  int8_t* state;         // 0 free 1 live 2 dead
  int64_t* death_step;
  int32_t* peak;
  unsigned int* done;    // CTA completion ticket
  long long* stats;      // [0] adoptions this step, [1] newly dead this step
};

struct Events {
  int64_t* src;   // per cell: global source index of the adopting winner, or -1
  float* q;
  int32_t* def;
};

struct StepGeom {
  int W, H;            // strip width / height
  long long row0;      // first global row of the strip
  int Hg;              // global torus height
  long long stride;    // elements per plane including ghost rows
  int own_ghosts;      // 1: single strip, kernels write the wrapped ghost rows themselves
};

struct Pass1Args {
  StepGeom g;
  Planes front, back;
  Mid mid;
  Params net;
  Scalars s;
  int phases;
  const float* src_map;      // nullable, (H,W)
  const float* act_in;       // inject: (H*W,13), or with act_rank: rank-ordered rows of 16
  const uint8_t* act_flag;   // inject: (H*W)
  const int32_t* act_rank;   // nullable: row of each cell in act_in (-1 = no actions)
  int act_decided;           // with act_rank: 1 -> 8-float decided records {inv, liq, m0..m2, xmax, kstar, 0}
                             // at each occupied CELL's index (spatial order; act_rank unused),
                             // 0 -> 16-float rows of the 13 squashed actuators at the cell's rank
  float* act_out;            // export: (H*W,13)
  uint8_t* act_out_flag;     // export: (H*W)
  int capacity;
  long long* stats;
};

struct Pass2Args {
  StepGeom g;
  Planes back;  // writes I, gi, rot
  const uint8_t* rot_front;  // pre-step rotation (pass 1 does not change it)
  Mid mid;
  const float* mid_rec;  // non-null: pass-1 outputs as 32-byte records at the cell index instead of the mid
                         // planes (FusedPhysics below); pass 2 then also writes the back E and C planes
  float* tex_out;        // with mid_rec, non-null (lazy): E', C' and the final I go to the texture records
                         // [(H + 2) * W][8] (the next step's sense texture) instead of the back E, I, C planes
  Census census;
  Events ev;     // ev.src == nullptr -> not recorded
  int capacity;
  int run_census;  // 1 -> last CTA runs the census epilogue
  long long t;
};

// Batched CPPN expression (evoca_cppn.cu): device copies of the linearised
// programs (paper_2406_09654_b200/neat.py:compile_programs).
struct CppnBatch {
  int n;                  // genomes
  int max_nodes;          // largest program
  const int32_t* slots;   // [n] destination pool slots
  const int32_t* node_off;  // [n + 1]
  const int4* nodes;      // {act | -1, input position | -1, edge begin, edge end}
  const int32_t* edge_src;  // node position within the genome
  const double* edge_w;
  const int32_t* outs;    // [n][2] weight / bias signal node positions
  const double* coords;   // (45 + hidden + 13) x 2 neuron coordinates
  double tau, w_max;
};

// Hidden-layer controller on tcgen05 (evoca_hidden_tc.cu): per-step buffers.
struct HidBuffers {
  int32_t* counts;   // [cap]
  int32_t* offs;     // [cap + 1]
  int32_t* tiles;    // [cap + 1]
  int32_t* cursor;   // [cap]
  int32_t* n_tiles;  // [1]
  int32_t* cta_hist;  // [sort CTAs][cap] per-CTA slot histograms -> row bases
  float* sens;       // [ncell][48]
  int4* tile_info;     // [ncell / 128 + cap] {slot, first row, rows, 0} per 128-row tile
  float* act;        // [ncell][16] actuator rows in sorted-row order, or [ncell][8] decided records in cell order
  int32_t* rank;     // [ncell] sorted row of each cell, -1 = empty
};
// Direct nets of large pools by gather (evoca_gather.cu): per-step buffers.
// Physics fused into the gather net (whole-torus evo_step, TMA texture
// build): the net's epilogue runs cell_physics on the cell's own texture
// record and writes one 32-byte pass-1 record {E', C0', C1', C2' | I', q,
// genome, proposal byte} at the cell index (unoccupied cells: the texture
// build writes theirs), which pass 2 consumes instead of the mid planes.
struct FusedPhysics {
  Scalars s;
  int phases;
  const float* src_map;  // nullable, (H,W)
  long long* stats;      // zeroed like pass 1 does
};
constexpr int kGatherMaxCap = 8192;  // per-CTA slot histogram in shared memory (32 KB)
struct GatherBuffers {
  float* tex;          // [(H + 2) * W][8] sense records {E, I, C0, C1, C2, 0, 0, 0}
  int32_t* cta_hist;   // [count CTAs][bins] per-CTA group counts -> bases inside the band's groups
  uint16_t* lrank;     // [ncell] rank of each cell inside its count CTA's group
  int32_t* band_hist;  // [nbands][bins] group sizes
  int32_t* goff;       // [nbands][bins + 1] group cell offsets within the band
  int32_t* ght;        // [nbands][bins + 1] group tile offsets within the band
  int32_t* band_tot;   // [nbands][2]
  int32_t* band_base;  // [nbands + 1][2]
  int32_t* n_ht;       // [2]: half-tiles, gather work counter
  uint32_t* sorted;    // [ncell] (rot << 29) | (y << 15) | x by (band, slot)
  int4* info;          // [max_ht] {slot, first, cells, 0}
};
// TMA tensor maps of one plane buffer for the texture build (k_gs_count_tma):
// E, I, C0, C1, C2 (f32) and the genome plane (i32), each 2-D [H + 2][W] from
// ghost row -1, box 256 x 1; the texture 3-D [H + 2][W][8], box 8 x 256 x 1
struct GatherMaps {
  CUtensorMap plane[6];
  CUtensorMap tex;
};
bool make_gather_maps(const Planes& f, const StepGeom& g, float* tex, GatherMaps* out);
struct GatherSizes {
  int nbands, nctas, bins;
  long long max_ht;
};
bool gather_supported(int W, int H, int cap);
GatherSizes gather_sizes(int W, int H, int cap, int num_sms);
constexpr int kGatherFfma2 = 0, kGatherTc = 2;  // net variants of the gather path
// cells sorted by (row band, slot) (one band: by slot over the whole strip),
// the sense texture, `tile`-cell tiles; rank (nullable): cell -> cell for
// occupied cells, -1 otherwise
cudaError_t launch_gather_sort(const GatherBuffers& b, const StepGeom& g, const Planes& front, int cap, int num_sms,
                               int tile, bool one_band, int32_t* rank, cudaStream_t st,
                               const GatherMaps* maps = nullptr, const FusedPhysics* fused = nullptr,
                               float* mid_rec = nullptr, bool tex_is_state = false);
// hidden-layer net (k_hid_net2) over the gather sort: rows at the cell index
cudaError_t launch_hidden_gather(const GatherBuffers& b, const StepGeom& g, const Params& net, int cap, int num_sms,
                                 const unsigned char* htab, float* act, cudaStream_t st);
size_t hidden_table_bytes(int hidden);  // per slot
cudaError_t launch_hidden_tables(const Params& net, int cap, unsigned char* out, cudaStream_t st);
bool hidden_gather_supported(int hidden);
cudaError_t launch_direct_gather(const GatherBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                                 int cap, int num_sms, int variant, bool export_rows, float* act, int32_t* rank,
                                 cudaStream_t st, const GatherMaps* maps = nullptr,
                                 const FusedPhysics* fused = nullptr, bool tex_is_state = false);
// E, I, C planes of `front` (ghost rows included) from the texture records
cudaError_t launch_tex_to_planes(const float* tex, const StepGeom& g, const Planes& front, int num_sms,
                                 cudaStream_t st);

bool hidden_tc_supported(int hidden);
bool hidden_net2_used(int hidden, bool l2_cuda_core);
int hidden_sort_ctas(int W, int H);
int hidden_tc_nh(int hidden);
size_t hidden_tc_smem(int hidden);
cudaError_t launch_hidden_tc(const HidBuffers& b, const StepGeom& g, const Planes& front, const Params& net,
                             int capacity, int num_sms, bool decided, bool l2_cuda_core, cudaStream_t st);

int select_chunks(long long n);
cudaError_t launch_select_cells(const int32_t* gi, long long n, unsigned long long k0, unsigned long long k1, double p,
                                int32_t* chunk_cnt, long long* chunk_off, int32_t* list, unsigned long long* n_sel,
                                int32_t* parent_cnt, int capacity, long long first_draw, cudaStream_t st);
// occupied cells of the plane: chunk_off[select_chunks(n)] <- the total
cudaError_t launch_count_occupied(const int32_t* gi, long long n, int32_t* chunk_cnt, long long* chunk_off,
                                  cudaStream_t st);
cudaError_t launch_remap_selected(int32_t* gi, const int32_t* list, const unsigned long long* n_sel,
                                  const int32_t* map, long long max_n, cudaStream_t st);
int cppn_threads(int max_nodes);  // 0 -> program too large
cudaError_t launch_express_cppn(const CppnBatch& b, const Params& net, float* wA, float* bA, float* wB, float* bB,
                                cudaStream_t st);
cudaError_t launch_pass1(const Pass1Args& a, bool inject, bool export_actions, cudaStream_t st);
cudaError_t launch_frag_relayout(const Params& net, int capacity, float* wF, cudaStream_t st);
cudaError_t launch_pass2(const Pass2Args& a, cudaStream_t st);
size_t shard_smem_bytes(int Q);
cudaError_t launch_shard_plan(const int8_t* state, int cap, int Q, int* map, int* resident, const Params& net,
                              float* tables, cudaStream_t st);
cudaError_t launch_pass1_shard(const Pass1Args& a, const int* map, const float* tables, int Q, int num_sms,
                               cudaStream_t st);
cudaError_t debug_phase_cycles(unsigned long long* out, bool reset);
cudaError_t debug_rcp_check(unsigned long long* host_out);
cudaError_t debug_hidden_cycles(unsigned long long* out, bool reset);
cudaError_t launch_census_finish(const Census& c, int capacity, long long t, cudaStream_t st,
                                 const int* skip = nullptr);
cudaError_t launch_refresh_ghosts(const Planes& p, const StepGeom& g, cudaStream_t st);
cudaError_t launch_render_rgb(const Planes& f, const StepGeom& g, double norm_e, double norm_i, uint32_t* out,
                              cudaStream_t st);
// observables (evoca_metrics.cu)
int msc_side(int W, int H);
long long msc_workspace_doubles(int side);
int msc_digits();
cudaError_t launch_msc(const float* plane, int W, int H, int n_scales, double* work, long long* accs, double* out,
                       int* k_max_out, cudaStream_t st);
long long plane_sum_chunks(long long n);
cudaError_t launch_plane_sum(const float* plane, long long n, double* chunks, double* out, cudaStream_t st);
cudaError_t launch_wrap_mid(const Mid& m, const StepGeom& g, cudaStream_t st);
cudaError_t launch_check_cells(int32_t* gi, uint8_t* rot, long long n, int capacity, int* bad, cudaStream_t st);
cudaError_t launch_halo(const Planes& f, const Mid& m, const StepGeom& g, int which, bool pack, void* buf,
                        cudaStream_t st);
// the same exchange on the fused step's buffers (texture records for which = 0, pass-1 records for which = 1)
cudaError_t launch_halo_rec(float* tex, float* rec, const StepGeom& g, int which, bool pack, void* buf,
                            cudaStream_t st);
cudaError_t launch_scatter_actions(float* act, uint8_t* flag, const int64_t* cells, const float* rows, long long n,
                                   long long ncell, cudaStream_t st);
cudaError_t launch_patch_genomes(int32_t* gi, int W, const int64_t* cells, const int32_t* slots, long long n,
                                 cudaStream_t st);

}  // namespace evo
