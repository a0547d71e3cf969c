/*
 * evoca_b200.h — C ABI of the B200-native substrate step.
 *
 * Drop-in boundary for the reference's per-step substrate update
 * (`evoca.engine.step`, /root/reference/pkg/src/evoca/engine.py:233-248) and
 * its operator-level phase functions (physics.py:178-404).  The reference is
 * pure Python; its FFI for this path would be a ctypes binding of exactly
 * these symbols (INTEGRATION.md shows the stub).  Plain pointers and sizes
 * only: no torch / CUDA types in any signature (streams are `void*` holding a
 * cudaStream_t, NULL = the context's own stream).
 *
 * Every function returns 0 on success, EVO_EINVAL on a rejected argument (the
 * reference raises ValueError there, e.g. physics.py:55-56, config.py), or a
 * positive cudaError_t code; evo_last_error() gives the message for the
 * calling thread.  The step itself never fails on valid state
 * ("physics itself never fails").
 *
 * State layout (one context = one row strip; a single GPU is one strip that
 * holds the whole torus): structure-of-arrays planes, row-major, linear index
 * y*W + x (substrate.py:9-11):
 *   energy f32 (H,W), infrastructure f32 (H,W), communication f32 (3,H,W),
 *   genome_index i32 (H,W) (-1 = empty), rotation u8 (H,W) in 0..7
 * (substrate.py:45-75).  Device copies carry one ghost row above and below.
 */
#ifndef EVOCA_B200_H
#define EVOCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVO_API __attribute__((visibility("default")))

#define EVO_OK 0
#define EVO_EINVAL (-1)

/* Phase mask for evo_step / evo_pass1 (engine.py:240-243 order). */
#define EVO_PH_ENERGY 1   /* physics.energy_cycle        physics.py:178-194 */
#define EVO_PH_INVEST 2   /* physics.apply_invest_liquidate physics.py:197-233 */
#define EVO_PH_COMM 4     /* physics.write_communication physics.py:236-247 */
#define EVO_PH_EXPLORE 8  /* physics.resolve_exploration physics.py:250-343 */
#define EVO_PH_ALL 15

/* Step flags. */
#define EVO_F_INJECT_ACTIONS 1  /* use the ActionField set by evo_set_actions instead of sense+net */
#define EVO_F_EXPORT_ACTIONS 2  /* keep the computed ActionField for evo_get_actions (engine.py:193) */
#define EVO_F_RECORD_EVENTS 4   /* keep AdoptionEvents for evo_read_events (physics.py:134-175) */
#define EVO_F_NO_CENSUS 8       /* strip mode: census epilogue runs after the cross-rank count reduction */
#define EVO_F_CUDA_CORE_NET 16  /* hidden-layer nets: per-cell CUDA-core FP32 forward instead of the tcgen05 path */
#define EVO_F_TILE_NET 32       /* direct nets of pools > 68 slots: per-tile kernel instead of genome-sorted rows */
#define EVO_F_MMA_NET 64        /* direct nets of pools <= 64 slots: mma.sync 3xTF32 tile kernel (measured slower; A/B) */
#define EVO_F_TC_NET 128        /* hidden layers narrower than 64: tcgen05 3xTF32 net instead of FP32 CUDA cores */
#define EVO_F_SHARD_NET 256     /* direct nets of pools > 68 slots: cluster-sharded tile kernel (measured slower; A/B) */
#define EVO_F_ROWS_NET 512      /* direct nets of pools > 68 slots: genome-sorted sensor rows in HBM (round-2 path; A/B) */
#define EVO_F_GATHER_NET 1024   /* the gather path for direct pools <= 68 slots and for tensor-core hidden nets (A/B) */
#define EVO_F_TC_DIRECT 2048    /* gather path: the direct net as tcgen05 3xTF32 MMAs (A in TMEM) instead of FFMA2 warps */
#define EVO_F_L2_CUDA_CORE 4096 /* tensor-core hidden net: layer 2 as FP32 FMAs on the CUDA cores (round-2 kernel; A/B) */
#define EVO_F_UNFUSED 8192      /* gather path in evo_step/evo_run: physics as its own kernel over the mid planes (round-2d; A/B) */
#define EVO_F_FUSE_MID 16384    /* evo_pass1: the evo_pass2 of the same step follows (a strip's evo_halo_pack/unpack(1)
                                   between them is fine), so pass-1 outputs may stay 32-byte records instead of the mid
                                   planes (evo_step sets it; gather path only) */
#define EVO_F_LAZY 32768        /* evo_pass1, with EVO_F_FUSE_MID: evo_pass2 and evo_swap follow, so pass 2 may leave E, I, C
                                   in the sense texture and skip the planes until an entry point needs them (evo_step
                                   sets it; strips: evo_halo_pack/unpack(0) then exchange texture rows) */

/* Host-computed per-step scalars, exactly as the reference derives them:
 * rho = A*sin(2*pi*t/P) in float64 (physics.py:186); rho_mode 1 if rho > 0,
 * 2 if rho < 0, else 0; rho_f32 = float32(rho); drain_f32 =
 * float32(drain_fraction * -rho); the rest are np.float32(PhysicsParams.x). */
typedef struct evo_scalars {
  int32_t rho_mode;
  float rho_f32;
  float drain_f32;
  float invest_rate;
  float liquidate_rate;
  float invest_efficiency;
  float liquidate_efficiency;
  float explore_fraction;
  float upkeep;
  float decay_on_starvation;
  float death_threshold;
} evo_scalars;

typedef struct evo_ctx evo_ctx;

/* Context lifetime.  Replaces create_substrate + the pool's dense-param cache
 * (substrate.py:111-123, neuroevo.py:415-441).  hidden = 0 selects the direct
 * 45->13 controller (BASELINE extension), hidden >= 1 the reference
 * 45->hidden(tanh)->13 DenseParams net (hypernet.py:77-84, 233-252). */
EVO_API int evo_create(evo_ctx** out, int width, int height, int capacity, int hidden, int device);
/* Row strip [row0, row0+height) of a torus with height_global rows (multi-GPU,
 * SURVEY.md §8e).  Ghost rows are filled by the caller's halo exchange. */
EVO_API int evo_create_strip(evo_ctx** out, int width, int height, int64_t row0, int height_global,
                             int capacity, int hidden, int device);
EVO_API int evo_destroy(evo_ctx* ctx);
EVO_API const char* evo_last_error(void);
EVO_API int evo_version(void);

/* Front-buffer transfer (engine hooks / server brush read and write the front,
 * substrate.py:86-108, server.py:204-226).  Pointers are host memory; pinned
 * memory makes the copies asynchronous on `stream`. communication is (3,H,W). */
EVO_API int evo_upload_planes(evo_ctx* ctx, const float* energy, const float* infra, const float* comm,
                              const int32_t* genome, const uint8_t* rotation, void* stream);
EVO_API int evo_download_planes(evo_ctx* ctx, float* energy, float* infra, float* comm, int32_t* genome,
                                uint8_t* rotation, void* stream);

/* Per-slot controller parameters (DenseParams, hypernet.py:77-84), slots
 * [slot0, slot0+n).  hidden >= 1: w1 (n,hidden,45), b1 (n,hidden), w2
 * (n,13,hidden), b2 (n,13).  hidden == 0: w1/b1 ignored (may be NULL),
 * w2 (n,13,45), b2 (n,13). */
EVO_API int evo_set_params(evo_ctx* ctx, int slot0, int n, const float* w1, const float* b1, const float* w2,
                           const float* b2);
/* Inverse of evo_set_params: read slots [slot0, slot0+n) back in the same
 * reference layouts (used after evo_express_cppn to sync the host pool's
 * cached DenseParams, neuroevo.py:476). */
EVO_API int evo_get_params(evo_ctx* ctx, int slot0, int n, float* w1, float* b1, float* w2, float* b2);
/* Slot liveness (GenomePool slot states: 0 free, 1 live, 2 dead) and peak
 * populations, for the device census (neuroevo.py:521-542). */
EVO_API int evo_set_slots(evo_ctx* ctx, const int8_t* state, const int32_t* peak);
/* Optional per-cell energy source map (PhysicsParams.energy_source_map,
 * physics.py:69, 190-191); NULL restores the uniform default. */
EVO_API int evo_set_source_map(evo_ctx* ctx, const float* map);

/* One full step t -> t+1 (engine.py:233-248 without host radiation):
 * sense + net + energy + invest/liquidate + comm + explore proposal (pass 1),
 * explore resolve + adoption + census (pass 2), front/back swap. */
EVO_API int evo_step(evo_ctx* ctx, const evo_scalars* s, int64_t t, int phases, int flags, void* stream);
/* One step of a HOST-resident state, the drop-in for engine.step on a
 * SimState whose planes live in host memory (engine.py:233-248 on the
 * reference's numpy double buffer, substrate.py:52-110): uploads the front planes
 * (E, I, C as (3,H,W), genome_index, rotation), steps, and writes the new
 * planes to the *_out arrays, pipelined over `bands` row bands (0 = auto) so
 * the host->device copy, the two passes and the device->host copy overlap.
 * Genome / rotation ranges are checked on the device (EVO_EINVAL, outputs
 * undefined, device state not advanced).  Optional outputs: the census counts
 * (capacity int32; not with EVO_F_NO_CENSUS) and {adoptions, extinctions}.
 * Flags: 0 or EVO_F_RECORD_EVENTS | EVO_F_NO_CENSUS (host radiation).  The
 * call returns once the outputs are written; `stream` orders it after prior
 * work.  Host planes should be page-locked (evo_host_register) for DMA. */
EVO_API int evo_step_host(evo_ctx* ctx, const evo_scalars* s, int64_t t, int flags, const float* E, const float* I,
                          const float* C, const int32_t* gi, const uint8_t* rot, float* E_out, float* I_out,
                          float* C_out, int32_t* gi_out, uint8_t* rot_out, int32_t* counts, int64_t* stats,
                          int bands, void* stream);
/* RGBA frame of the device front buffer (substrate.py:147-165 render_rgb):
 * rgba = H*W*4 bytes, row-major; bit-identical to the reference's numpy
 * frame; moves 4 B/cell to the host instead of the 25 B/cell planes. */
EVO_API int evo_render_rgb(evo_ctx* ctx, double norm_energy, double norm_infrastructure, uint8_t* rgba,
                           void* stream);
/* Multi-scale complexity inputs of one front plane (metrics.py:57-103
 * msc_of_substrate; plane 0 energy, 1 infrastructure, 2..4 communication):
 * the centre power-of-two crop's block-mean pyramid and its overlaps as
 * correctly rounded exact sums, squares[k] = fsum over scale k of f_k^2 and
 * cross[k] = fsum of f_k * f_{k+1} (distinct products, k = 0..k_max); the
 * reference's overlap is ldexp(sum, 2k) / side^2.  n_scales <= 0: all
 * scales.  squares needs 32 entries, cross 31. */
EVO_API int evo_msc(evo_ctx* ctx, int plane, int n_scales, double* squares, double* cross, int* side, int* k_max);
/* float64 totals of the front energy / infrastructure planes in numpy's
 * summation order (metrics.py:200-213 census: plane.sum(dtype=float64)). */
EVO_API int evo_plane_sums(evo_ctx* ctx, double* energy, double* infrastructure);
/* Per-step device timing of evo_step / evo_run (bench.py's roofline split):
 * with profiling enabled every step records three events on its stream -
 * start, between pass 1 and pass 2, end.  evo_profile_read waits for the
 * recorded steps, returns the summed milliseconds of the two passes and the
 * number of steps, and clears the record.  No reference counterpart
 * (engine.py:233-248 times nothing); measurement only. */
EVO_API int evo_profile(evo_ctx* ctx, int enable);
EVO_API int evo_profile_read(evo_ctx* ctx, double* pass1_ms, double* pass2_ms, int* steps);

/* k consecutive steps t0..t0+k-1 with per-step scalars s[0..k-1]. */
EVO_API int evo_run(evo_ctx* ctx, const evo_scalars* s, int64_t t0, int k, void* stream);
/* The two launches of a step, for halo exchange between them (multi-GPU) and
 * for per-kernel timing.  evo_swap publishes the back buffer. */
EVO_API int evo_pass1(evo_ctx* ctx, const evo_scalars* s, int64_t t, int phases, int flags, void* stream);
EVO_API int evo_pass2(evo_ctx* ctx, int64_t t, int flags, void* stream);
EVO_API int evo_census_finish(evo_ctx* ctx, int64_t t, void* stream);
EVO_API int evo_swap(evo_ctx* ctx);
/* Single-GPU ghost-row refresh after a host upload (rows wrap on the torus). */
EVO_API int evo_refresh_ghosts(evo_ctx* ctx, void* stream);
EVO_API int evo_sync(evo_ctx* ctx);

/* Parity-mode ActionField transfer (physics.py:97-119): n listed cells
 * (linear indices, local to the strip) and their (n,13) actuator rows in
 * column order invest, liquidate, comm x3, explore x8 (engine.py:224-230). */
EVO_API int evo_set_actions(evo_ctx* ctx, const int64_t* cells, int64_t n, const float* acts);
/* Computed actions of the last EVO_F_EXPORT_ACTIONS step for every cell
 * occupied at sensing time, ascending index: cells (n), acts (n,13). */
EVO_API int evo_get_actions(evo_ctx* ctx, int64_t capacity, int64_t* cells, float* acts, int64_t* n);

/* Census of the last step: counts (capacity), slot state (0/1/2), death step
 * (-1 = alive), peak population.  Any pointer may be NULL. */
EVO_API int evo_read_census(evo_ctx* ctx, int32_t* counts, int8_t* state, int64_t* death_step, int32_t* peak);
/* Census counts accumulated by an EVO_F_NO_CENSUS step (per slot, the
 * genome plane before host radiation), copied out and cleared; the slot
 * table is left to the caller (host census after radiation, then
 * evo_set_slots).  counts: capacity int32. */
EVO_API int evo_census_take(evo_ctx* ctx, int32_t* counts);
/* Last step's adoption count and newly dead slot count
 * (SimState.last_adoptions / last_extinctions, engine.py:247-248). */
EVO_API int evo_read_stats(evo_ctx* ctx, int64_t* adoptions, int64_t* extinctions);
/* AdoptionEvents of the last EVO_F_RECORD_EVENTS step, ascending target
 * (physics.py:134-175, 340-343). */
EVO_API int evo_read_events(evo_ctx* ctx, int64_t capacity, int64_t* target, int64_t* source, int32_t* winner,
                            int32_t* defender, int64_t* direction, float* quantity, int64_t* m);
/* Patch genome slots on the device front buffer after host radiation
 * (physics.py:389-392): n cells (local linear index) get slot values. */
EVO_API int evo_patch_genomes(evo_ctx* ctx, const int64_t* cells, const int32_t* slots, int64_t n);

/* Batched CPPN expression: replaces the per-admission host call
 * hypernet.generate_network(genome, layout, tau, w_max) (hypernet.py:183-220,
 * invoked through GenomePool.admit's net_factory, neuroevo.py:476) for n
 * genomes at once, writing the dense tables of their pool slots on the
 * device (the layouts evo_set_params fills).  hidden == 0 substrates get the
 * direct 45->13 block (input -> actuator queries, biases from the bias
 * signal).  Programs come from paper_2406_09654_b200.neat.compile_programs:
 *   node_off [n+1]; nodes [node_off[n]][4] = {act (0 sine, 1 gaussian,
 *   2 sigmoid, 3 tanh, 4 identity, 5 abs; -1 input), input position | -1,
 *   edge begin, edge end}; edge_src (node position within the genome) and
 *   edge_w (float64) per enabled edge in connection-list order; outs [n][2]
 *   (weight-signal, bias-signal node positions); coords = neuron layout
 *   (45 inputs, hidden, 13 actuators) x (u, v) as make_layout builds it
 *   (hypernet.py:64-74).  All host pointers.  tau in [0, 1) and w_max > 0
 *   as hypernet.py:195-198 requires (else EVO_EINVAL). */
EVO_API int evo_express_cppn(evo_ctx* ctx, int n, const int32_t* slots, const int32_t* node_off,
                             const int32_t* nodes, const int32_t* edge_src, const double* edge_w,
                             const int32_t* outs, const double* coords, double tau, double w_max,
                             void* stream);

/* Field radiation (BASELINE config 3 extension).
 * evo_select_cells: every occupied cell of the front genome plane, in
 * ascending index order, takes the next double of the host Philox stream
 * whose 128-bit key is (key_hi:key_lo) - NumPy's Philox4x64-10, i.e.
 * np.random.Generator(np.random.Philox(key=k)).random(n_occupied) with k the
 * rng.stream(seed, t, "field_radiation") key (rng.py:19-33) - and is
 * selected iff u < p.  The selection stays on the device; parent_counts
 * (capacity, may be NULL) receives the number of selected cells per slot.
 * evo_remap_selected then moves each selected cell from slot g to
 * slot_map[g] (-1 keeps it), e.g. to the children the host admitted.
 * evo_read_selected copies the selected cells (ascending) for inspection. */
EVO_API int evo_select_cells(evo_ctx* ctx, uint64_t key_lo, uint64_t key_hi, double p, int32_t* parent_counts,
                             int64_t* n_selected);
/* Row strips: the strip's r-th occupied cell takes draw first_draw + r (the
 * occupied cells of the strips above it, e.g. an exclusive scan of
 * evo_count_occupied over the ranks), so N strips select exactly the cells
 * one context holding the whole torus would. */
EVO_API int evo_count_occupied(evo_ctx* ctx, int64_t* n_occupied);
EVO_API int evo_select_cells_at(evo_ctx* ctx, uint64_t key_lo, uint64_t key_hi, double p, int64_t first_draw,
                                int32_t* parent_counts, int64_t* n_selected);
EVO_API int evo_read_selected(evo_ctx* ctx, int64_t capacity, int64_t* cells, int64_t* n);
EVO_API int evo_remap_selected(evo_ctx* ctx, const int32_t* slot_map);

/* Host NEAT for the radiation feed (north_star (6): mutation stays on the
 * host), native: `mutate` of the reference (neuroevo.py:233-299) for n
 * genomes in order, each on its own NumPy Philox4x64-10 stream (keys: 2n
 * words, low first, = rng.stream(...) keys, rng.py:19-33), with NumPy's
 * exact random / uniform / normal (ziggurat) / integers draws; the shared
 * innovation counter (counter[0] next innovation, counter[1] next node id,
 * in/out) is consumed genome by genome as the reference's loop would.
 * Genomes are flat arrays: nodes [node_off[g], node_off[g+1]) with id, role
 * (0 input, 1 hidden, 2 output) and activation code (evo_express_cppn's);
 * connections [conn_off[g], conn_off[g+1]) with innovation, src, dst,
 * weight, enabled.  rates = {weight_reset_prob, weight_perturb_prob,
 * weight_perturb_sigma, add_connection_prob, add_node_prob,
 * toggle_enable_prob}.  Outputs in the same form; capacity: + 1 node and
 * + 3 connections per genome.  Host-only (no device involved). */
EVO_API int evo_neat_mutate(int n, const uint64_t* keys, const double* rates, int64_t* counter,
                            const int32_t* node_off, const int64_t* node_id, const int8_t* node_role,
                            const int8_t* node_act, const int32_t* conn_off, const int64_t* c_innov,
                            const int64_t* c_src, const int64_t* c_dst, const double* c_w, const uint8_t* c_en,
                            int32_t* o_node_off, int64_t* o_node_id, int8_t* o_node_role, int8_t* o_node_act,
                            int32_t* o_conn_off, int64_t* o_innov, int64_t* o_src, int64_t* o_dst, double* o_w,
                            uint8_t* o_en);
/* evo_neat_mutate with the numbering deferred: the same draws, but the k-th
 * new connection of a genome gets innovation -1 - k and its new node (at
 * most one) the id EVO_NEAT_DEFERRED_NODE (above every real id, so program
 * order is unaffected); no counter is read or consumed.  The caller numbers
 * the genomes it admits, in order, from the shared counter afterwards
 * (paper_2406_09654_b200.neat.number_deferred) - equal to evo_neat_mutate
 * over the admitted genomes alone.  Lets the host draws of a radiation
 * event run while the step before it is still on the device. */
#define EVO_NEAT_DEFERRED_NODE INT64_MAX
EVO_API int evo_neat_mutate_deferred(int n, const uint64_t* keys, const double* rates, const int32_t* node_off,
                                     const int64_t* node_id, const int8_t* node_role, const int8_t* node_act,
                                     const int32_t* conn_off, const int64_t* c_innov, const int64_t* c_src,
                                     const int64_t* c_dst, const double* c_w, const uint8_t* c_en,
                                     int32_t* o_node_off, int64_t* o_node_id, int8_t* o_node_role,
                                     int8_t* o_node_act, int32_t* o_conn_off, int64_t* o_innov, int64_t* o_src,
                                     int64_t* o_dst, double* o_w, uint8_t* o_en);
/* The evo_express_cppn program arrays of n flat genomes (hypernet.py:100-155
 * order; paper_2406_09654_b200.neat.compile_programs layout): prog_off
 * [n+1], nodes_out [total nodes][4], edge_src / edge_w [total enabled
 * connections], outs [n][2].  Host-only. */
EVO_API int evo_neat_compile(int n, const int32_t* node_off, const int64_t* node_id, const int8_t* node_role,
                             const int8_t* node_act, const int32_t* conn_off, const int64_t* c_src,
                             const int64_t* c_dst, const double* c_w, const uint8_t* c_en, int32_t* prog_off,
                             int32_t* nodes_out, int32_t* edge_src, double* edge_w, int32_t* outs);
EVO_API const char* evo_neat_last_error(void);

/* Page-lock caller-owned host planes (cudaHostRegister) so that the
 * upload/download copies of evo_upload_planes / evo_download_planes run as
 * direct DMA at full link bandwidth; the substrate's front/back arrays live
 * for the whole run (substrate.py:86-108), so the engine registers them once.
 * Registering an already registered range is not an error. */
EVO_API int evo_host_register(void* ptr, int64_t bytes);
EVO_API int evo_host_unregister(void* ptr);

/* Strip halo staging in one launch each (multi-GPU).
 * which 0: the five sensed front planes (E, I, C0..C2) before pass 1;
 * which 1: the pass-1 outputs pass 2 reads (post-death genome, shipped
 * quantity, proposal byte widened to 32 bits).  Device buffers of
 * 2 x row_words 32-bit words: pack writes [first row | last row], unpack
 * reads [ghost row above | ghost row below]; the caller moves them between
 * ranks (NCCL send/recv). */
EVO_API int evo_halo_row_words(evo_ctx* ctx, int which, int64_t* row_words);
EVO_API int evo_halo_pack(evo_ctx* ctx, int which, void* send, void* stream);
EVO_API int evo_halo_unpack(evo_ctx* ctx, int which, const void* recv, void* stream);

/* Device pointers of a plane (halo exchange / interop).  which: 0 energy,
 * 1 infra, 2 comm (3 planes, stride = plane_stride), 3 genome, 4 rotation,
 * 5 mid infra, 6 mid genome, 7 mid proposal byte, 8 mid quantity, 9 census
 * counts being accumulated (int32 [capacity]), 10 step stats (int64 [2]).
 * buffer: 0 front, 1 back (ignored for mid planes).  The pointer addresses
 * ghost row -1; row y lives at + (y+1)*W.  plane_stride counts elements. */
EVO_API int evo_plane_ptr(evo_ctx* ctx, int which, int buffer, void** ptr, int64_t* plane_stride);

/* Diagnostics: per-phase cycle sums of the hot pass-1 kernel, summed over
 * CTAs (0 bucketing, 1 controller, 2 physics tail, 3 halo commit, 4 setup);
 * non-zero only in a library built with -DEVO_PHASE_TIMING. */
EVO_API int evo_debug_phase_cycles(uint64_t* out8, int reset);
/* Test hook: the sigmoid's inline reciprocal (hypernet.py:246-251's 1 / (1 + exp(-z)), correctly rounded)
 * against __frcp_rn over every float in [1, 2^125); *mismatches must come back 0. */
EVO_API int evo_debug_rcp_check(uint64_t* mismatches);
/* Same for the tensor-core hidden-layer kernel (8 phases of its tile loop). */
EVO_API int evo_debug_hidden_cycles(uint64_t* out8, int reset);

/* 64-bit FNV-1a continuation over host bytes (engine.digest, engine.py:283-315):
 * *out = fold(h, data[0..n)).  Host code, no device involved. */
EVO_API int evo_fnv1a64(uint64_t h, const uint8_t* data, int64_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* EVOCA_B200_H */
