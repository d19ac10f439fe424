/*
 * synscale_b200.h — C ABI of the B200-native spiking-network step engine.
 *
 * This is the drop-in boundary for the reference's hot path, one
 * `Simulation::step()` of a clock-driven network (Poisson sources, conductance
 * LIF populations, dense and CRS synapse groups).  The reference has no FFI of
 * its own; its only boundary is the C++ API in
 *   /root/reference/proj/include/synscale/engine.hpp:75-104   (Simulation, run)
 *   /root/reference/proj/include/synscale/engine.hpp:59-67    (detect_nans, propagate)
 *   /root/reference/proj/include/synscale/network.hpp:14-144  (NetworkSpec, builders)
 *   /root/reference/proj/include/synscale/matrix.hpp:14-81    (connectivity)
 *   /root/reference/proj/include/synscale/occupancy.hpp:14-70 (occupancy model)
 * Every entry point below names the reference symbol it replaces.  The C++
 * facade in include/synscale/ (same names as the reference) sits on these.
 *
 * Conventions: plain pointers and sizes, no C++ or torch types; no exception
 * crosses this boundary.  Return codes: SSB_OK (0), SSB_ERR_INTERNAL (1, CUDA
 * or allocation failure), SSB_ERR_SPEC (2, the reference's SpecError: bad
 * spec, misuse, out-of-range argument).  The CLI mapping of the reference
 * (SpecError -> exit 2, anything else -> exit 1; tools/main.cpp:403-412) is
 * kept numerically.  Functions taking `char* err, size_t errlen` write the
 * message of a failure there (NUL-terminated, truncated); the last error of
 * a handle is also available from ssb_last_error().
 *
 * Threading: one ssb_sim per host thread; handles are independent (each owns
 * its CUDA stream and buffers), so concurrent sweeps are safe
 * (reference: src/calibration.cpp:76-84 runs one Simulation per thread).
 */
#ifndef SYNSCALE_B200_H
#define SYNSCALE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SSB_API __attribute__((visibility("default")))
#else
#define SSB_API
#endif

#define SSB_OK 0
#define SSB_ERR_INTERNAL 1
#define SSB_ERR_SPEC 2

/* ModelKind (network.hpp:14) */
enum { SSB_MODEL_IZHIKEVICH = 0, SSB_MODEL_POISSON = 1, SSB_MODEL_CONDLIF = 2,
       SSB_MODEL_TRAUBMILES = 3 /* extension: Traub-Miles HH (F1) */ };
/* SynapseSign (network.hpp:15) */
enum { SSB_SIGN_EXC = 0, SSB_SIGN_INH = 1 };
/* StorageKind (network.hpp:16) */
enum { SSB_STORAGE_DENSE = 0, SSB_STORAGE_SPARSE = 1 };
/* Synapse plasticity (extension F2: the reference has no
 * learning).  STDP = pair-based spike-timing-dependent
 * plasticity with exponential traces on a dense all-to-all excitatory group;
 * the rule is stated in DESIGN.md §1 (row A22). */
enum { SSB_PLASTICITY_NONE = 0, SSB_PLASTICITY_STDP = 1 };
/* StorageMode (engine.hpp:18) */
enum { SSB_MODE_FROM_SPEC = 0, SSB_MODE_FORCE_DENSE = 1, SSB_MODE_FORCE_SPARSE = 2,
       SSB_MODE_AUTO = 3 /* extension: dense iff outDegree / nPost >= ssb_auto_dense_threshold() */ };
/* WeightDist::Kind (matrix.hpp:15-16) */
enum { SSB_WEIGHT_CONSTANT = 0, SSB_WEIGHT_UNIFORM = 1 };
/* PopulationState fields (engine.hpp:48-54) */
enum {
    SSB_FIELD_V = 0,       /* float[n]   */
    SSB_FIELD_U = 1,       /* float[n]   Izhikevich only */
    SSB_FIELD_GEXC = 2,    /* float[n]   */
    SSB_FIELD_GINH = 3,    /* float[n]   */
    SSB_FIELD_EXCIN = 4,   /* float[n]   accumulator for the next step */
    SSB_FIELD_INHIN = 5,   /* float[n]   accumulator for the next step */
    SSB_FIELD_NANFLAG = 6, /* uint8[n]   sticky non-finite flag */
    SSB_FIELD_FLAGGED = 7, /* int64[1]   neurons ever flagged */
    SSB_FIELD_M = 8,       /* float[n]   Traub-Miles gating variables (extension) */
    SSB_FIELD_H = 9,
    SSB_FIELD_N = 10
};

/* NeuronPopulation (network.hpp:47-53) with its parameter variant flattened. */
typedef struct ssb_pop_desc {
    const char* name;
    int32_t size;
    int32_t model; /* SSB_MODEL_* */
    uint64_t seed; /* entity seed */
    /* PoissonParams (network.hpp:29-31) */
    double rate_hz;
    /* CondLifParams (network.hpp:37-45) */
    double tau_m_ms, e_leak_mv, v_thresh_mv, v_reset_mv, e_exc_mv, e_inh_mv, tau_syn_ms;
    /* IzhikevichParams (network.hpp:21-26): per-neuron arrays of `size` doubles */
    const double *izh_a, *izh_b, *izh_c, *izh_d, *izh_noise, *izh_bias;
    /* TraubMilesParams (extension, F1); the synapses use e_exc_mv, e_inh_mv and
     * tau_syn_ms above */
    double hh_gna, hh_ena, hh_gk, hh_ek, hh_gl, hh_el, hh_c;
    int32_t hh_substeps;
} ssb_pop_desc;

/* SynapseGroupSpec (network.hpp:59-70) with WeightDist (matrix.hpp:14-24). */
typedef struct ssb_group_desc {
    const char* name;
    const char* pre;
    const char* post;
    int32_t sign; /* SSB_SIGN_* */
    int32_t out_degree;
    int32_t weight_kind; /* SSB_WEIGHT_* */
    double weight_lo, weight_hi, weight_value;
    double g_scale;
    int32_t storage; /* SSB_STORAGE_* */
    int32_t pre_offset;
    int32_t pre_count; /* -1 = rest of the population */
    /* extension F2 (zero = static, as in the reference): SSB_PLASTICITY_* and
     * the STDP constants (cast to fp32; trace decays float(exp(-dt/tau))) */
    int32_t plasticity;
    double stdp_a_plus, stdp_a_minus, stdp_tau_plus_ms, stdp_tau_minus_ms, stdp_w_max;
} ssb_group_desc;

/* NetworkSpec (network.hpp:72-80). */
typedef struct ssb_net_desc {
    int32_t n_pops;
    const ssb_pop_desc* pops;
    int32_t n_groups;
    const ssb_group_desc* groups;
    double dt_ms;
    double duration_ms;
    uint64_t global_seed;
} ssb_net_desc;

/* MBodyBuildOptions (network.hpp:130-140); lif uses the CondLif fields. */
typedef struct ssb_mbody_opts {
    double dt_ms, duration_ms, pn_rate_hz, pn_kc_out_fraction;
    double tau_m_ms, e_leak_mv, v_thresh_mv, v_reset_mv, e_exc_mv, e_inh_mv, tau_syn_ms;
    double pn_kc_weight_hi, pn_lhi_weight, lhi_kc_weight, kc_dn_weight;
    /* extension: KC model (SSB_MODEL_CONDLIF or SSB_MODEL_TRAUBMILES) and the HH
     * parameters (synapses: e_exc_mv / e_inh_mv above, kc_tau_syn_ms) */
    int32_t kc_model;
    double hh_gna, hh_ena, hh_gk, hh_ek, hh_gl, hh_el, hh_c, hh_e_inh_mv, kc_tau_syn_ms;
    int32_t hh_substeps;
} ssb_mbody_opts;

/* IzhBuildOptions (network.hpp:105-114). */
typedef struct ssb_izh_opts {
    double dt_ms, duration_ms, noise_exc, noise_inh, exc_weight_hi, inh_weight_hi, bias_current;
    int32_t storage;
} ssb_izh_opts;

/* B200 engine knobs (no reference counterpart; zero = default). */
typedef struct ssb_engine_opts {
    int32_t device;              /* CUDA device ordinal */
    int32_t window;              /* max steps fused per launch window (default 64) */
    int32_t block_size;          /* neuron-update block size; 0 = occupancy policy */
    int32_t block_policy;        /* 0 = occupancy model + SM fill, 1 = paper model only */
    int32_t use_graphs;          /* 0 = default (on), 1 = on, -1 = off */
    int32_t heavy_pre_threshold; /* groups with >= this many pre rows use the buffered path */
    int64_t raster_capacity;     /* raster bitmask words kept on device between host flushes
                                  * (at least two graph launches of windows) */
    int32_t profile;             /* 1 = time every launch with CUDA events */
    int32_t force_step_mode;     /* 1 = never fuse steps (window forced to 1) */
    /* multi-GPU: one process per GPU, rank of world_size, NCCL
     * communicator from comm_id (ssb_comm_unique_id on rank 0, broadcast by
     * the caller).  CondLif populations of >= shard_min_size neurons are split
     * by neuron ranges; each window's spike bitmasks are all-gathered.
     * virtual_world > 1 instead runs that many shards in this process on one
     * GPU (exchange by device copies; for testing the split path). */
    int32_t rank;
    int32_t world_size;          /* 0 or 1 = single GPU */
    int32_t virtual_world;
    int32_t shard_min_size;      /* 0 = default (64) */
    int32_t has_comm_id;
    uint8_t comm_id[128];
    /* pinned host memory (MB) allocated at creation for raster drains: a
     * drain that fits copies straight into it at PCIe speed (0 = none:
     * drains go through pinned staging into pageable memory) */
    int32_t raster_pinned_mb;
    /* split runs (world_size > 1, not virtual_world): 1 = each rank records
     * only its own neurons of split populations, and rank 0 alone the whole
     * (replicated) ones; the global raster is the union over ranks (spike
     * counts likewise sum over ranks; ssb_finish's rates are already the
     * global ones: it all-reduces the per-population totals).  0 = every
     * rank records the global raster. */
    int32_t raster_local;
} ssb_engine_opts;

/* Result summary (RunResult, engine.hpp:35-42). */
typedef struct ssb_run_summary {
    int64_t steps;
    int64_t steps_done;
    double duration_ms;
    int64_t sum_nans;
    int64_t n_events;
    double wall_time_ms;
} ssb_run_summary;

/* Occupancy model (occupancy.hpp:14-48). */
typedef struct ssb_device_spec {
    char name[32];
    int64_t warp_size, max_warps_per_sm, max_blocks_per_sm, max_threads_per_block;
    int64_t shared_mem_per_sm, regs_per_sm, reg_alloc_unit, shared_alloc_unit;
} ssb_device_spec;

typedef struct ssb_occupancy_result {
    int64_t warps_per_block, limit_warps, limit_blocks, limit_shared, limit_regs;
    int64_t active_blocks, active_warps;
    double occupancy;
    int32_t limiter_mask; /* bit0 warps, bit1 blocks, bit2 shared, bit3 registers */
} ssb_occupancy_result;

/* Per-kernel launch statistics (profile mode). */
typedef struct ssb_kernel_stat {
    char name[48];
    int64_t launches;
    double total_ms;
    double bytes; /* algorithmic bytes summed over launches */
} ssb_kernel_stat;

typedef struct ssb_sim ssb_sim;

/* ---- library ------------------------------------------------------------ */
SSB_API const char* ssb_version(void);
/* StorageMode Auto's density threshold (extension; env SSB_AUTO_DENSITY). */
SSB_API double ssb_auto_dense_threshold(void);
SSB_API int ssb_device_count(void);

/* ---- spec helpers (network.cpp) ------------------------------------------- */
/* validate (network.hpp:89-91): returns the number of violations; the
 * messages, one per line "field: message", go to `out`. */
SSB_API int ssb_validate(const ssb_net_desc* net, char* out, size_t outlen);
/* build_mbody_net (network.cpp:286-362). The returned desc owns its memory;
 * release it with ssb_net_desc_free. gscales order: pn_kc, pn_lhi, lhi_kc, kc_dn. */
SSB_API int ssb_build_mbody(int32_t n_pn, int32_t n_lhi, int32_t n_kc, int32_t n_dn,
                            const double gscales[4], uint64_t seed, const ssb_mbody_opts* opts,
                            ssb_net_desc** out, char* err, size_t errlen);
/* build_izhikevich_net (network.cpp:198-284). */
SSB_API int ssb_build_izhikevich(int32_t n_neurons, int32_t n_conn, double exc_fraction,
                                 double g_scale, uint64_t seed, const ssb_izh_opts* opts,
                                 ssb_net_desc** out, char* err, size_t errlen);
SSB_API void ssb_net_desc_free(ssb_net_desc* net);
SSB_API void ssb_mbody_default_opts(ssb_mbody_opts* opts);
SSB_API void ssb_izh_default_opts(ssb_izh_opts* opts);
SSB_API void ssb_engine_default_opts(ssb_engine_opts* opts);

/* ---- RNG streams (random.hpp) --------------------------------------------- */
SSB_API uint64_t ssb_fnv1a64(const char* label);
SSB_API uint64_t ssb_splitmix64(uint64_t x);
SSB_API uint64_t ssb_derive_seed(uint64_t parent, const char* label); /* random.hpp:30-32 */
/* First n outputs of RandomStream(global, entity, label).next_u64 (random.hpp:40-46). */
SSB_API int ssb_stream_u64(uint64_t global_seed, uint64_t entity_seed, const char* label,
                           int64_t n, uint64_t* out);

/* ---- connectivity (matrix.cpp) -------------------------------------------- */
/* gen_fixed_outdegree (matrix.cpp:91-142): writes nPre*nPost floats. */
SSB_API int ssb_gen_fixed_outdegree(int32_t n_pre, int32_t n_post, int32_t k, int32_t weight_kind,
                                    double lo, double hi, double value, int32_t sign,
                                    uint64_t seed, float* out, char* err, size_t errlen);
/* Connectivity of group `group` exactly as Simulation's constructor builds it
 * (engine.cpp:214-244; host setup, no GPU needed).  Call with values == NULL
 * to get the sizes; *nnz is nPre*nPost for dense storage.  Sparse results
 * fill values (gValues), post_ind and row_start (n_pre + 1 entries). */
SSB_API int ssb_build_group(const ssb_net_desc* net, int32_t storage_mode, int32_t group,
                            int32_t* storage, int32_t* n_pre, int32_t* n_post, int64_t* nnz,
                            float* values, int32_t* post_ind, int64_t* row_start, int64_t cap,
                            char* err, size_t errlen);
SSB_API uint64_t ssb_mem_sparse_elements(uint64_t nnz, uint64_t n_post); /* matrix.cpp:176 */

/* ---- calibration sweep (calibration.cpp:16-86) ------------------------------ */
/* Runs n_cells independent networks (one sweep cell each, built by the caller
 * from its template) to their end on the GPU, `parallelism` at a time, and
 * records the target population's avgSpike and the run's sumNaNs per cell.  A
 * cell that fails gets failed[i] = 1, avg_spike NaN, sum_nans -1 and its error
 * text in errors + i * err_stride (may be NULL). */
SSB_API int ssb_sweep(const ssb_net_desc* const* cells, int32_t n_cells, int32_t storage_mode,
                      const char* target_population, int32_t parallelism,
                      const ssb_engine_opts* opts, double* avg_spike, int64_t* sum_nans,
                      int32_t* failed, char* errors, size_t err_stride, char* err, size_t errlen);

/* ---- multi-GPU decomposition (host, no GPU needed) ------------------------- */
/* Neuron ranges of a world of `world` ranks: bounds[p*(world+1) + r] = first
 * neuron of rank r in population p (r = world: the size), or -1 for every r
 * when population p is whole (replicated).  SpecError for recurrent nets. */
SSB_API int ssb_shard_plan(const ssb_net_desc* net, int32_t world, int32_t min_size,
                           int64_t* bounds, char* err, size_t errlen);
/* Group `group` as rank `rank` holds it (ssb_build_group of the column slice
 * of a split post population; n_post = the local column count). */
SSB_API int ssb_shard_group(const ssb_net_desc* net, int32_t storage_mode, int32_t group,
                            int32_t world, int32_t rank, int32_t min_size, int32_t* storage,
                            int32_t* n_pre, int32_t* n_post, int64_t* nnz, float* values,
                            int32_t* post_ind, int64_t* row_start, int64_t cap, char* err,
                            size_t errlen);
/* NCCL unique id for ssb_engine_opts.comm_id (loads libnccl; no GPU work). */
SSB_API int ssb_comm_unique_id(uint8_t* out128, char* err, size_t errlen);
/* Self-test of the exchange on one device: a one-rank communicator, the
 * all-gather and the sum the split engine issues (graph-captured and not). */
SSB_API int ssb_comm_selftest(int32_t device, char* err, size_t errlen);
SSB_API uint64_t ssb_mem_dense_elements(uint64_t n_pre, uint64_t n_post); /* matrix.cpp:180 */

/* ---- standalone device kernels -------------------------------------------- */
/* propagate(DenseMatrix) (engine.cpp:53-67) on host arrays; runs on the GPU. */
SSB_API int ssb_propagate_dense(const float* w, int32_t n_pre, int32_t n_post,
                                const int32_t* spikes, int64_t n_spikes, float* acc,
                                int64_t acc_len, char* err, size_t errlen);
/* propagate(CrsMatrix) (engine.cpp:69-80) on host arrays; runs on the GPU. */
SSB_API int ssb_propagate_crs(const float* g, const int32_t* post_ind, const int64_t* row_start,
                              int32_t n_pre, int32_t n_post, const int32_t* spikes,
                              int64_t n_spikes, float* acc, int64_t acc_len, char* err,
                              size_t errlen);
/* Device-pointer variants (all pointers are CUDA device memory; enqueued on
 * `stream`, a cudaStream_t or NULL). No argument checks beyond sizes. */
SSB_API int ssb_propagate_dense_dev(const float* w, int32_t n_pre, int32_t n_post,
                                    const int32_t* spikes, int32_t n_spikes, float* acc,
                                    void* stream);
/* `seg` is the post-tile segment table built by ssb_crs_segments_dev for `tile`. */
SSB_API int ssb_crs_segments_dev(const int32_t* post_ind, const int64_t* row_start,
                                 int32_t n_pre, int32_t n_post, int32_t tile, int32_t* seg,
                                 void* stream);
SSB_API int ssb_propagate_crs_dev(const float* g, const int32_t* post_ind,
                                  const int32_t* seg, int32_t tile, int32_t n_pre, int32_t n_post,
                                  const int32_t* spikes, int32_t n_spikes, float* acc,
                                  void* stream);
/* Column-sliced CRS (extension): the matrix re-laid as slices of 32 post
 * columns (entry k of column 32 s + l at slice_off[s] + 32 k + l: its pre row,
 * -1 for padding, and value; rows ascending within a column).  With rows /
 * vals NULL only *needed (entries incl. padding) and slice_off
 * [ceil(n_post / 32) + 1] are written.  Host arrays. */
SSB_API int ssb_crs_slices(const float* g, const int32_t* post_ind, const int64_t* row_start,
                           int32_t n_pre, int32_t n_post, int64_t* slice_off, int32_t* rows,
                           float* vals, int64_t cap, int64_t* needed, char* err, size_t errlen);
/* propagate(CrsMatrix) over column slices (device pointers): bit-identical to
 * the reference for a spike list in ascending order without repeats (the
 * engine's lists); coalesced loads at every density. */
SSB_API int ssb_propagate_crs_sliced_dev(const int32_t* rows, const float* vals,
                                         const int64_t* slice_off, int32_t n_pre, int32_t n_post,
                                         const int32_t* spikes, int32_t n_spikes, float* acc,
                                         void* stream);
/* detect_nans (engine.cpp:27-51) on host arrays; runs on the GPU. Pointers a
 * model does not use may be NULL. Returns newly flagged via *newly. */
SSB_API int ssb_detect_nans(int32_t model, const float* v, const float* u, const float* g_exc,
                            const float* g_inh, uint8_t* nan_flag, int64_t n, int64_t* flagged,
                            int64_t* newly, char* err, size_t errlen);

/* ---- simulation (engine.hpp:75-104) --------------------------------------- */
/* Simulation::Simulation(spec, mode) (engine.cpp:146-245). */
SSB_API int ssb_create(const ssb_net_desc* net, int32_t storage_mode, const ssb_engine_opts* opts,
                       ssb_sim** out, char* err, size_t errlen);
SSB_API void ssb_destroy(ssb_sim* sim);
SSB_API const char* ssb_last_error(const ssb_sim* sim);
/* Simulation::step() repeated n times (engine.cpp:316-356). Fails with
 * SSB_ERR_SPEC when finished or when fewer than n steps remain. */
SSB_API int ssb_step(ssb_sim* sim, int64_t n);
SSB_API int64_t ssb_steps_total(const ssb_sim* sim);
/* Ranks the network is split over and this process's range of population
 * `pop`: neurons [lo, lo + n_local) of n_global. */
SSB_API int32_t ssb_world(const ssb_sim* sim);
SSB_API int ssb_shard_range(const ssb_sim* sim, int32_t pop, int64_t* lo, int64_t* n_local,
                            int64_t* n_global);
SSB_API int64_t ssb_steps_done(const ssb_sim* sim);
/* Waits for all queued work of the handle. */
SSB_API int ssb_sync(ssb_sim* sim);
/* population_state (engine.hpp:84-85): copy a field out of / into the device
 * state. `pop` is the spec index; n is the element count (1 for FLAGGED). */
SSB_API int ssb_pull_state(ssb_sim* sim, int32_t pop, int32_t field, void* dst, int64_t n);
SSB_API int ssb_push_state(ssb_sim* sim, int32_t pop, int32_t field, const void* src, int64_t n);
/* group_dense / group_sparse (engine.hpp:88-89): storage actually used after
 * gScale and StorageMode. *storage is SSB_STORAGE_*. */
SSB_API int ssb_group_info(const ssb_sim* sim, int32_t group, int32_t* storage, int32_t* n_pre,
                           int32_t* n_post, int64_t* nnz);
SSB_API int ssb_group_dense(const ssb_sim* sim, int32_t group, float* w, int64_t n);
/* Extension F2: the dense group's weights as they are now (a plastic group's
 * learned weights, read from the device after the steps so far; a static
 * group's are ssb_group_dense's).  n = n_pre * n_post. */
SSB_API int ssb_group_weights(ssb_sim* sim, int32_t group, float* w, int64_t n);
SSB_API int ssb_group_sparse(const ssb_sim* sim, int32_t group, float* g, int32_t* post_ind,
                             int64_t* row_start);
/* Simulation::finish() (engine.cpp:385-401): runs the remaining steps and
 * collects results. Callable once. */
SSB_API int ssb_finish(ssb_sim* sim, ssb_run_summary* out);
/* Results after finish: rates (avgSpike, per spec population order) and the
 * raster ordered by (step, population, neuron) (engine.hpp:26-33). */
SSB_API int ssb_result_rates(const ssb_sim* sim, double* rates, int32_t n_pops);
SSB_API int64_t ssb_result_n_events(const ssb_sim* sim);
SSB_API int ssb_result_raster(const ssb_sim* sim, int64_t* step, int32_t* pop, int32_t* neuron,
                              int64_t cap);
/* Compact raster: per-(step, population) spike counts [steps*n_pops] and the
 * neuron ids in raster order. Valid after finish, or after ssb_raster_flush. */
SSB_API int ssb_result_counts(const ssb_sim* sim, int32_t* counts, int64_t n);
SSB_API int ssb_result_neurons(const ssb_sim* sim, int32_t* neuron, int64_t cap);
/* Spike counts so far per population (device-side totals; syncs). */
SSB_API int ssb_spike_counts(ssb_sim* sim, int64_t* counts, int32_t n_pops);
/* Drops every recorded event (counts and ids) held so far; bench helper for
 * long runs whose raster is not wanted. */
SSB_API int ssb_raster_discard(ssb_sim* sim);
/* Waits for the steps issued so far and moves every event recorded so far into
 * host memory (the engine otherwise drains in the background); returns the
 * number of events held on the host in *n_events. */
SSB_API int ssb_raster_drain(ssb_sim* sim, int64_t* n_events);
/* Starts moving the events recorded so far to host memory in the background
 * and returns at once (steps issued next overlap the copy); a later
 * ssb_raster_drain or ssb_finish waits for it. */
SSB_API int ssb_raster_drain_async(ssb_sim* sim);

/* ---- introspection / measurement ------------------------------------------- */
SSB_API void* ssb_stream(ssb_sim* sim); /* the handle's cudaStream_t */
SSB_API int32_t ssb_window(const ssb_sim* sim); /* effective steps per launch window */
SSB_API int32_t ssb_block_size(const ssb_sim* sim, int32_t pop);
/* blocks of the population's update kernel (0: no update kernel) */
SSB_API int32_t ssb_grid_size(const ssb_sim* sim, int32_t pop);
SSB_API int32_t ssb_n_kernel_stats(const ssb_sim* sim);
SSB_API int ssb_kernel_stats(ssb_sim* sim, ssb_kernel_stat* out, int32_t n);
SSB_API int ssb_kernel_stats_reset(ssb_sim* sim);
/* Device bytes held by the handle. */
SSB_API int64_t ssb_device_bytes(const ssb_sim* sim);
/* Kernel launches issued by ssb_step so far (graph nodes count individually). */
SSB_API int64_t ssb_kernel_launches(const ssb_sim* sim);

/* ---- occupancy model (occupancy.cpp) -------------------------------------- */
SSB_API int ssb_device_preset(const char* name, ssb_device_spec* out, char* err, size_t errlen);
/* Preset names, comma separated ("cc20,cc30,cc50,sm100"). */
SSB_API const char* ssb_device_preset_names(void);
/* Fills an ssb_device_spec from cudaGetDeviceProperties of `device`. */
SSB_API int ssb_device_query(int32_t device, ssb_device_spec* out, char* err, size_t errlen);
SSB_API int ssb_occupancy(const ssb_device_spec* dev, int64_t threads_per_block,
                          int64_t regs_per_thread, int64_t shared_per_block,
                          ssb_occupancy_result* out, char* err, size_t errlen);
SSB_API int ssb_recommend_block_size(const ssb_device_spec* dev, int64_t regs_per_thread,
                                     int64_t shared_per_block, int64_t* block_size,
                                     ssb_occupancy_result* out, char* err, size_t errlen);
/* Registers / static shared memory of the engine's kernels (cudaFuncGetAttributes). */
SSB_API int ssb_kernel_attributes(const char* kernel, int32_t* regs, int32_t* shared_bytes,
                                  int32_t* max_threads);

#ifdef __cplusplus
}
#endif

#endif /* SYNSCALE_B200_H */
