/*
 * sparse2d_b200.h -- C ABI of the B200-native 2D-sparse-parallel embedding
 * step (libsparse2d_b200.so).  Plain pointers and sizes only; no torch or
 * CUDA types cross this boundary (streams are passed as void*).
 *
 * Every entry point returns an int status (S2D_OK = 0) and leaves a message
 * for s2d_last_error() (thread-local) on failure.  The status codes map onto
 * the exceptions the reference library throws:
 *   S2D_EINVAL     std::invalid_argument   (bad config, N x N mismatch, zero batch)
 *   S2D_ERANGE     std::out_of_range       (id outside every shard, embedding.cpp:61-63)
 *   S2D_ENONFINITE std::invalid_argument   ("nonfinite row gradient", optimizer.cpp:69-72)
 *   S2D_ERUNTIME   std::runtime_error      (checkpoint IO, embedding.cpp:133-219)
 *   S2D_ECUDA / S2D_ENCCL                  device / collective failures (new)
 *
 * Each declaration names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 */
#ifndef SPARSE2D_B200_H
#define SPARSE2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2D_OK 0
#define S2D_EINVAL 1
#define S2D_ERANGE 2
#define S2D_ENONFINITE 3
#define S2D_ERUNTIME 4
#define S2D_ECUDA 5
#define S2D_ENCCL 6

/* ShardingStrategy (include/sparse2d/planner.hpp:29) */
#define S2D_TABLE_WISE 0
#define S2D_ROW_WISE 1
/* OptimizerVariant (include/sparse2d/optimizer.hpp:10) */
#define S2D_ROWWISE_ADAGRAD 0
#define S2D_SGD 1
/* weight storage */
#define S2D_F32 0
#define S2D_BF16 1
/* where a buffer argument lives */
#define S2D_HOST 0
#define S2D_DEVICE 1

/* TableLoadProfile (include/sparse2d/planner.hpp:12-20) */
typedef struct {
  uint32_t table_id;
  uint64_t size_bytes;
  double expected_lookups_per_batch;
  uint64_t num_rows;
} s2d_table_load_profile;

/* PlanEntry (include/sparse2d/planner.hpp:22-27) */
typedef struct {
  uint32_t table_id;
  uint32_t row_lo;
  uint32_t row_hi; /* half-open */
  uint32_t local_rank;
} s2d_plan_entry;

/* OptimizerConfig (include/sparse2d/optimizer.hpp:15-22) */
typedef struct {
  double eta;
  double eps;
  double c;        /* moment scaling factor; c = 1 is plain row-wise AdaGrad */
  int32_t variant; /* S2D_ROWWISE_ADAGRAD | S2D_SGD */
} s2d_optimizer_config;

/* Topology (include/sparse2d/topology.hpp:13-26) */
typedef struct {
  uint32_t total_ranks;
  uint32_t groups;
  uint32_t ranks_per_group;
} s2d_topology;

/* pooling mode of a table (s2d_table_desc.pooling) */
#define S2D_POOL_SUM 0  /* the reference's pool_ids (embedding.cpp:39-92) */
#define S2D_POOL_MEAN 1 /* extension: out = f32((sum_o f64(partial_o)) * (1/L)); the
                           bag's gradient row is f32(f64(up) * (1/L)) */

/* One embedding table (FeatureSpec + EmbeddingTable shape, data.hpp:11-18,
 * embedding.hpp:12-23); per-table rows, dims and pooling are extensions. */
typedef struct {
  uint32_t table_id; /* must equal its index in the registered list */
  uint32_t rows;
  uint32_t dim;     /* multiple of 4, <= 512 (trainer.cpp:99 kMaxDim) */
  uint32_t pooling; /* S2D_POOL_SUM | S2D_POOL_MEAN */
} s2d_table_desc;

/* Per-step counters of the last step on this rank. */
typedef struct {
  uint64_t nnz_local;      /* ids in this rank's batch */
  uint64_t nnz_owned;      /* ids this rank served as owner */
  uint64_t entries_owned;  /* non-empty (bag, owner) pairs served (E) */
  uint64_t unique_rows;    /* rows updated (U) */
  uint64_t long_segments;  /* rows whose gradient was reduced in chunks */
  uint64_t dirty_rows;     /* rows averaged by the last replica sync */
  uint64_t a2a_bytes_sent; /* lookup+grad+id all-to-all bytes to other ranks */
  uint64_t a2a_bytes_recv;
  uint64_t sync_bytes;     /* replica-sync payload bytes sent */
  uint32_t error_flags;    /* device-side fault bits of the last step */
  uint32_t sync_mode;      /* last replica sync: 0 none, 1 pair snapshot exchange (M = 2), 2 slice push/mean/scatter, 3 NCCL all-gather */
  uint64_t ids_bytes_sent;    /* part of a2a_bytes_sent: lengths + ids (K1 permute) */
  uint64_t lookup_bytes_sent; /* part of a2a_bytes_sent: partials / pooled rows (K2) */
  uint64_t grad_bytes_sent;   /* part of a2a_bytes_sent: gradient rows (grad gather) */
  uint64_t host_wait_ns;      /* host time blocked on the device count read (N > 1), cumulative */
} s2d_step_stats;

const char* s2d_last_error(void);
const char* s2d_version(void);

/* ---- host-side planning (no GPU needed) --------------------------------- */

/* Topology(total, groups) ctor (src/topology.cpp:7-17). */
int s2d_topology_init(uint32_t total_ranks, uint32_t groups, s2d_topology* out);

/* plan_greedy (include/sparse2d/planner.hpp:47-48, src/planner.cpp:38-89).
 * Writes at most `cap` entries; *n_out = entry count. */
int s2d_plan_greedy(const s2d_table_load_profile* profiles, uint32_t n_profiles, uint32_t n,
                    int32_t strategy, s2d_plan_entry* out, uint32_t cap, uint32_t* n_out);

/* validate_plan (src/planner.cpp:91-123). */
int s2d_validate_plan(const s2d_plan_entry* plan, uint32_t n_entries, uint32_t ranks_per_group,
                      const s2d_table_load_profile* profiles, uint32_t n_profiles);

/* ShardingPlan::owner_of (src/planner.cpp:20-28). */
int s2d_plan_owner_of(const s2d_plan_entry* plan, uint32_t n_entries, uint32_t table_id,
                      uint32_t row, uint32_t* owner);

/* imbalance_ratio (src/planner.cpp:125-143). */
int s2d_imbalance_ratio(const double* per_rank, uint32_t n, double* out);

/* OptimizerConfig::validate (src/optimizer.cpp:19-23) + effective_lr (61-63). */
int s2d_effective_lr(double v, const s2d_optimizer_config* cfg, double* out);

/* Analytic helpers of the reference's Python module (bindings/module.cpp:43-89,
 * 133-145); host-only, outside the step. */
/* memory_overhead / sync_latency / qps_scaling_factor (src/cost_model.cpp:24-55) */
int s2d_memory_overhead(double table_size_gb, uint32_t groups, uint32_t total_gpus, double* out);
int s2d_sync_latency(double table_size_gb, uint32_t groups, uint32_t total_gpus, double sync_bw_gbps, double* out);
int s2d_qps_scaling_factor(double qps_base, double gpus_base, double qps_new, double gpus_new, double* out);
/* evaluate_ne (src/trainer.cpp:14-43): mean log-loss / entropy of the mean-CTR predictor */
int s2d_evaluate_ne(const double* probs, const float* labels, uint64_t n, double* ne, double* baseline_ctr);
/* Proposition 1 moment analysis (src/moment_analysis.cpp:69-148) behind the
 * choice of the AdaGrad scaling factor c */
int s2d_closed_form_ratio(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups, double* out);
int s2d_recommend_c(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups, double* out);
int s2d_estimate_increment_ratio(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups,
                                 uint64_t trials, uint64_t seed, double* ratio, double* std_error);

/* ---- device context --------------------------------------------------- */

typedef struct s2d_ctx s2d_ctx;

int s2d_device_count(int* out);

/* 128-byte NCCL bootstrap id; rank 0 creates it and the caller broadcasts it
 * (e.g. over torch.distributed) before s2d_ctx_create on every rank. */
int s2d_nccl_unique_id(uint8_t out[128]);

/* Replaces the Trainer ctor's mesh set-up (src/trainer.cpp:180-214): one
 * context per GPU, global rank `rank` of `total_ranks`, `groups` DP replicas.
 * nccl_id may be NULL when total_ranks == 1. */
int s2d_ctx_create(int device, uint32_t total_ranks, uint32_t groups, uint32_t rank,
                   const uint8_t* nccl_id, s2d_ctx** out);
int s2d_ctx_destroy(s2d_ctx* ctx);

/* Single-process mesh ("virtual ranks", as the reference Trainer runs its
 * T ranks inside one process: src/trainer.cpp:80-97, 164-257).  A hub is the
 * in-process rendezvous of total_ranks contexts; each context is driven by
 * its own host thread (calls of different ranks block on each other exactly
 * like NCCL ranks do).  Ranks may share one GPU or sit on different GPUs of
 * the process; peer buffers are plain device pointers, and every kernel of
 * the step -- K1 bucketing, the fused exchanges, the device barriers, the
 * K5 replica sync -- is the code the NCCL mesh runs.  The hub must outlive
 * its contexts (s2d_hub_destroy drops the caller's reference; contexts keep
 * their own). */
typedef struct s2d_hub s2d_hub;
int s2d_hub_create(uint32_t total_ranks, s2d_hub** out);
int s2d_hub_destroy(s2d_hub* hub);
int s2d_ctx_create_local(int device, uint32_t total_ranks, uint32_t groups, uint32_t rank, s2d_hub* hub,
                         s2d_ctx** out);

/* Runs all work of this context on `cuda_stream` (a cudaStream_t); NULL
 * selects the context's own stream. */
int s2d_ctx_set_stream(s2d_ctx* ctx, void* cuda_stream);

/* strict = 1 (default): every call waits for its device work and reports
 * device faults at the call, like the reference's exceptions.  strict = 0:
 * calls return once work is queued; faults surface at s2d_synchronize. */
int s2d_ctx_set_strict(s2d_ctx* ctx, int strict);

/* async = 0 (default): an S2D_HOST pooled output is complete when
 * s2d_lookup_forward returns.  async = 1: host inputs go up on the context's
 * H2D copy stream and the pooled read-back runs on its D2H copy stream,
 * overlapping the upstream upload, the sort and the update; at N = 1 two
 * staging buffers alternate, so the next step's lookup also overlaps it and
 * the read-back is complete at s2d_synchronize (or when the forward after
 * next reuses its staging); at N > 1 it completes by the end of the
 * following s2d_backward_update's work.  Host buffers must stay valid (and
 * unchanged) until then. */
int s2d_ctx_set_async_host(s2d_ctx* ctx, int async);

/* Tables + plan (the identical-in-every-group plan).  The
 * context allocates only the shards its local rank owns: fp32 or bf16
 * weights, fp32 moments (embedding.hpp:16-17).  Replaces the replica
 * allocation at src/trainer.cpp:216-224. */
int s2d_register_tables(s2d_ctx* ctx, const s2d_table_desc* tables, uint32_t n_tables,
                        const s2d_plan_entry* plan, uint32_t n_entries, int32_t weight_dtype);

/* OptimizerConfig for the fused update; validates like
 * OptimizerConfig::validate (src/optimizer.cpp:19-23). */
int s2d_set_optimizer(s2d_ctx* ctx, const s2d_optimizer_config* cfg);

/* Bit-exact device port of init_table (src/embedding.cpp:17-37) for the
 * owned shards; moments start at zero. */
int s2d_init_tables(s2d_ctx* ctx, uint64_t seed);

/* Copy rows [row_lo,row_hi) of `table` (owned by this rank) in or out of the
 * device shard; w: (hi-lo)*dim fp32, v: (hi-lo) fp32 (either may be NULL).
 * Used for checkpoint / parity (apply_row_update-style writes,
 * src/embedding.cpp:108-129). */
int s2d_shard_write(s2d_ctx* ctx, uint32_t table, uint32_t row_lo, uint32_t row_hi,
                    const float* w, const float* v);
int s2d_shard_read(s2d_ctx* ctx, uint32_t table, uint32_t row_lo, uint32_t row_hi, float* w,
                   float* v);
/* Rows of `table` by global id (each owned by this rank, any order, repeats
 * allowed): w n x dim fp32 (bf16 shards widened exactly), v n fp32; either
 * may be NULL.  The row-access half of EmbeddingTable::row()
 * (include/sparse2d/embedding.hpp:19-22) for scattered rows. */
int s2d_shard_gather(s2d_ctx* ctx, uint32_t table, uint32_t n_rows, const uint32_t* rows, float* w, float* v);
/* apply_row_update (src/embedding.cpp:108-129) for n_rows rows of `table`
 * (global row ids owned by this rank): w[row][j] = f32(f64(w) + delta[i][j])
 * (bf16 tables: one RNE rounding of the f64 sum), v[row] = f32(new_moment[i]).
 * delta is n_rows x dim f64, row-major, in call order; a row listed twice is
 * updated twice in that order.  S2D_ERANGE for a row outside the owned range,
 * S2D_EINVAL for a new_moment < 0 or nonfinite; nothing is written then. */
int s2d_apply_row_updates(s2d_ctx* ctx, uint32_t table, uint32_t n_rows, const uint32_t* rows,
                          const double* delta, const double* new_moment);
/* Owned range of `table` on this rank ([0,0) when none). */
int s2d_shard_range(s2d_ctx* ctx, uint32_t table, uint32_t* row_lo, uint32_t* row_hi);

/* S2DCKPT1 checkpoint, byte-compatible with the reference's
 * save_checkpoint / load_checkpoint (src/embedding.cpp:133-219): "S2DCKPT1",
 * u32 count, per table u32 version = 1, u32 table_id, u64 rows, u64 dim,
 * f32 weights[rows*dim], f32 moments[rows], little-endian, written to
 * path.tmp and renamed.  Collective over all ranks of the context: DP group
 * 0's ranks write their own row ranges in place (the replica
 * Trainer::save_tables saves, src/trainer.cpp:875-878); every rank loads its
 * owned rows into its replica (Trainer::load_tables copies the file into
 * all replicas, trainer.cpp:880-896).  Table count / shape mismatch and IO
 * failures -> S2D_ERUNTIME; bf16 shards are widened on save and rounded to
 * nearest-even on load. */
int s2d_save_tables(s2d_ctx* ctx, const char* path);
int s2d_load_tables(s2d_ctx* ctx, const char* path);

/* Device-side synthetic input: the reference DataGenerator's ids for one
 * rank's batch (DataGenerator ctor Zipf CDF, src/data.cpp:85-98;
 * gen_batch_into, data.cpp:115-136; train lane), bit-exact.  Table f has
 * the registered rows as num_ids, Zipf exponent zipf[f] (>= 0) and
 * ids_per_sample[f] ids per bag.  Writes lengths[batch*F] (sample-major
 * bags) and ids[batch * sum_f ids_per_sample[f]] in (sample, feature, draw)
 * order -- the s2d_lookup_forward input layout.  mem says where lengths/ids
 * live.  Invalid specs -> S2D_EINVAL (FeatureSpec::validate, data.cpp:26-35). */
int s2d_gen_batch(s2d_ctx* ctx, uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, const double* zipf,
                  const uint32_t* ids_per_sample, uint32_t* lengths, uint32_t* ids, int32_t mem);

/* Forward of one step for this rank's batch of `batch` samples: sample-major
 * bags (s, f) given as lengths[batch*F] and the `nnz` global row ids of all
 * bags concatenated.  Runs K1 input-dist bucketing + id all-to-all, K2 owner
 * partial pooling, the pooled all-to-all and the requester combine, writing
 * pooled[batch][sum_f dim_f] fp32.  Replaces build_demand + owner_lookup +
 * route_all_to_all(LookupA2A) + the pooling half of pool_and_forward
 * (src/trainer.cpp:283-390).  `mem` (S2D_HOST | S2D_DEVICE) says where the
 * three buffers live; host buffers are copied inside the call. */
int s2d_lookup_forward(s2d_ctx* ctx, uint32_t batch, const uint32_t* lengths, const uint32_t* ids,
                       uint64_t nnz, float* pooled, int32_t mem);

/* Zero-copy output: with mem == S2D_DEVICE and pooled == NULL,
 * s2d_lookup_forward writes into this engine-owned buffer ([batch][sum dim]
 * fp32, valid until the next forward), which the other ranks of the MP group
 * map: owners of single-owner tables store their pooled rows straight into
 * it over NVLink and the requester-side combine skips them.  *out = NULL
 * before the first forward. */
int s2d_pooled_buffer(s2d_ctx* ctx, float** out);

/* Backward + fused optimizer for the batch of the last s2d_lookup_forward:
 * upstream[batch][sum_f dim_f] fp32 per-sample gradients (not batch-divided,
 * src/trainer.cpp:424-427).  Runs the gradient all-to-all, K3 radix-sort
 * dedup + segment reduce (x 1/(N*B)) and K4 moment-scaled row-wise AdaGrad
 * (or SGD) reading and writing each row and its accumulator once.  Replaces
 * build_grad_payloads + route_all_to_all(GradA2A) + owner_update
 * (src/trainer.cpp:440-505, src/optimizer.cpp:25-90). */
int s2d_backward_update(s2d_ctx* ctx, const float* upstream, int32_t mem);

/* K5: weight + moment mean over the DP replicas of every row updated in any
 * replica since the last sync (src/trainer.cpp:547-596).  No-op when M = 1.
 * The caller decides the cadence ((step+1) % sync_interval == 0,
 * src/trainer.cpp:661). */
int s2d_replica_sync(s2d_ctx* ctx);

/* Waits for the context's stream and reports deferred device faults
 * (id out of range -> S2D_ERANGE, nonfinite gradient -> S2D_ENONFINITE). */
int s2d_synchronize(s2d_ctx* ctx);

int s2d_get_step_stats(s2d_ctx* ctx, s2d_step_stats* out);

/* Per-phase device time (CUDA events on the context's stream), summed since
 * the last query.  Phases: 0 input staging, 1 K1 bucketing, 2 id all-to-all,
 * 3 K2 lookup, 4 pooled all-to-all, 5 combine, 6 grad gather, 7 grad
 * all-to-all, 8 radix sort, 9 host count sync (N > 1), 10 fused update,
 * 11 replica sync (dirty-row union), 12 sync push, 13 sync mean, 14 sync
 * scatter.  n must be >= 12 (the first n phases are written).  Profiling is
 * off by default; on = 1 times every phase, on = 2 only the fused update
 * (phase 10; fewer stream drains). */
#define S2D_NUM_PHASES 15
int s2d_ctx_set_profiling(s2d_ctx* ctx, int on);
int s2d_get_phase_times(s2d_ctx* ctx, double* ms, uint32_t* counts, uint32_t n);

/* MetricsRow moment statistics (include/sparse2d/trainer.hpp:72-79,
 * src/trainer.cpp:745-771) of this rank's MP group replica (group 0's is the
 * reference's, which reads replicas[0]): over every row of every table,
 * eff_lr_p50 / eff_lr_p99 = effective_lr at ascending index ceil(q*n)-1 of
 * the per-row effective learning rates, v_mean = mean moment.  Collective
 * over the MP group.  The percentiles are exact (radix select of the moment
 * at the matching descending index, effective_lr is non-increasing in v);
 * v_mean sums in a fixed blocked order (the reference's is sequential). */
typedef struct {
  double eff_lr_p50;
  double eff_lr_p99;
  double v_mean;
  uint64_t rows;
} s2d_metrics_row;
int s2d_metrics(s2d_ctx* ctx, s2d_metrics_row* out);

/* Synthetic upstream gradient for one rank's batch:
 * out[s][coff_f + j] = f32(1e-3 * z), z the Box-Muller normals of
 * CounterRng({seed, step, rank, s, f}) (rng.hpp) in draw order.  mem says
 * where out ([batch][sum dims] fp32) lives. */
int s2d_gen_upstream(s2d_ctx* ctx, uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, float* out,
                     int32_t mem);

/* ---- Trainer facade (include/sparse2d/trainer.hpp:106-132) ---------------
 * The reference's one-object training loop over the 2D mesh: every rank a
 * virtual rank of this process on the GPUs given (rank r -> devices[r %
 * n_devices], all GPUs round-robin when devices is NULL).  Per step and
 * rank: the reference DataGenerator's ids (fixed pooling, trainer.hpp
 * ids_per_sample), the lookup, the upstream gradient, the backward + fused
 * update, and the replica sync every sync_interval steps
 * ((step+1) % sync_interval == 0, trainer.cpp:661).  The upstream gradient
 * comes from the caller's callback when one is set, else (dense_model = 1,
 * the reference's Trainer) from the toy DLRM MLPs on the device: the
 * DataGenerator's dense features and labels (data.cpp:37-68, 137-145),
 * dense_arch + over_arch forward, sigmoid / log-loss, backward
 * (trainer.cpp:366-438), and after every step the dense DP step -- the
 * gradient left fold over (rank, sample) and one SGD step with eta / (T*B)
 * adopted by every rank (trainer.cpp:507-545) -- else (dense_model = 0) from
 * s2d_gen_upstream. */
typedef struct {
  uint32_t total_ranks, groups;                 /* Topology */
  uint32_t num_tables, rows_per_table, dim;     /* DlrmConfig (embedding part) */
  int32_t strategy;                             /* S2D_ROW_WISE (reference default) | S2D_TABLE_WISE */
  double zipf_exponent;
  uint32_t ids_per_sample;
  uint32_t per_rank_batch;
  uint64_t steps;
  uint32_t sync_interval;
  uint64_t data_seed, init_seed;
  s2d_optimizer_config opt;
  int32_t weight_dtype;                         /* S2D_F32 | S2D_BF16 */
  uint32_t n_devices;
  const int32_t* devices;
  int32_t dense_model;                          /* 1: device MLPs (reference Trainer); 0: synthetic upstream */
  uint32_t dense_dim;                           /* DataParams::dense_dim (data.hpp:51-56), default 8 */
  uint32_t dense_hidden, over_hidden;           /* DlrmConfig (model.hpp:68-77), defaults 32, 64 */
  double gt_id_scale, gt_dense_scale, gt_bias;  /* DataParams ground truth, defaults 0.25, 0.35, -0.8 */
  uint64_t eval_cadence;                        /* 0 = evaluate only after the final step (trainer.hpp:62-64) */
  uint32_t eval_samples;                        /* default 100000 */
  uint64_t eval_seed;                           /* default 3 */
} s2d_trainer_options;

/* MetricsRow (trainer.hpp:72-79) and NEReport (trainer.hpp:29-36). */
typedef struct {
  uint64_t step;
  double loss, ne, eff_lr_p50, eff_lr_p99, v_mean;
} s2d_train_metrics_row;
typedef struct {
  double ne, baseline_ctr;
  uint64_t eval_samples;
} s2d_ne_report;

/* Called on rank `rank`'s thread after the step's forward: fill upstream
 * ([batch][num_tables*dim] fp32, device, per-sample, not batch-divided:
 * trainer.cpp:424-427) from the pooled rows (device) of the batch whose bag
 * lengths are `lengths` (device); cuda_stream is the rank's stream.
 * Non-zero return aborts the step. */
typedef int (*s2d_upstream_fn)(void* user, uint32_t rank, uint64_t step, uint32_t batch, const uint32_t* lengths,
                               const float* pooled, float* upstream, void* cuda_stream);

typedef struct s2d_trainer s2d_trainer;
int s2d_trainer_create(const s2d_trainer_options* opts, s2d_trainer** out);
int s2d_trainer_destroy(s2d_trainer* t);
int s2d_trainer_set_upstream(s2d_trainer* t, s2d_upstream_fn fn, void* user);
/* Trainer::step_n (trainer.hpp:117) and run (opts.steps - steps done). */
int s2d_trainer_step_n(s2d_trainer* t, uint64_t count);
int s2d_trainer_run(s2d_trainer* t);
int s2d_trainer_steps_done(s2d_trainer* t, uint64_t* out);
/* Trainer::plan (trainer.hpp:124). */
int s2d_trainer_plan(s2d_trainer* t, s2d_plan_entry* out, uint32_t cap, uint32_t* n);
/* Trainer::replica_tables(group)[table] (trainer.hpp:123): w rows*dim, v rows
 * (tables() = group 0). */
int s2d_trainer_replica_table(s2d_trainer* t, uint32_t group, uint32_t table, float* w, float* v);
/* Trainer::save_tables / load_tables (trainer.hpp:126-127), S2DCKPT1. */
int s2d_trainer_save_tables(s2d_trainer* t, const char* path);
int s2d_trainer_load_tables(s2d_trainer* t, const char* path);
/* MetricsRow moment columns of group 0's replica. */
int s2d_trainer_metrics(s2d_trainer* t, s2d_metrics_row* out);
/* Trainer::rank_model(rank) (trainer.hpp:125): arch 0 = dense_arch, 1 =
 * over_arch; w1 [hidden][in], b1 [hidden], w2 [out][hidden], b2 [out] fp32
 * (any may be NULL).  S2D_EINVAL without the dense model. */
int s2d_trainer_rank_model(s2d_trainer* t, uint32_t rank, int32_t arch, float* w1, float* b1, float* w2, float* b2);
/* MetricsRow::loss of the last step (trainer.cpp:538): the global-batch mean
 * training loss; S2D_EINVAL without the dense model or before a step. */
int s2d_trainer_last_loss(s2d_trainer* t, double* out);
/* TrainResult::metrics (trainer.hpp:87-98): with the dense model, one row
 * after every eval_cadence-th step and after step opts.steps -- loss, NE of
 * the eval set (DataGenerator lane kEval, eval_seed, chunks of 1024;
 * trainer.cpp:687-712) pooled from group 0's replica with rank 0's MLPs
 * (eval_probs, trainer.cpp:714-743), and the moment columns
 * (trainer.cpp:745-771).  n = rows so far; out may be NULL. */
int s2d_trainer_metrics_rows(s2d_trainer* t, s2d_train_metrics_row* out, uint32_t cap, uint32_t* n);
/* Trainer::finalize's final_ne (trainer.cpp:788-793): evaluates now unless
 * the last step already did.  S2D_EINVAL without the dense model. */
int s2d_trainer_final_ne(s2d_trainer* t, s2d_ne_report* out);
/* The context of one virtual rank (owned by the trainer). */
int s2d_trainer_rank_ctx(s2d_trainer* t, uint32_t rank, s2d_ctx** out);

/* Number of kernels this library has launched in the process. */
uint64_t s2d_launch_count(void);

/* K4 on caller rows (the binding behind Python adagrad_row_step,
 * bindings/module.cpp:93-107): n_rows rows of `dim`, w fp32 [n][dim],
 * v fp32 [n], g f64 [n][dim], host buffers; lr_out[n] receives the effective
 * learning rate (may be NULL).  Runs the same device code as the step. */
int s2d_adagrad_rows(const s2d_optimizer_config* cfg, uint32_t n_rows, uint32_t dim, float* w,
                     float* v, const double* g, double* lr_out);

/* pool_ids / lookup_and_pool (include/sparse2d/embedding.hpp:41-58,
 * src/embedding.cpp:39-106) on the device: n_bags bags, bag b = ids
 * [bag_off[b], bag_off[b+1]) of table `table_id` (w: rows x dim fp32, host,
 * indexed by global row), over the shards [lo[s], hi[s]) in presentation
 * order: per shard the f64 sum of its hits in id order rounded to f32, then
 * the f64 sum of those partials rounded to f32, into out [n_bags][dim]
 * (host).  An id covered by no shard: S2D_ERANGE "lookup id I outside shard
 * ranges of table T: [lo,hi) ..." (the first in bag order, checked before
 * any pooling); no shard or dim > 512: S2D_EINVAL. */
int s2d_pool_ids(const float* w, uint32_t rows, uint32_t dim, uint32_t table_id, uint32_t n_shards,
                 const uint32_t* lo, const uint32_t* hi, uint64_t n_bags, const uint64_t* bag_off,
                 const uint32_t* ids, float* out);
/* aggregate_group_gradient (include/sparse2d/optimizer.hpp:36-44,
 * src/optimizer.cpp:25-59) on the device: contribution i is (rows[i],
 * grads[i*dim .. +dim) f64) in canonical arrival order; for every row with a
 * contribution, ascending: out_rows[k], out_g[k][dim] = (f64 sum in arrival
 * order) * (1/group_batch), out_count[k] = contributions (sample_count).
 * *n_out = rows (all outputs NULL: size query; else cap >= rows).
 * group_batch == 0: S2D_EINVAL. */
int s2d_aggregate_group_gradient(const uint32_t* rows, const double* grads, uint64_t n, uint32_t group_batch,
                                 uint32_t dim, uint32_t* out_rows, double* out_g, uint32_t* out_count, uint64_t cap,
                                 uint64_t* n_out);

/* Debug view of the last step's wire buffers for bit-exact layout tests.
 * which: 0 demand lengths received [N requester][B*F] u32,
 *        1 demand ids received (canonical order) u32,
 *        2 pooled partials received from the owners, concatenated by owner, f32,
 *        3 gradient rows received from the requesters, concatenated by requester, f32,
 *        4 owner mask per local bag u32 [B*F],
 *        5 unique rows updated (global row ids, ascending by (table,row)) u32,
 *        6 engine-owned pooled output [B][sum dims] f32,
 *        8 table id of each row of view 5 u32,
 *        7 f64 gradient of every row of the last update, rows as in view 5,
 *          max dim columns (needs s2d_ctx_set_debug_grad(ctx, 1) before the
 *          backward; aggregate_group_gradient's output, optimizer.cpp:25-59).
 * Copies min(cap, size) elements; *n = size. */
int s2d_debug_read(s2d_ctx* ctx, int32_t which, void* out, uint64_t cap, uint64_t* n);
/* on = 1: every backward also records the f64 row gradients (debug view 7;
 * one extra scan and a host read of the row count per step). */
int s2d_ctx_set_debug_grad(s2d_ctx* ctx, int on);

#ifdef __cplusplus
}
#endif

#endif /* SPARSE2D_B200_H */
