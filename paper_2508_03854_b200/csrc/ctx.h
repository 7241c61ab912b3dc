// Per-GPU context: owns the rank's shards, workspaces, stream and NCCL
// communicators, and sequences one 2D-sparse-parallel step.  Mirrors
// Trainer::Impl's per-rank state (src/trainer.cpp:164-257) minus the dense
// MLP, with the simulated collectives replaced by NCCL over NVLink.
#pragma once

#include <nccl.h>

#include <vector>

#include "comm.h"
#include "common.h"

#define S2D_NCCL(call)                                                                    \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      throw ::s2d::Error(S2D_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

namespace s2d {

// Phases timed with CUDA events when profiling is on (s2d_get_phase_times).
enum Phase : int {
  kPhInput = 0,   // H2D staging + bag offsets
  kPhBucket,      // K1 count / scans / permute
  kPhA2AIds,      // counts + lengths + ids all-to-all
  kPhLookup,      // K2 owner lookup
  kPhA2ALookup,   // C1 pooled partials all-to-all
  kPhCombine,     // requester combine (+ D2H in host mode)
  kPhGradGather,  // C2 send layout
  kPhA2AGrad,     // C2 all-to-all
  kPhSort,        // K3a radix sort
  kPhCountSync,   // N > 1: host read of the count matrix (GPU waits for the next launch)
  kPhUpdate,      // K3b chunk sums + K4 fused update
  kPhSync,        // K5 replica sync: dirty-row union (flag compaction, list exchange, host reads)
  kPhSyncPush,    // K5: rows pushed to the slice owners (snapshot sync: dirty rows to every peer) + barrier
  kPhSyncMean,    // K5: slice means stored into every replica + barrier (snapshot sync: every union mean, local)
  kPhSyncScatter, // K5: means scattered into the shard, dirty flags cleared
  kNumPhases
};

// A buffer every rank of the MP group maps (CUDA IPC over NVLink).
struct PeerBuf {
  DevBuf buf;
  size_t cap = 0;               // identical on every rank of the group
  std::vector<void*> ptr;       // [N] (own entry = buf.p)
  std::vector<void*> opened;    // IPC mappings to close
};

struct Ctx {
  // mesh (topology.hpp:13-26): rank -> (group = r / N, local = r % N)
  int device = 0;
  uint32_t T = 1, M = 1, N = 1, rank = 0, group = 0, local = 0;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  // host<->device copies of S2D_HOST calls run on their own streams so the
  // pooled read-back (D2H) overlaps the upstream upload (H2D) and the sort
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_fwd = nullptr, ev_d2h = nullptr, ev_up = nullptr;
  // host-mode staging pairs (ids + lengths, upstream, N == 1 pooled
  // read-back): buffer k is refilled only after the event of its last use
  cudaEvent_t ev_in_ready = nullptr, ev_in_used[2] = {nullptr, nullptr}, ev_up_used[2] = {nullptr, nullptr},
              ev_d2h_done[2] = {nullptr, nullptr};
  bool in_used_rec[2] = {false, false}, up_used_rec[2] = {false, false}, d2h_done_rec[2] = {false, false};
  int in_sel = 0, up_sel = 0, out_sel = 0;
  bool async_host = false;  // S2D_HOST pooled output valid at return (false) or after s2d_synchronize (true)
  bool d2h_pending = false;
  // N > 1: the (slot, row) sort runs on its own stream from the end of the
  // owner lookup, beside the combine and the gradient all-to-all
  cudaStream_t sort_stream = nullptr;
  cudaEvent_t ev_keys = nullptr, ev_sorted = nullptr;
  bool sort_pending = false;
  // M > 1: the replica sync's device tail runs on sync_stream (overlapping
  // the next forward's bucketing / id exchange); join_sync orders the main
  // stream after it wherever weights, moments or dirty flags are touched
  cudaStream_t sync_stream = nullptr;
  cudaEvent_t ev_union = nullptr, ev_sync_done = nullptr;
  bool sync_pending = false, sync_stats_pending = false;
  uint32_t sync_cmax = 0;
  uint64_t sync_sent_rows = 0;  // rows this replica pushed at the last sync (stats)
  uint64_t sync_pair_rows = 0;  // pair sync: both replicas' list lengths (stats)
  bool sync_snapshot_used = false;
  // M > 1 snapshot log (StreamUpdateArgs::snap): snap_ub = log rows the
  // interval's updates span (every item of every update since the last
  // sync); snap_broken marks an interval with writes the log did not see
  // (shard_io / apply_row_updates) or a log that could not grow -- the next
  // sync then exchanges every union row instead
  DevBuf snap, snap_pos;
  uint64_t snap_cap_rows = 0, snap_ub = 0;
  DevBuf head_ord_buf;  // heads before each sorted position (the dense snapshot log's row index)
  // the update's own dirty list (M = 2): valid while no other write followed
  // the first update after a sync
  DevBuf dlist;
  bool dirty_clean = true;  // no row dirtied since the last replica sync
  bool list_ready = false;  // dlist is this replica's whole dirty set
  uint64_t list_n = 0;      // items of the update that wrote dlist (head_ord_buf[list_n] = its rows)
  size_t dev_total = 0;  // device memory size (bounds the snapshot log)
  bool snap_broken = false;
  bool snapshot_enabled() const;
  bool sync_list_mode_enabled() const;
  uint64_t snap_reserve(uint64_t items);
  void join_sync();
  void launch_sort(cudaStream_t st);
  const uint32_t* sorted_k = nullptr;  // sorted pairs of the last launch_sort
  const uint32_t* sorted_v = nullptr;
  Comm world, mp, dp;
  std::shared_ptr<LocalHub> hub;  // virtual ranks of one process (null: NCCL)
  // runs after every member destructor: the last virtual rank frees the
  // deferred buffers (comm.h)
  struct LocalGuard {
    bool armed = false;
    ~LocalGuard() {
      if (armed) local_ctx_leave();
    }
  } local_guard;
  bool strict = true;

  // tables + plan
  uint32_t F = 0, sum_dims = 0, max_dim = 0;
  int bf16 = 0;
  bool any_mean = false;  // some table uses S2D_POOL_MEAN
  std::vector<s2d_table_desc> tables;
  std::vector<s2d_plan_entry> plan;
  std::vector<FeatDev> feats;
  std::vector<RangeDev> ranges;
  std::vector<uint32_t> vbase_sorted, feat_of_vbase;  // owned features by slot base
  uint32_t n_slots = 0;
  uint32_t uni_dim = 0;
  bool all_same_dim = false;  // dim shared by every owned table (0: mixed)
  bool slot_rows = false;     // all_same_dim and weights offset = slot * dim
  uint64_t n_weight_elems = 0;
  DevBuf d_feats, d_ranges, d_vbase_sorted, d_feat_of_vbase;
  DevBuf weights, moments, dirty;

  s2d_optimizer_config opt{0.05, 1e-8, 1.0, S2D_ROWWISE_ADAGRAD};
  bool have_opt = false;

  // device fault flag
  DevBuf err;
  HostBuf err_host;

  // ---- per-step state ----
  uint32_t B = 0;
  uint64_t nnz_local = 0, nnz_own = 0;
  bool fwd_done = false;
  DevBuf in_len2[2], in_ids2[2], in_off, upstream_stage, up_stage2[2], p_pooled_host[2], mean_stage;
  DevBuf cnt, send_off, eoff_req;  // requester side (N > 1)
  DevBuf own_idoff, own_eoff;      // owner side (N > 1)
  // MP-group peer buffers: barrier flags, count matrix, received bag
  // lengths [N][B*F], received ids, received partials (requester), received
  // gradient rows (owner)
  PeerBuf p_flags, p_xcnt, p_len, p_ids, p_part, p_grad, p_pooled;
  DevBuf p_pooled_local;  // engine-owned pooled output when N == 1
  DevBuf hbuf, row_upd_scratch;
  uint64_t epoch = 0;
  uint32_t engine_mask = 0;  // requesters of the current step that asked for the engine-owned output
  DevBuf keys_a, vals_a, keys_b, vals_b, sort_tmp, scan_tmp;
  DevBuf uslot, useg, counters, chunk_base, chunk_seg, chunk_part;
  DevBuf sync_list, sync_lists, sync_count, sync_packed, sync_gathered, sync_tmp;
  HostBuf h_counts, h_xcnt;
  uint64_t host_wait_total_ns = 0;  // host blocked on the count read, since creation
  std::vector<uint64_t> nnz_to, nnz_from, ef_to, ef_from, send_bound, eoff_req_bound, own_eoff_bound,
      ids_base_at_owner, part_base_at_req, grad_base_at_owner;
  s2d_step_stats stats{};
  bool stats_counters_valid = false;
  void refresh_stats();

  // profiling
  bool profile = false;
  bool profile_hot_only = false;  // events only around the update kernels (the dominant phase)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_marks;  // (phase, index of start event)
  int open_phase = -1;
  void phase_begin(int ph);
  void phase_end();
  void phase_times(double* ms, uint32_t* counts);

  ~Ctx();
  void create(int device, uint32_t T, uint32_t M, uint32_t rank, const uint8_t* nccl_id,
              std::shared_ptr<LocalHub> hub = nullptr);
  void register_tables(const s2d_table_desc* t, uint32_t n, const s2d_plan_entry* p, uint32_t np,
                       int dtype);
  void set_optimizer(const s2d_optimizer_config& c);
  void init_tables(uint64_t seed);
  void shard_io(uint32_t table, uint32_t lo, uint32_t hi, float* w, float* v, bool write);
  void apply_row_updates(uint32_t table, uint32_t n, const uint32_t* rows, const double* delta,
                         const double* new_moment);
  void lookup_forward(uint32_t batch, const uint32_t* lengths, const uint32_t* ids, uint64_t nnz,
                      float* pooled, int mem);
  void backward_update(const float* upstream, int mem);
  void replica_sync();
  void synchronize_and_check();
  // S2DCKPT1 checkpoint of DP group 0's replica (checkpoint.cpp)
  DevBuf bar_buf;
  int world_barrier(int failed);
  void save_tables(const char* path);
  void load_tables(const char* path);
  // device-side synthetic input (gen.cpp): per-table Zipf CDFs cached by exponent
  DevBuf gen_cdf, gen_meta, gen_lengths, gen_ids;
  std::vector<double> gen_zipf;
  std::vector<uint64_t> gen_cdf_off;
  void gen_batch(uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, const double* zipf,
                 const uint32_t* ids_per_sample, uint32_t* lengths, uint32_t* ids, int mem, uint64_t lane = 0);
  void gen_upstream(uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, float* out, int mem);
  void debug_read(int which, void* out, uint64_t cap, uint64_t* n);
  void gather_rows(uint32_t table, uint32_t n, const uint32_t* rows, float* w, float* v);
  DevBuf gather_scratch, dbg_head, dbg_grad;
  bool debug_grad = false;
  uint64_t dbg_rows = 0;
  void metrics(s2d_metrics_row* out);
  DevBuf metric_buf;

 private:
  void finish_call();
  void check_faults();
  PeerPtrs ptrs(const PeerBuf& pb) const;
  void peer_alloc(PeerBuf& pb, size_t bytes);
  void peer_alloc_in(PeerBuf& pb, size_t bytes, Comm& comm);
  void peer_barrier();
  // DP group over NVLink peer memory (replica sync): every replica's
  // weights / moments mapped, a group barrier, a staging slice
  int dp_p2p = -1;  // -1 undecided, 0 NCCL path, 1 P2P path
  std::vector<void*> dp_w, dp_v, dp_opened;
  PeerBuf dp_flags, dp_stage;
  uint64_t dp_epoch = 0;
  void dp_setup();
  void dp_barrier(cudaStream_t st);
  void read_counts();
 public:
  float* pooled_buffer();
};

}  // namespace s2d
