// Shared declarations of libsparse2d_b200: error type, device-side table
// metadata, kernel launch wrappers.  Kernels live in k_*.cu, the per-rank
// step driver in ctx.cu, the C ABI in capi.cpp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sparse2d_b200.h"

namespace s2d {

// Carries an S2D_* status; capi.cpp turns it into the return code +
// s2d_last_error() message.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define S2D_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::s2d::Error(S2D_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Every kernel launch is followed by S2D_LAUNCH_CHECK, which also counts it
// (s2d_launch_count: the bench's gpu_launches evidence).
void count_launch();
// the thread's s2d_last_error() message (capi.cpp)
void set_last_error(const char* m);
#define S2D_LAUNCH_CHECK()            \
  do {                                \
    ::s2d::count_launch();            \
    S2D_CUDA(cudaGetLastError());     \
  } while (0)

// Kernel launch with programmatic stream serialization (PDL): the kernel may
// be scheduled during its predecessor's tail and must call pdl_wait() first.
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  S2D_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  S2D_LAUNCH_CHECK();
}

// cudaFuncAttributeMaxDynamicSharedMemorySize for `kernel` on the current
// device, set once per (kernel, device) (the attribute is per device: a
// single-process mesh may drive several GPUs)
void set_max_dynamic_smem_raw(const void* kernel, size_t bytes);
template <typename... KArgs>
inline void set_max_dynamic_smem(void (*kernel)(KArgs...), size_t bytes) {
  set_max_dynamic_smem_raw(reinterpret_cast<const void*>(kernel), bytes);
}

// zero `bytes` at p on st as a PDL kernel (keeps the launch chain unbroken,
// unlike cudaMemsetAsync)
void launch_zero(void* p, size_t bytes, cudaStream_t st);

// Device fault bits (checked once per step, SURVEY.md 5 failure detection).
enum : uint32_t { kErrIdRange = 1u, kErrNonfinite = 2u, kErrPeerTimeout = 4u };
// batch word of the published count matrix: bit 32 = requester uses the
// engine-owned pooled output
constexpr uint64_t kEngineOutFlag = 1ull << 32;

constexpr int kMaxPeers = 32;
// Per-peer device pointers of one IPC-shared buffer (index = local rank in
// the MP group; the own entry is the local buffer).
struct PeerPtrs {
  void* p[kMaxPeers];
};

// Per-feature metadata visible to every kernel.
struct FeatDev {
  uint32_t dim;     // D_f, multiple of 4
  uint32_t rows;    // global rows of the table
  uint32_t lo, hi;  // row range this rank owns (lo == hi: none)
  uint64_t wbase;   // element offset of owned row `lo` in the weight store
  uint32_t vbase;   // slot of owned row `lo` (slot = vbase + row - lo)
  uint32_t coff;    // column offset inside a [sum_f D_f] pooled/upstream row
  uint32_t rbeg;    // owner ranges of this table: ranges[rbeg, rend)
  uint32_t rend;
  uint32_t single;  // the plan gives the table one owner: partial == pooled row
  uint32_t mean;    // S2D_POOL_MEAN: pooled row scaled by 1/L, gradient row by 1/L
};

// Owner range of a table inside the MP group (sorted by lo per table).
struct RangeDev {
  uint32_t lo, hi, owner, pad;
};

constexpr int kMaxDim = 512;       // trainer.cpp:99
constexpr int kMaxRanksPerGroup = 32;  // owner bitmask width (trainer.cpp:193-195)

// ---- launch wrappers (all asynchronous on `st`) --------------------------

// scans (k_scan.cu)
enum class ScanOp : int { Identity = 0, NonzeroDim = 1 };
// out[i] = sum_{k<i} op(in[k]) for i in [0, n]; out has n+1 entries.
// NonzeroDim: op(x at flat index k) = x ? feats[k % F].dim : 0.
void scan_u32_to_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st, void* tmp,
                     size_t tmp_bytes);
void scan_nonzero_dim_u64(const uint32_t* in, uint64_t* out, uint64_t n, uint32_t F,
                          const FeatDev* feats, cudaStream_t st, void* tmp, size_t tmp_bytes);
// out[i] = number of segment heads (first index of a run of equal keys
// < n_slots) before i.
void scan_heads_u32(const uint32_t* keys, uint32_t* out, uint64_t n, uint32_t n_slots, cudaStream_t st,
                    void* tmp, size_t tmp_bytes);
size_t scan_tmp_bytes(uint64_t n);
// fused: out32 = scan_u32_to_u32(in), out64 = scan_nonzero_dim_u64(in) in one pass
void scan_count_pair(const uint32_t* in, uint32_t* out32, uint64_t* out64, uint64_t n, uint32_t F,
                     const FeatDev* feats, cudaStream_t st, void* tmp, size_t tmp_bytes);

// radix sort (k_sort.cu): stable LSD sort of (key, val) pairs by the low
// `bits` bits of key.  keys/vals ping-pong between a and b; returns true if
// the result ended in b.
size_t radix_tmp_bytes(uint64_t n, int bits);
bool radix_sort_pairs(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                      uint64_t n, int bits, void* tmp, size_t tmp_bytes, cudaStream_t st);

// embedding kernels (k_embed.cu)
void launch_init_rows(void* w, int bf16, const FeatDev* feats_host, uint32_t F, uint64_t seed,
                      cudaStream_t st);

struct LookupArgs {
  const FeatDev* feats;
  uint32_t F, B, n_req;        // bags = n_req * B * F (flattened [n][s][f])
  uint32_t sum_dims;
  const uint32_t* lengths;     // [n_req*B*F]
  const uint32_t* id_off;      // [n_req*B*F + 1]
  const uint32_t* ids;         // global row ids
  const void* weights;
  float* out;                  // direct: pooled [B][sumD]; else partial send buffer
  const uint64_t* eoff;        // non-direct: float offset of each non-empty bag
  uint32_t* keys;              // per id: slot (0xffffffff if invalid)
  uint32_t* vals;              // per id: gradient row offset in float4 units
  uint32_t* err;
  int direct;                  // N == 1: write pooled rows (zero for empty bags)
  int emit_keys;
  uint32_t uni_d4;             // dim/4 shared by every table (0: mixed dims)
  int uni_rows;                // uni_d4 != 0 and weights offset = slot * dim (slot-indexed rows)
  uint32_t zero_row;           // slot index of the all-zero row after the shard (uni_rows)
  uint32_t* ticket;            // work counter of the persistent warps (zeroed per launch)
  uint32_t blocks_per_sm;      // 0: as many as fit; else a cap (leaves room for a concurrent kernel)
  uint64_t unit_rot;           // ticket t processes 32-bag unit (t + unit_rot) % units: owners
                               // start at different requesters so their NVLink stores spread out
  // non-direct: the partial of a bag of requester n goes to
  // peer_out.p[n] + peer_adj[n] + eoff[bag] (requester n's receive buffer,
  // over NVLink); the sort vals stay local (eoff[bag] / 4)
  PeerPtrs peer_out;
  int64_t peer_adj[kMaxPeers];
  // zero-copy output: bags of single-owner tables are stored as final pooled
  // rows straight into requester n's pooled buffer peer_pooled.p[n]
  PeerPtrs peer_pooled;
  uint32_t use_peer_pooled;    // bit n: requester n takes single-owner pooled rows from the owners
};

struct CombineArgs {
  const FeatDev* feats;
  uint32_t F, B, N, sum_dims;
  const uint32_t* cnt;         // [N][B*F] ids of local bag b owned by o
  const uint64_t* eoff;        // [N*B*F + 1] float offsets into the per-owner blocks
  const float* recv;           // partials received, concatenated by owner
  float* pooled;               // [B][sumD]
  int skip_single;             // single-owner bags were written by their owners
  const uint32_t* bag_off;     // [B*F+1] local bag offsets (mean pooling: L = bag_off[b+1] - bag_off[b])
};
void launch_combine(const CombineArgs& a, int max_dim, cudaStream_t st);

struct GradGatherArgs {
  const FeatDev* feats;
  const RangeDev* ranges;      // owner of a single-owner table = ranges[rbeg].owner
  uint32_t F, B, N, sum_dims;
  const uint32_t* cnt;
  const uint64_t* eoff;
  const float* upstream;       // [B][sumD]
  const uint32_t* bag_off;     // [B*F+1] local bag offsets (mean pooling scales by 1/L)
  // gradient row of bag b for owner o -> peer_dst.p[o] + peer_adj[o] + eoff[o*BF+b]
  PeerPtrs peer_dst;
  int64_t peer_adj[kMaxPeers];
};
void launch_grad_gather(const GradGatherArgs& a, int max_dim, cudaStream_t st);

struct BucketArgs {
  const FeatDev* feats;
  const RangeDev* ranges;
  uint32_t F, BF, N;
  const uint32_t* lengths;     // [BF]
  const uint32_t* id_off;      // [BF+1]
  const uint32_t* ids;
  uint32_t* cnt;               // [N][BF]
  const uint32_t* send_off;    // [N*BF+1] (permute pass)
  uint32_t* err;
  uint32_t me;                 // local rank in the MP group
  // count pass: cnt[o][b] is also stored into owner o's receive lengths
  // peer_len.p[o] + me*BF + b; permute pass: id k of bag b owned by o goes
  // to peer_ids.p[o] + ids_adj[o] + send_off[o*BF+b] + k
  PeerPtrs peer_len;
  PeerPtrs peer_ids;
  int64_t ids_adj[kMaxPeers];
};
void launch_bucket_count(const BucketArgs& a, cudaStream_t st);
void launch_bucket_permute(const BucketArgs& a, cudaStream_t st);

// peer primitives (k_peer.cu)
void launch_peer_barrier(const PeerPtrs& flags, uint64_t* my_flags, uint32_t me, uint32_t n, uint64_t epoch,
                         uint32_t* err, cudaStream_t st);
void launch_publish_counts(const uint32_t* send_off, const uint64_t* eoff, uint32_t N, uint64_t BF, uint64_t batch,
                           const PeerPtrs& xcnt, uint32_t me, cudaStream_t st);

// update kernels (k_update.cu)
// streaming kernels (k_stream.cu): K2 lookup and K3b+K4 segment-reduce +
// fused update over the sorted pairs
struct StreamUpdateArgs {
  const uint32_t* keys;          // sorted slots (invalid = 0xffffffff, sorted last)
  const uint32_t* vals;          // gradient row offsets (float4 units), arrival order per slot
  uint64_t n;
  uint32_t n_slots;
  const FeatDev* feats;
  const uint32_t* vbase_sorted;
  const uint32_t* feat_of_vbase;
  uint32_t n_feat_owned;
  uint32_t uni_dim;              // every owned table has this dim (0: mixed dims)
  uint32_t max_d4;
  const float* grad;
  void* weights;
  float* moments;
  uint8_t* dirty;                // may be null
  double* part1;                 // level-1 range partials [n/C][max_dim]
  double* part2;                 // level-2 partials [n/(C*P)][max_dim]
  double* part3;                 // level-3 partials [n/(C*P*P)][max_dim]
  double inv_batch, eta, eps, c;
  double inv_c;                  // 1/c, exact when c_pow2
  int c_pow2;                    // c is a power of two: v/c == v*inv_c bit for bit
  int sgd;
  uint32_t* err;
  uint32_t* counters;            // [0] unique rows updated, [1] rows spanning ranges
  double* grad_dbg;              // debug: row gradients [U][max_dim] at head ordinals (null: off)
  const uint32_t* head_ord;      // debug: heads before each sorted position (scan_heads_u32)
  // M > 1 snapshot log (null: off): a row flushed while its dirty flag is
  // clear first saves its pre-update value (f32 row, moment at rf - 1) at
  // snap[pos], pos = snap_base + the head's sorted position (or, snap_dense,
  // its ordinal head_ord[position]), and snap_pos[slot] = pos (the host
  // reserves snap_base + n items, or + the update's rows when dense)
  float* snap;
  uint32_t* snap_pos;
  uint64_t snap_base;
  uint64_t snap_cap;
  uint32_t snap_rf;
  int snap_dense;
  // M > 1, the first update of a sync interval (null: off): each written
  // row's slot at its head ordinal (head_ord) -- the replica's ascending
  // dirty list, so the sync needs no scan of the dirty flags
  uint32_t* dirty_list;
};
// mean pooling, N = 1 (k_embed.cu): out = upstream with the columns of
// mean-pooled tables replaced by f32(f64(up) * (1/L_bag))
void launch_mean_prescale(const FeatDev* feats, uint32_t F, uint32_t B, uint32_t sum_dims, const uint32_t* bag_off,
                          const float* up, float* out, cudaStream_t st);
// MetricsRow moment statistics (k_metrics.cu)
void launch_moment_hist(const float* v, uint32_t n, int shift, uint32_t mask, uint32_t prefix, uint32_t* hist,
                        cudaStream_t st);
void launch_moment_sum(const float* v, uint32_t n, double* part, cudaStream_t st);
uint32_t moment_sum_blocks();
// device-side synthetic input (k_gen.cu): DataGenerator ids, data.cpp:85-136
struct GenArgs {
  uint64_t seed, step;
  uint32_t rank, B, F, per_sample;  // per_sample = sum_f L_f
  const uint32_t* cum;              // [F+1] exclusive prefix of L_f
  const uint32_t* rows;             // [F] table rows (num_ids)
  const uint64_t* cdf_off;          // [F] offset of table f's CDF in cdf
  const double* cdf;
  uint32_t* lengths;                // [B*F]
  uint32_t* ids;                    // [B*per_sample]
  uint64_t lane;                    // DataGenerator::Lane: 0 train, 1 eval
};
void launch_gen_batch(const GenArgs& a, cudaStream_t st);
void launch_gen_upstream(uint64_t seed, uint64_t step, uint32_t rank, uint32_t B, uint32_t F, const FeatDev* feats,
                         uint32_t sum_dims, uint32_t max_dim, float* out, cudaStream_t st);

size_t stream_partial_bytes(uint64_t n, uint32_t max_dim);
uint64_t stream_partial1_rows(uint64_t n);  // level-1 partial rows (part2 follows them)
uint64_t stream_partial2_rows(uint64_t n);  // level-2 partial rows (part3 follows them)
void launch_lookup_stream(const LookupArgs& a, int bf16, int max_dim, cudaStream_t st);
// N = 1: the lookup's (slot, upstream-row) sort pairs from the ids alone
void launch_emit_pairs(const FeatDev* feats, uint32_t F, uint32_t B, uint32_t sum_dims, const uint32_t* id_off,
                       const uint32_t* ids, uint32_t* keys, uint32_t* vals, cudaStream_t st);
void launch_update_stream(const StreamUpdateArgs& a, int bf16, cudaStream_t st);

// standalone fused row step on caller rows (s2d_adagrad_rows)
void launch_apply_rows(void* w, bool bf16, float* v, const uint32_t* order, const uint32_t* seg,
                       const uint32_t* seg_row, const double* delta, const double* moment, uint32_t nseg,
                       uint32_t dim, uint8_t* dirty, cudaStream_t st);
// gather rows of one table into f32 rows (fp32 or bf16 storage): out[i] =
// row rows_local[i] of the shard (local row index), v_out[i] its moment
void launch_gather_rows(const void* w, int bf16, const float* v, const uint32_t* rows_local, uint32_t n, uint32_t dim,
                        float* w_out, float* v_out, cudaStream_t st);
void launch_rows_adagrad(float* w, float* v, const double* g, double* lr, uint32_t n, uint32_t dim,
                         double eta, double eps, double c, int sgd, uint32_t* err, cudaStream_t st);

// replica sync kernels (k_sync.cu)
void launch_flag_count(const uint8_t* dirty, uint32_t n_slots, uint32_t* count, void* tmp, size_t tmp_bytes,
                       cudaStream_t st);
void launch_flag_write(const uint8_t* dirty, uint32_t n_slots, uint32_t* list, const void* tmp, cudaStream_t st);
// dirty[list[i]] = 0 for i < *count (count on the device, at most n)
void launch_clear_listed(uint8_t* dirty, const uint32_t* list, const uint32_t* count, uint32_t n, cudaStream_t st);
size_t flag_tmp_bytes(uint32_t n_slots);
void launch_mark_slots(const uint32_t* lists, uint64_t n, uint32_t n_slots, uint8_t* dirty, cudaStream_t st);
// Pair (M = 2) snapshot replica sync (k_sync.cu): each replica sends the
// rows it dirtied once -- the final mean for a row only it dirtied (from its
// row and the update's snapshot of the row's pre-interval value), its copy
// for a row both dirtied -- and the receiver stores / averages them.
void launch_pair_push(float* peer_stage, uint32_t me, const uint32_t* mine, const uint32_t* counts,
                      const uint32_t* theirs, uint32_t mine_n, const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat, const float* snap, const uint32_t* snap_pos,
                      uint32_t row_floats, void* weights, int bf16, float* moments, int sgd, uint32_t* n_both,
                      cudaStream_t st);
void launch_pair_recv(const float* stage, uint32_t me, const uint32_t* theirs, const uint32_t* counts,
                      uint32_t theirs_n, const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat, uint32_t row_floats, void* weights, int bf16,
                      float* moments, int sgd, cudaStream_t st);
void launch_pack_rows(const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat_owned, const uint32_t* list,
                      const uint32_t* count, const void* weights, int bf16, const float* moments,
                      uint32_t row_floats, float* packed, uint32_t max_rows, cudaStream_t st);
// P2P replica sync (k_sync.cu): push every union row into its slice owner's
// peer-mapped staging; the owner averages its slice into every replica's
// staging means; each replica scatters the means into its shard
void launch_p2p_push(const PeerPtrs& stage, uint32_t me, uint32_t M, const FeatDev* feats,
                     const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase, uint32_t n_feat,
                     const uint32_t* list, const uint32_t* count, uint32_t count_ub, const void* weights, int bf16,
                     const float* moments, uint32_t row_floats, uint64_t slice_cap, cudaStream_t st);
void launch_p2p_mean(const float* local, const PeerPtrs& means, uint32_t M, uint32_t me, const uint32_t* count,
                     uint32_t count_ub, uint32_t row_floats, uint64_t slice_cap, int sgd, cudaStream_t st);
void launch_p2p_scatter(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                        uint32_t n_feat, const uint32_t* list, const uint32_t* count, uint32_t count_ub,
                        const float* means, uint32_t row_floats, void* weights, int bf16, float* moments, int sgd,
                        cudaStream_t st);
void launch_mean_rows(const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat_owned, const uint32_t* list,
                      const uint32_t* count, const float* gathered, uint32_t M, uint32_t row_floats,
                      uint32_t rows_cap, void* weights, int bf16, float* moments, int sgd,
                      uint8_t* dirty, cudaStream_t st);

// host planning (host_plan.cpp)
void check_optimizer(const s2d_optimizer_config& c);
s2d_topology make_topology(uint32_t total, uint32_t groups);
std::vector<s2d_plan_entry> plan_greedy(const std::vector<s2d_table_load_profile>& profiles, uint32_t n,
                                        int strategy);
void validate_plan(const std::vector<s2d_plan_entry>& plan, uint32_t ranks_per_group,
                   const std::vector<s2d_table_load_profile>& profiles);
uint32_t plan_owner_of(const s2d_plan_entry* plan, uint32_t n, uint32_t table, uint32_t row);
double imbalance_ratio(const double* v, uint32_t n);
double effective_lr(double v, const s2d_optimizer_config& c);

}  // namespace s2d
