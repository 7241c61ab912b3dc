// extern "C" boundary of libsparse2d_b200.so (include/sparse2d_b200.h).
// Exceptions never cross it: every entry point returns an S2D_* status and
// stores the message for s2d_last_error().
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ctx.h"

using s2d::Error;

namespace s2d {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace s2d

namespace {

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return S2D_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("allocation failed: ") + e.what();
    return S2D_ERUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return S2D_ERUNTIME;
  }
}

s2d::Ctx* as_ctx(s2d_ctx* c) {
  if (!c) throw Error(S2D_EINVAL, "null context");
  return reinterpret_cast<s2d::Ctx*>(c);
}

}  // namespace

namespace s2d {
void set_last_error(const char* m) { g_last_error = m ? m : ""; }
}  // namespace s2d

extern "C" {

const char* s2d_last_error(void) { return g_last_error.c_str(); }

const char* s2d_version(void) { return "sparse2d_b200 0.1.0 (sm_100a)"; }

int s2d_topology_init(uint32_t total_ranks, uint32_t groups, s2d_topology* out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    *out = s2d::make_topology(total_ranks, groups);
  });
}

int s2d_plan_greedy(const s2d_table_load_profile* profiles, uint32_t n_profiles, uint32_t n, int32_t strategy,
                    s2d_plan_entry* out, uint32_t cap, uint32_t* n_out) {
  return guarded([&] {
    std::vector<s2d_table_load_profile> p(profiles, profiles + n_profiles);
    auto plan = s2d::plan_greedy(p, n, strategy);
    if (n_out) *n_out = (uint32_t)plan.size();
    if (plan.size() > cap) throw Error(S2D_EINVAL, "plan output capacity too small");
    if (out) std::memcpy(out, plan.data(), plan.size() * sizeof(s2d_plan_entry));
  });
}

int s2d_validate_plan(const s2d_plan_entry* plan, uint32_t n_entries, uint32_t ranks_per_group,
                      const s2d_table_load_profile* profiles, uint32_t n_profiles) {
  return guarded([&] {
    s2d::validate_plan(std::vector<s2d_plan_entry>(plan, plan + n_entries), ranks_per_group,
                       std::vector<s2d_table_load_profile>(profiles, profiles + n_profiles));
  });
}

int s2d_plan_owner_of(const s2d_plan_entry* plan, uint32_t n_entries, uint32_t table_id, uint32_t row,
                      uint32_t* owner) {
  return guarded([&] { *owner = s2d::plan_owner_of(plan, n_entries, table_id, row); });
}

int s2d_imbalance_ratio(const double* per_rank, uint32_t n, double* out) {
  return guarded([&] { *out = s2d::imbalance_ratio(per_rank, n); });
}

int s2d_effective_lr(double v, const s2d_optimizer_config* cfg, double* out) {
  return guarded([&] {
    if (!cfg || !out) throw Error(S2D_EINVAL, "null argument");
    s2d::check_optimizer(*cfg);
    *out = s2d::effective_lr(v, *cfg);
  });
}

int s2d_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *out = n;
  });
}

int s2d_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw Error(S2D_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, 128);
  });
}

int s2d_ctx_create(int device, uint32_t total_ranks, uint32_t groups, uint32_t rank, const uint8_t* nccl_id,
                   s2d_ctx** out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    auto c = std::make_unique<s2d::Ctx>();
    c->create(device, total_ranks, groups, rank, nccl_id);
    *out = reinterpret_cast<s2d_ctx*>(c.release());
  });
}

struct s2d_hub {
  std::shared_ptr<s2d::LocalHub> hub;
};

int s2d_hub_create(uint32_t total_ranks, s2d_hub** out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    if (total_ranks == 0) throw Error(S2D_EINVAL, "total_ranks must be >= 1");
    *out = new s2d_hub{std::make_shared<s2d::LocalHub>(total_ranks)};
  });
}

int s2d_hub_destroy(s2d_hub* hub) {
  return guarded([&] { delete hub; });
}

int s2d_ctx_create_local(int device, uint32_t total_ranks, uint32_t groups, uint32_t rank, s2d_hub* hub,
                         s2d_ctx** out) {
  return guarded([&] {
    if (!out || !hub) throw Error(S2D_EINVAL, "null hub / output");
    auto c = std::make_unique<s2d::Ctx>();
    c->create(device, total_ranks, groups, rank, nullptr, hub->hub);
    *out = reinterpret_cast<s2d_ctx*>(c.release());
  });
}

int s2d_ctx_destroy(s2d_ctx* ctx) {
  return guarded([&] { delete reinterpret_cast<s2d::Ctx*>(ctx); });
}

int s2d_ctx_set_stream(s2d_ctx* ctx, void* cuda_stream) {
  return guarded([&] {
    auto* c = as_ctx(ctx);
    c->stream = cuda_stream ? reinterpret_cast<cudaStream_t>(cuda_stream) : c->own_stream;
  });
}

int s2d_ctx_set_strict(s2d_ctx* ctx, int strict) {
  return guarded([&] { as_ctx(ctx)->strict = strict != 0; });
}

int s2d_ctx_set_async_host(s2d_ctx* ctx, int async) {
  return guarded([&] { as_ctx(ctx)->async_host = async != 0; });
}

int s2d_register_tables(s2d_ctx* ctx, const s2d_table_desc* tables, uint32_t n_tables, const s2d_plan_entry* plan,
                        uint32_t n_entries, int32_t weight_dtype) {
  return guarded([&] { as_ctx(ctx)->register_tables(tables, n_tables, plan, n_entries, weight_dtype); });
}

int s2d_set_optimizer(s2d_ctx* ctx, const s2d_optimizer_config* cfg) {
  return guarded([&] {
    if (!cfg) throw Error(S2D_EINVAL, "null optimizer config");
    as_ctx(ctx)->set_optimizer(*cfg);
  });
}

int s2d_init_tables(s2d_ctx* ctx, uint64_t seed) {
  return guarded([&] { as_ctx(ctx)->init_tables(seed); });
}

int s2d_shard_write(s2d_ctx* ctx, uint32_t table, uint32_t row_lo, uint32_t row_hi, const float* w, const float* v) {
  return guarded([&] { as_ctx(ctx)->shard_io(table, row_lo, row_hi, const_cast<float*>(w), const_cast<float*>(v), true); });
}

int s2d_shard_read(s2d_ctx* ctx, uint32_t table, uint32_t row_lo, uint32_t row_hi, float* w, float* v) {
  return guarded([&] { as_ctx(ctx)->shard_io(table, row_lo, row_hi, w, v, false); });
}

int s2d_apply_row_updates(s2d_ctx* ctx, uint32_t table, uint32_t n_rows, const uint32_t* rows, const double* delta,
                          const double* new_moment) {
  return guarded([&] { as_ctx(ctx)->apply_row_updates(table, n_rows, rows, delta, new_moment); });
}

int s2d_save_tables(s2d_ctx* ctx, const char* path) {
  return guarded([&] { as_ctx(ctx)->save_tables(path); });
}

int s2d_load_tables(s2d_ctx* ctx, const char* path) {
  return guarded([&] { as_ctx(ctx)->load_tables(path); });
}

int s2d_gen_batch(s2d_ctx* ctx, uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, const double* zipf,
                  const uint32_t* ids_per_sample, uint32_t* lengths, uint32_t* ids, int32_t mem) {
  return guarded([&] { as_ctx(ctx)->gen_batch(seed, step, rank, batch, zipf, ids_per_sample, lengths, ids, mem); });
}

int s2d_shard_range(s2d_ctx* ctx, uint32_t table, uint32_t* row_lo, uint32_t* row_hi) {
  return guarded([&] {
    auto* c = as_ctx(ctx);
    if (table >= c->F) throw Error(S2D_EINVAL, "table out of range");
    *row_lo = c->feats[table].lo;
    *row_hi = c->feats[table].hi;
  });
}

int s2d_lookup_forward(s2d_ctx* ctx, uint32_t batch, const uint32_t* lengths, const uint32_t* ids, uint64_t nnz,
                       float* pooled, int32_t mem) {
  return guarded([&] { as_ctx(ctx)->lookup_forward(batch, lengths, ids, nnz, pooled, mem); });
}

int s2d_pooled_buffer(s2d_ctx* ctx, float** out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    *out = as_ctx(ctx)->pooled_buffer();
  });
}

int s2d_backward_update(s2d_ctx* ctx, const float* upstream, int32_t mem) {
  return guarded([&] { as_ctx(ctx)->backward_update(upstream, mem); });
}

int s2d_replica_sync(s2d_ctx* ctx) {
  return guarded([&] { as_ctx(ctx)->replica_sync(); });
}

int s2d_ctx_set_profiling(s2d_ctx* ctx, int on) {
  return guarded([&] {
    auto* c = as_ctx(ctx);
    c->phase_end();
    c->profile = on != 0;
    c->profile_hot_only = on == 2;
  });
}

int s2d_get_phase_times(s2d_ctx* ctx, double* ms, uint32_t* counts, uint32_t n) {
  return guarded([&] {
    if (n < 12) throw Error(S2D_EINVAL, "need room for at least the 12 step phases");
    double all_ms[s2d::kNumPhases];
    uint32_t all_cnt[s2d::kNumPhases];
    as_ctx(ctx)->phase_times(all_ms, all_cnt);
    for (uint32_t i = 0; i < n && i < (uint32_t)s2d::kNumPhases; ++i) {
      ms[i] = all_ms[i];
      if (counts) counts[i] = all_cnt[i];
    }
  });
}

uint64_t s2d_launch_count(void) { return s2d::g_launches.load(); }

int s2d_synchronize(s2d_ctx* ctx) {
  return guarded([&] { as_ctx(ctx)->synchronize_and_check(); });
}

int s2d_get_step_stats(s2d_ctx* ctx, s2d_step_stats* out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    auto* c = as_ctx(ctx);
    c->refresh_stats();
    *out = c->stats;
    out->host_wait_ns = c->host_wait_total_ns;
  });
}

int s2d_gen_upstream(s2d_ctx* ctx, uint64_t seed, uint64_t step, uint32_t rank, uint32_t batch, float* out,
                     int32_t mem) {
  return guarded([&] { as_ctx(ctx)->gen_upstream(seed, step, rank, batch, out, mem); });
}

int s2d_shard_gather(s2d_ctx* ctx, uint32_t table, uint32_t n_rows, const uint32_t* rows, float* w, float* v) {
  return guarded([&] { as_ctx(ctx)->gather_rows(table, n_rows, rows, w, v); });
}

int s2d_ctx_set_debug_grad(s2d_ctx* ctx, int on) {
  return guarded([&] { as_ctx(ctx)->debug_grad = on != 0; });
}

int s2d_metrics(s2d_ctx* ctx, s2d_metrics_row* out) {
  return guarded([&] {
    if (!out) throw Error(S2D_EINVAL, "null output");
    as_ctx(ctx)->metrics(out);
  });
}

int s2d_debug_read(s2d_ctx* ctx, int32_t which, void* out, uint64_t cap, uint64_t* n) {
  return guarded([&] { as_ctx(ctx)->debug_read(which, out, cap, n); });
}

int s2d_adagrad_rows(const s2d_optimizer_config* cfg, uint32_t n_rows, uint32_t dim, float* w, float* v,
                     const double* g, double* lr_out) {
  return guarded([&] {
    if (!cfg) throw Error(S2D_EINVAL, "null optimizer config");
    s2d::check_optimizer(*cfg);
    if (dim == 0 || dim > (uint32_t)s2d::kMaxDim) throw Error(S2D_EINVAL, "dim must be in [1, 512]");
    if (n_rows == 0) return;
    // rows are padded to a multiple of 4 columns with zero gradient
    const uint32_t dp = (dim + 3) / 4 * 4;
    std::vector<float> hw((size_t)n_rows * dp, 0.0f);
    std::vector<double> hg((size_t)n_rows * dp, 0.0);
    for (uint32_t r = 0; r < n_rows; ++r) {
      std::memcpy(&hw[(size_t)r * dp], w + (size_t)r * dim, dim * 4);
      std::memcpy(&hg[(size_t)r * dp], g + (size_t)r * dim, dim * 8);
    }
    float *dw, *dv;
    double *dg, *dlr;
    uint32_t* derr;
    S2D_CUDA(cudaMalloc(&dw, hw.size() * 4));
    S2D_CUDA(cudaMalloc(&dv, (size_t)n_rows * 4));
    S2D_CUDA(cudaMalloc(&dg, hg.size() * 8));
    S2D_CUDA(cudaMalloc(&dlr, (size_t)n_rows * 8));
    S2D_CUDA(cudaMalloc(&derr, 4));
    struct Free {
      void* p[5];
      ~Free() {
        for (void* q : p) s2d::dev_free(q);
      }
    } fr{{dw, dv, dg, dlr, derr}};
    S2D_CUDA(cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemcpy(dv, v, (size_t)n_rows * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemcpy(dg, hg.data(), hg.size() * 8, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemset(derr, 0, 4));
    s2d::launch_rows_adagrad(dw, dv, dg, dlr, n_rows, dp, cfg->eta, cfg->eps, cfg->c, cfg->variant == S2D_SGD, derr,
                             nullptr);
    uint32_t e = 0;
    S2D_CUDA(cudaMemcpy(&e, derr, 4, cudaMemcpyDeviceToHost));
    if (e & s2d::kErrNonfinite) throw Error(S2D_ENONFINITE, "nonfinite row gradient");
    S2D_CUDA(cudaMemcpy(hw.data(), dw, hw.size() * 4, cudaMemcpyDeviceToHost));
    S2D_CUDA(cudaMemcpy(v, dv, (size_t)n_rows * 4, cudaMemcpyDeviceToHost));
    if (lr_out) S2D_CUDA(cudaMemcpy(lr_out, dlr, (size_t)n_rows * 8, cudaMemcpyDeviceToHost));
    for (uint32_t r = 0; r < n_rows; ++r) std::memcpy(w + (size_t)r * dim, &hw[(size_t)r * dp], dim * 4);
  });
}

}  // extern "C"
