// C++ face of the C ABI in sparse2d_b200.h, shaped like the reference's C++
// API (include/sparse2d/planner.hpp, optimizer.hpp, topology.hpp) so a
// maintainer can swap the simulator's embedding phases for the B200 step
// without touching call sites: same argument meaning, and the status codes
// come back as the reference's exception types (std::invalid_argument,
// std::out_of_range, std::runtime_error; SURVEY.md 8(b) "Error conventions").
// Header-only; link libsparse2d_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparse2d_b200.h"

namespace sparse2d_b200 {

enum class ShardingStrategy : int32_t { kTableWise = S2D_TABLE_WISE, kRowWise = S2D_ROW_WISE };

// status -> the reference's exception type
inline void check(int rc) {
  if (rc == S2D_OK) return;
  const std::string m = s2d_last_error();
  switch (rc) {
    case S2D_ERANGE:
      throw std::out_of_range(m);
    case S2D_EINVAL:
    case S2D_ENONFINITE:
      throw std::invalid_argument(m);
    default:
      throw std::runtime_error(m);
  }
}

// Topology(total, groups) (topology.hpp:13-26, topology.cpp:7-17)
inline s2d_topology make_topology(uint32_t total_ranks, uint32_t groups) {
  s2d_topology t{};
  check(s2d_topology_init(total_ranks, groups, &t));
  return t;
}

// plan_greedy (planner.hpp:47-48)
inline std::vector<s2d_plan_entry> plan_greedy(const std::vector<s2d_table_load_profile>& profiles, uint32_t n,
                                               ShardingStrategy strategy) {
  std::vector<s2d_plan_entry> out((size_t)profiles.size() * (n ? n : 1));
  uint32_t k = 0;
  check(s2d_plan_greedy(profiles.data(), (uint32_t)profiles.size(), n, (int32_t)strategy, out.data(),
                        (uint32_t)out.size(), &k));
  out.resize(k);
  return out;
}

// validate_plan (planner.cpp:91-123)
inline void validate_plan(const std::vector<s2d_plan_entry>& plan, uint32_t ranks_per_group,
                          const std::vector<s2d_table_load_profile>& profiles) {
  check(s2d_validate_plan(plan.data(), (uint32_t)plan.size(), ranks_per_group, profiles.data(),
                          (uint32_t)profiles.size()));
}

// ShardingPlan::owner_of (planner.cpp:20-28)
inline uint32_t owner_of(const std::vector<s2d_plan_entry>& plan, uint32_t table_id, uint32_t row) {
  uint32_t o = 0;
  check(s2d_plan_owner_of(plan.data(), (uint32_t)plan.size(), table_id, row, &o));
  return o;
}

// imbalance_ratio (planner.cpp:125-143)
inline double imbalance_ratio(const std::vector<double>& per_rank) {
  double r = 0;
  check(s2d_imbalance_ratio(per_rank.data(), (uint32_t)per_rank.size(), &r));
  return r;
}

// effective_lr (optimizer.cpp:61-63), with OptimizerConfig::validate
inline double effective_lr(double v, const s2d_optimizer_config& cfg) {
  double lr = 0;
  check(s2d_effective_lr(v, &cfg, &lr));
  return lr;
}

// adagrad_row_step (optimizer.hpp:52-53) on one row, through the device
// kernel of the fused update; returns the effective learning rate
inline double adagrad_row_step(std::vector<float>& w, float& v, const std::vector<double>& g,
                               const s2d_optimizer_config& cfg) {
  if (g.size() != w.size()) throw std::invalid_argument("g and w must have the same length");
  double lr = 0;
  check(s2d_adagrad_rows(&cfg, 1, (uint32_t)w.size(), w.data(), &v, g.data(), &lr));
  return lr;
}

// One rank's step engine (replaces the embedding phases of
// Trainer::Impl::run_step, trainer.cpp:615-663).  RAII over s2d_ctx.
class Engine {
 public:
  Engine(int device, uint32_t total_ranks, uint32_t groups, uint32_t rank, const uint8_t* nccl_id = nullptr) {
    check(s2d_ctx_create(device, total_ranks, groups, rank, nccl_id, &ctx_));
  }
  ~Engine() {
    if (ctx_) s2d_ctx_destroy(ctx_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void register_tables(const std::vector<s2d_table_desc>& tables, const std::vector<s2d_plan_entry>& plan,
                       int32_t dtype = S2D_F32) {
    check(s2d_register_tables(ctx_, tables.data(), (uint32_t)tables.size(), plan.data(), (uint32_t)plan.size(),
                              dtype));
  }
  void set_optimizer(const s2d_optimizer_config& cfg) { check(s2d_set_optimizer(ctx_, &cfg)); }
  void init_tables(uint64_t seed) { check(s2d_init_tables(ctx_, seed)); }
  void set_stream(void* cuda_stream) { check(s2d_ctx_set_stream(ctx_, cuda_stream)); }
  void set_strict(bool on) { check(s2d_ctx_set_strict(ctx_, on ? 1 : 0)); }
  void set_async_host(bool on) { check(s2d_ctx_set_async_host(ctx_, on ? 1 : 0)); }

  // forward: sample-major bags; mem = S2D_HOST | S2D_DEVICE for all buffers
  void lookup_forward(uint32_t batch, const uint32_t* lengths, const uint32_t* ids, uint64_t nnz, float* pooled,
                      int32_t mem) {
    check(s2d_lookup_forward(ctx_, batch, lengths, ids, nnz, pooled, mem));
  }
  void backward_update(const float* upstream, int32_t mem) { check(s2d_backward_update(ctx_, upstream, mem)); }
  void replica_sync() { check(s2d_replica_sync(ctx_)); }
  void synchronize() { check(s2d_synchronize(ctx_)); }

  // Trainer::save_tables / load_tables (trainer.cpp:875-896)
  void save_tables(const std::string& path) { check(s2d_save_tables(ctx_, path.c_str())); }
  void load_tables(const std::string& path) { check(s2d_load_tables(ctx_, path.c_str())); }

  void shard_read(uint32_t table, uint32_t lo, uint32_t hi, float* w, float* v) {
    check(s2d_shard_read(ctx_, table, lo, hi, w, v));
  }
  void shard_write(uint32_t table, uint32_t lo, uint32_t hi, const float* w, const float* v) {
    check(s2d_shard_write(ctx_, table, lo, hi, w, v));
  }
  // apply_row_update (src/embedding.cpp:108-129) for n rows in call order;
  // delta is n x dim doubles.  Throws std::out_of_range / std::invalid_argument.
  void apply_row_updates(uint32_t table, uint32_t n, const uint32_t* rows, const double* delta,
                         const double* new_moment) {
    check(s2d_apply_row_updates(ctx_, table, n, rows, delta, new_moment));
  }
  s2d_step_stats stats() {
    s2d_step_stats s{};
    check(s2d_get_step_stats(ctx_, &s));
    return s;
  }
  s2d_ctx* raw() const { return ctx_; }

 private:
  s2d_ctx* ctx_ = nullptr;
};

// Host-side table view (EmbeddingTable, include/sparse2d/embedding.hpp:12-23).
struct TableCopy {
  uint32_t rows = 0, dim = 0;
  std::vector<float> weights, moments;
  const float* row(uint32_t r) const { return weights.data() + (size_t)r * dim; }
};

// ShardRef (embedding.hpp:30-38) over a host table copy, and the
// function-level pool_ids (embedding.hpp:52-53), run on the device.
struct ShardView {
  const TableCopy* table = nullptr;
  uint32_t row_lo = 0, row_hi = 0;
};
inline void pool_ids(const std::vector<ShardView>& shards, const std::vector<uint32_t>& ids, float* out,
                     uint32_t table_id = 0) {
  if (shards.empty()) throw std::invalid_argument("empty shard set");
  const TableCopy& t = *shards.front().table;
  std::vector<uint32_t> lo, hi;
  for (const auto& s : shards) {
    lo.push_back(s.row_lo);
    hi.push_back(s.row_hi);
  }
  const uint64_t off[2] = {0, ids.size()};
  check(s2d_pool_ids(t.weights.data(), t.rows, t.dim, table_id, (uint32_t)shards.size(), lo.data(), hi.data(), 1,
                     off, ids.data(), out));
}

// aggregate_group_gradient (optimizer.hpp:23-44), run on the device.
struct RowGradient {
  uint32_t row = 0;
  std::vector<double> g;
  uint32_t sample_count = 0;
};
struct RowGradContribution {
  uint32_t row = 0;
  std::vector<double> grad;
};
inline std::vector<RowGradient> aggregate_group_gradient(const std::vector<RowGradContribution>& cs,
                                                         uint32_t group_batch_size, uint32_t dim) {
  std::vector<uint32_t> rows(cs.size());
  std::vector<double> g(cs.size() * (size_t)dim);
  for (size_t i = 0; i < cs.size(); ++i) {
    if (cs[i].grad.size() != dim) throw std::invalid_argument("gradient dim mismatch");
    rows[i] = cs[i].row;
    std::copy(cs[i].grad.begin(), cs[i].grad.end(), g.begin() + i * dim);
  }
  uint64_t n = 0;
  check(s2d_aggregate_group_gradient(rows.data(), g.data(), cs.size(), group_batch_size, dim, nullptr, nullptr,
                                     nullptr, 0, &n));
  std::vector<uint32_t> r(n), c(n);
  std::vector<double> og(n * (size_t)dim);
  if (n)
    check(s2d_aggregate_group_gradient(rows.data(), g.data(), cs.size(), group_batch_size, dim, r.data(), og.data(),
                                       c.data(), n, &n));
  std::vector<RowGradient> out(n);
  for (uint64_t k = 0; k < n; ++k) {
    out[k].row = r[k];
    out[k].g.assign(og.begin() + k * dim, og.begin() + (k + 1) * dim);
    out[k].sample_count = c[k];
  }
  return out;
}

// Host copy of one Mlp's parameters (model.hpp:56): w1 [hidden][in], b1,
// w2 [out][hidden], b2.
struct MlpCopy {
  uint32_t in = 0, hidden = 0, out = 0;
  std::vector<float> w1, b1, w2, b2;
};
struct RankModelCopy {
  MlpCopy dense_arch, over_arch;  // RankModel (model.hpp:80-83)
};

// Trainer (include/sparse2d/trainer.hpp:106-132) over s2d_trainer_*: the
// whole 2D mesh as virtual ranks of this process.  The upstream gradient
// comes from the device dense model (opts.dense_model = 1), set_upstream,
// or the synthetic generator.
class Trainer {
 public:
  explicit Trainer(const s2d_trainer_options& opts) : opts_(opts) { check(s2d_trainer_create(&opts, &t_)); }
  ~Trainer() {
    if (t_) s2d_trainer_destroy(t_);
  }
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  void set_upstream(s2d_upstream_fn fn, void* user) { check(s2d_trainer_set_upstream(t_, fn, user)); }
  void run() { check(s2d_trainer_run(t_)); }
  void step_n(uint64_t count) { check(s2d_trainer_step_n(t_, count)); }
  uint64_t steps_done() const {
    uint64_t n = 0;
    check(s2d_trainer_steps_done(t_, &n));
    return n;
  }
  std::vector<s2d_plan_entry> plan() const {
    uint32_t n = 0;
    check(s2d_trainer_plan(t_, nullptr, 0, &n));
    std::vector<s2d_plan_entry> out(n);
    check(s2d_trainer_plan(t_, out.data(), n, &n));
    return out;
  }
  std::vector<TableCopy> replica_tables(uint32_t group) const {
    std::vector<TableCopy> out(opts_.num_tables);
    for (uint32_t f = 0; f < opts_.num_tables; ++f) {
      TableCopy& t = out[f];
      t.rows = opts_.rows_per_table;
      t.dim = opts_.dim;
      t.weights.resize((size_t)t.rows * t.dim);
      t.moments.resize(t.rows);
      check(s2d_trainer_replica_table(t_, group, f, t.weights.data(), t.moments.data()));
    }
    return out;
  }
  std::vector<TableCopy> tables() const { return replica_tables(0); }
  void save_tables(const std::string& path) const { check(s2d_trainer_save_tables(t_, path.c_str())); }
  void load_tables(const std::string& path) { check(s2d_trainer_load_tables(t_, path.c_str())); }
  s2d_metrics_row metrics() const {
    s2d_metrics_row m{};
    check(s2d_trainer_metrics(t_, &m));
    return m;
  }
  // TrainResult::metrics so far and finalize()'s final_ne (dense model only)
  std::vector<s2d_train_metrics_row> metrics_rows() const {
    uint32_t n = 0;
    check(s2d_trainer_metrics_rows(t_, nullptr, 0, &n));
    std::vector<s2d_train_metrics_row> out(n);
    check(s2d_trainer_metrics_rows(t_, out.data(), n, &n));
    return out;
  }
  s2d_ne_report final_ne() {
    s2d_ne_report r{};
    check(s2d_trainer_final_ne(t_, &r));
    return r;
  }
  double last_loss() const {
    double x = 0;
    check(s2d_trainer_last_loss(t_, &x));
    return x;
  }
  RankModelCopy rank_model(uint32_t rank) const {
    RankModelCopy m;
    const uint32_t FD = opts_.num_tables * opts_.dim;
    MlpCopy* arch[2] = {&m.dense_arch, &m.over_arch};
    const uint32_t dims[2][3] = {{opts_.dense_dim, opts_.dense_hidden, opts_.dim},
                                 {FD + opts_.dim, opts_.over_hidden, 1}};
    for (int a = 0; a < 2; ++a) {
      MlpCopy& c = *arch[a];
      c.in = dims[a][0], c.hidden = dims[a][1], c.out = dims[a][2];
      c.w1.resize((size_t)c.hidden * c.in);
      c.b1.resize(c.hidden);
      c.w2.resize((size_t)c.out * c.hidden);
      c.b2.resize(c.out);
      check(s2d_trainer_rank_model(t_, rank, a, c.w1.data(), c.b1.data(), c.w2.data(), c.b2.data()));
    }
    return m;
  }

 private:
  s2d_trainer_options opts_;
  s2d_trainer* t_ = nullptr;
};

// Analytic helpers of the reference module (cost_model.hpp, trainer.hpp
// evaluate_ne, moment_analysis.hpp), same names.
inline double memory_overhead(double table_size_gb, uint32_t groups, uint32_t total_gpus) {
  double r = 0;
  check(s2d_memory_overhead(table_size_gb, groups, total_gpus, &r));
  return r;
}
inline double sync_latency(double table_size_gb, uint32_t groups, uint32_t total_gpus, double bw) {
  double r = 0;
  check(s2d_sync_latency(table_size_gb, groups, total_gpus, bw, &r));
  return r;
}
inline double qps_scaling_factor(double qps_base, double gpus_base, double qps_new, double gpus_new) {
  double r = 0;
  check(s2d_qps_scaling_factor(qps_base, gpus_base, qps_new, gpus_new, &r));
  return r;
}
inline double closed_form_ratio(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups) {
  double r = 0;
  check(s2d_closed_form_ratio(mu_norm, sigma, dim, batch, groups, &r));
  return r;
}
inline double recommend_c(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups) {
  double r = 0;
  check(s2d_recommend_c(mu_norm, sigma, dim, batch, groups, &r));
  return r;
}

}  // namespace sparse2d_b200
