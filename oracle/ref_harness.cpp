// ref_harness.cpp -- drives the UNMODIFIED reference library (sources under
// /root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/)
// through its public API.  TEST/BASELINE INFRASTRUCTURE ONLY: it produces the
// golden vectors (tests/golden/make_golden.py), pins oracle/s2d_oracle.c, and
// is the CPU "reference" arm of bench.py.  No reference source is copied here.
//
// The only private reference logic restated here is the demand bucketing of
// trainer.cpp:283-313 (build_demand) and the per-owner split of the step
// (trainer.cpp:316-338, 372-390, 440-505, 547-596), composed from the public
// functions pool_ids, aggregate_group_gradient, adagrad_row_step,
// sgd_row_step, deterministic_mean_inplace, init_table, plan_greedy and
// DataGenerator.  The survey verified this composition reproduces
// Trainer::replica_tables bitwise.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sparse2d/config.hpp"
#include "sparse2d/cost_model.hpp"
#include "sparse2d/experiment.hpp"
#include "sparse2d/data.hpp"
#include "sparse2d/moment_analysis.hpp"
#include "sparse2d/embedding.hpp"
#include "sparse2d/model.hpp"
#include "sparse2d/optimizer.hpp"
#include "sparse2d/planner.hpp"
#include "sparse2d/topology.hpp"
#include "sparse2d/trainer.hpp"

using namespace sparse2d;

namespace {

thread_local std::string g_err;

// Static chunking of trainer.cpp:82-97.
void par_for(uint32_t n, uint32_t threads, const std::function<void(uint32_t)>& fn) {
  if (threads <= 1 || n <= 1) {
    for (uint32_t i = 0; i < n; ++i) fn(i);
    return;
  }
  const uint32_t workers = std::min(threads, n);
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(workers);
  for (uint32_t w = 0; w < workers; ++w) {
    pool.emplace_back([&, w] {
      try {
        for (uint32_t i = w; i < n; i += workers) fn(i);
      } catch (...) {
        errs[w] = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

struct Cfg {
  uint32_t F, N, B;
  const uint32_t* rows;
  const uint32_t* dims;
  uint32_t n_entries;
  const uint32_t* plan;
  double eta, eps, c;
  int sgd;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// init_table (embedding.cpp:17-37) restricted to rows [lo, hi).
int ref_init_rows(uint32_t table_id, uint32_t rows, uint32_t lo, uint32_t hi, uint32_t dim,
                  uint64_t seed, float* out) {
  try {
    EmbeddingTable t = init_table(table_id, rows, dim, seed);
    std::memcpy(out, t.row(lo), sizeof(float) * (size_t)(hi - lo) * dim);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// aggregate_group_gradient (optimizer.cpp:25-59) as is: contributions
// (rows[i], grads[i*dim ..]); out_rows / out_g / out_count hold the result
// (capacity n), *n_out its length.
int ref_aggregate(const uint32_t* rows, const double* grads, uint32_t n, uint32_t group_batch, uint32_t dim,
                  uint32_t* out_rows, double* out_g, uint32_t* out_count, uint32_t* n_out) {
  try {
    std::vector<RowGradContribution> cs(n);
    for (uint32_t i = 0; i < n; ++i) cs[i] = {rows[i], std::span<const double>(grads + (size_t)i * dim, dim)};
    const auto out = aggregate_group_gradient(cs, group_batch, dim);
    *n_out = (uint32_t)out.size();
    for (size_t k = 0; k < out.size(); ++k) {
      out_rows[k] = out[k].row;
      out_count[k] = out[k].sample_count;
      std::memcpy(out_g + k * dim, out[k].g.data(), dim * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_pool_ids(const float* w, uint32_t rows, uint32_t dim, uint32_t n_shards,
                 const uint32_t* lo_hi, const uint32_t* ids, uint32_t n_ids, float* out) {
  EmbeddingTable t;
  t.rows = rows;
  t.dim = dim;
  t.weights.assign(w, w + (size_t)rows * dim);
  t.moments.assign(rows, 0.0f);
  std::vector<ShardRef> shards;
  for (uint32_t s = 0; s < n_shards; ++s) shards.push_back({&t, lo_hi[2 * s], lo_hi[2 * s + 1]});
  try {
    pool_ids(shards, std::span<const uint32_t>(ids, n_ids), out);
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_apply_row_update(float* w, float* v, uint32_t rows, uint32_t lo, uint32_t hi, uint32_t dim,
                         uint32_t row, const double* delta, double new_moment) {
  EmbeddingTable t;
  t.rows = rows;
  t.dim = dim;
  t.weights.assign(w, w + (size_t)rows * dim);
  t.moments.assign(v, v + rows);
  try {
    apply_row_update(ShardRef{&t, lo, hi}, row, std::span<const double>(delta, dim), new_moment);
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  std::copy(t.weights.begin(), t.weights.end(), w);
  std::copy(t.moments.begin(), t.moments.end(), v);
  return 0;
}

double ref_adagrad_row_step(float* w, float* v, const double* g, uint32_t dim, double eta,
                            double eps, double c, int* err) {
  OptimizerConfig cfg{eta, eps, c, OptimizerVariant::RowWiseAdagrad};
  try {
    *err = 0;
    return adagrad_row_step(std::span<float>(w, dim), *v, std::span<const double>(g, dim), cfg);
  } catch (const std::exception& e) {
    g_err = e.what();
    *err = -3;
    return 0.0;
  }
}

double ref_effective_lr(double v, double eta, double eps, double c) {
  OptimizerConfig cfg{eta, eps, c, OptimizerVariant::RowWiseAdagrad};
  return effective_lr(v, cfg);
}

int ref_plan_greedy(uint32_t n_tables, const uint32_t* table_ids, const double* lookups,
                    const uint64_t* num_rows, uint32_t n, int strategy, uint32_t* out) {
  try {
    std::vector<TableLoadProfile> p;
    for (uint32_t t = 0; t < n_tables; ++t)
      p.push_back({table_ids[t], num_rows[t] * 4, lookups[t], num_rows[t]});
    auto plan = plan_greedy(p, n, strategy ? ShardingStrategy::RowWise : ShardingStrategy::TableWise);
    validate_plan(plan, p);
    for (size_t i = 0; i < plan.entries.size(); ++i) {
      out[4 * i] = plan.entries[i].table_id;
      out[4 * i + 1] = plan.entries[i].row_lo;
      out[4 * i + 2] = plan.entries[i].row_hi;
      out[4 * i + 3] = plan.entries[i].local_rank;
    }
    return (int)plan.entries.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Ids of one rank's batch from the reference DataGenerator (data.cpp:115-147),
// uniform tables (FeatureSpec{f, rows, zipf, L}).  out_ids: B*F*L.
int ref_gen_batch_ids(uint64_t seed, uint64_t step, uint32_t rank, uint32_t F, uint32_t rows,
                      double zipf, uint32_t L, uint32_t B, uint32_t* out_ids) {
  try {
    std::vector<FeatureSpec> specs;
    for (uint32_t f = 0; f < F; ++f) specs.push_back({f, rows, zipf, L});
    DataGenerator gen(specs, DataParams{}, seed);
    MiniBatch mb = gen.gen_batch(step, rank, B);
    size_t k = 0;
    for (uint32_t s = 0; s < B; ++s)
      for (uint32_t f = 0; f < F; ++f)
        for (uint32_t id : mb.samples[s].ids[f]) out_ids[k++] = id;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// gen_batch ids with per-table rows / Zipf exponent / ids_per_sample
// (DataGenerator, data.cpp:70-136), sample-major (s, f, draw) order.
int ref_gen_batch_ids_tables(uint64_t seed, uint64_t step, uint32_t rank, uint32_t F, const uint32_t* rows,
                             const double* zipf, const uint32_t* L, uint32_t B, uint32_t* out_ids) {
  try {
    std::vector<FeatureSpec> specs;
    for (uint32_t f = 0; f < F; ++f) specs.push_back({f, rows[f], zipf[f], L[f]});
    DataGenerator gen(specs, DataParams{}, seed);
    MiniBatch mb = gen.gen_batch(step, rank, B);
    size_t k = 0;
    for (uint32_t s = 0; s < B; ++s)
      for (uint32_t f = 0; f < F; ++f)
        for (uint32_t id : mb.samples[s].ids[f]) out_ids[k++] = id;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_deterministic_mean(uint32_t m, float* const* reps, size_t len) {
  deterministic_mean_inplace(std::span<float* const>(reps, m), len);
}

// One MP group's step through the public API (see file header).  Same
// argument contract as or_group_step in oracle/s2d_oracle.c; `threads`
// parallelises over (owner, table) with the reference's static chunking.
int ref_group_step(uint32_t F, uint32_t N, uint32_t B, const uint32_t* rows, const uint32_t* dims,
                   uint32_t n_entries, const uint32_t* plan, double eta, double eps, double c,
                   int sgd, const uint32_t* const* lengths, const uint32_t* const* ids,
                   const float* const* upstream, float* const* pooled, float* w, float* v,
                   uint8_t* dirty, uint32_t threads, double* compute_seconds) {
  try {
    const uint32_t BF = B * F;
    OptimizerConfig opt{eta, eps, c, sgd ? OptimizerVariant::Sgd : OptimizerVariant::RowWiseAdagrad};
    opt.validate();
    // Wrap the flat replica as EmbeddingTables (copy in, copy out).
    std::vector<EmbeddingTable> tables(F);
    std::vector<size_t> woff(F + 1, 0), voff(F + 1, 0), coff(F + 1, 0);
    for (uint32_t f = 0; f < F; ++f) {
      woff[f + 1] = woff[f] + (size_t)rows[f] * dims[f];
      voff[f + 1] = voff[f] + rows[f];
      coff[f + 1] = coff[f] + dims[f];
    }
    const size_t sumD = coff[F];
    par_for(F, threads, [&](uint32_t f) {
      tables[f].table_id = f;
      tables[f].rows = rows[f];
      tables[f].dim = dims[f];
      tables[f].weights.assign(w + woff[f], w + woff[f + 1]);
      tables[f].moments.assign(v + voff[f], v + voff[f + 1]);
    });
    // timed region: everything between wrapping the replica and unwrapping it
    const auto t_begin = std::chrono::steady_clock::now();
    // Shard ranges per (table, owner) from the plan.
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> range(F, std::vector<std::pair<uint32_t, uint32_t>>(N, {0, 0}));
    for (uint32_t e = 0; e < n_entries; ++e) range[plan[4 * e]][plan[4 * e + 3]] = {plan[4 * e + 1], plan[4 * e + 2]};
    auto owner_of = [&](uint32_t f, uint32_t id) -> uint32_t {
      for (uint32_t o = 0; o < N; ++o)
        if (id >= range[f][o].first && id < range[f][o].second) return o;
      throw std::out_of_range("lookup id " + std::to_string(id) + " outside shard ranges of table " + std::to_string(f));
    };
    // build_demand (trainer.cpp:283-313), restated.
    struct Entry {
      uint32_t n, s, f, begin, count;
    };
    std::vector<std::vector<Entry>> entries(N);
    std::vector<std::vector<uint32_t>> dem_ids(N);
    std::vector<std::vector<uint32_t>> mask(N, std::vector<uint32_t>(BF, 0));
    for (uint32_t n = 0; n < N; ++n) {
      size_t off = 0;
      for (uint32_t s = 0; s < B; ++s) {
        for (uint32_t f = 0; f < F; ++f) {
          const uint32_t b = s * F + f;
          const uint32_t* bag = ids[n] + off;
          const uint32_t L = lengths[n][b];
          off += L;
          uint32_t m = 0;
          for (uint32_t o = 0; o < N; ++o) {
            const uint32_t begin = (uint32_t)dem_ids[o].size();
            uint32_t cnt = 0;
            for (uint32_t k = 0; k < L; ++k) {
              if (owner_of(f, bag[k]) == o) {
                dem_ids[o].push_back(bag[k]);
                ++cnt;
              }
            }
            if (cnt) {
              entries[o].push_back({n, s, f, begin, cnt});
              m |= 1u << o;
            }
          }
          mask[n][b] = m;
        }
      }
    }
    // owner_lookup via pool_ids over the owner's single shard: exactly the
    // f32-rounded f64 partial of trainer.cpp:324-335.
    std::vector<std::vector<std::vector<float>>> send(N, std::vector<std::vector<float>>(N));  // [o][n]
    for (uint32_t o = 0; o < N; ++o) {
      std::vector<size_t> first(entries[o].size() + 1, 0);
      for (uint32_t n = 0; n < N; ++n) {
        size_t cnt = 0;
        for (auto& e : entries[o])
          if (e.n == n) cnt += dims[e.f];
        send[o][n].resize(cnt);
      }
      // position of each entry inside send[o][n]
      std::vector<size_t> pos(entries[o].size());
      std::vector<size_t> fill(N, 0);
      for (size_t i = 0; i < entries[o].size(); ++i) {
        pos[i] = fill[entries[o][i].n];
        fill[entries[o][i].n] += dims[entries[o][i].f];
      }
      par_for((uint32_t)std::min<size_t>(entries[o].size(), 1u << 30), threads, [&](uint32_t i) {
        const Entry& e = entries[o][i];
        ShardRef sh{&tables[e.f], range[e.f][o].first, range[e.f][o].second};
        pool_ids(std::span<const ShardRef>(&sh, 1),
                 std::span<const uint32_t>(dem_ids[o].data() + e.begin, e.count),
                 send[o][e.n].data() + pos[i]);
      });
    }
    // requester combine (trainer.cpp:372-390)
    par_for(N, threads, [&](uint32_t n) {
      std::vector<size_t> cursor(N, 0);
      std::vector<double> pool(512);
      for (uint32_t s = 0; s < B; ++s)
        for (uint32_t f = 0; f < F; ++f) {
          const uint32_t D = dims[f];
          std::fill(pool.begin(), pool.begin() + D, 0.0);
          for (uint32_t o = 0; o < N; ++o) {
            if (!(mask[n][s * F + f] & (1u << o))) continue;
            const float* p = send[o][n].data() + cursor[o];
            for (uint32_t j = 0; j < D; ++j) pool[j] += (double)p[j];
            cursor[o] += D;
          }
          float* out = pooled[n] + (size_t)s * sumD + coff[f];
          for (uint32_t j = 0; j < D; ++j) out[j] = (float)pool[j];
        }
    });
    if (!upstream) return 0;  // forward only (the pooled rows, replica untouched)
    // grad payloads (trainer.cpp:440-457) and owner_update (459-505) with
    // aggregate_group_gradient + adagrad_row_step / sgd_row_step.
    // Per (owner, table) work items, static chunking.
    std::vector<std::vector<size_t>> grad_pos(N);  // per owner entry: requester-local float offset
    for (uint32_t o = 0; o < N; ++o) {
      std::vector<size_t> fill(N, 0);
      grad_pos[o].resize(entries[o].size());
      for (size_t i = 0; i < entries[o].size(); ++i) {
        grad_pos[o][i] = fill[entries[o][i].n];
        fill[entries[o][i].n] += dims[entries[o][i].f];
      }
    }
    const uint32_t group_batch = N * B;
    std::vector<int> bad(N * F, 0);
    par_for(N * F, threads, [&](uint32_t item) {
      const uint32_t o = item / F, f = item % F;
      const uint32_t D = dims[f];
      std::vector<double> gpool;
      size_t cnt = 0;
      for (auto& e : entries[o])
        if (e.f == f) cnt += 1;
      gpool.reserve(cnt * D);
      std::vector<RowGradContribution> contribs;
      for (size_t i = 0; i < entries[o].size(); ++i) {
        const Entry& e = entries[o][i];
        if (e.f != f) continue;
        // the requester's upstream row for bag (s, f): what send_grad carries
        const float* g = upstream[e.n] + (size_t)e.s * sumD + coff[f];
        const size_t base = gpool.size();
        for (uint32_t j = 0; j < D; ++j) gpool.push_back((double)g[j]);
        for (uint32_t k = 0; k < e.count; ++k)
          contribs.push_back({dem_ids[o][e.begin + k], std::span<const double>(gpool.data() + base, D)});
      }
      if (contribs.empty()) return;
      auto grads = aggregate_group_gradient(contribs, group_batch, D);
      EmbeddingTable& t = tables[f];
      for (const auto& rg : grads) {
        float* wr = t.row(rg.row);
        if (sgd) {
          sgd_row_step(std::span<float>(wr, D), rg.g, opt);
        } else {
          adagrad_row_step(std::span<float>(wr, D), t.moments[rg.row], rg.g, opt);
        }
        if (dirty) dirty[voff[f] + rg.row] = 1;
      }
    });
    if (compute_seconds)
      *compute_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count();
    par_for(F, threads, [&](uint32_t f) {
      std::memcpy(w + woff[f], tables[f].weights.data(), sizeof(float) * (woff[f + 1] - woff[f]));
      std::memcpy(v + voff[f], tables[f].moments.data(), sizeof(float) * (voff[f + 1] - voff[f]));
    });
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return -2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// sync_replicas (trainer.cpp:547-596) via deterministic_mean_inplace per
// dirty row (weights, then moments unless SGD).
int ref_sync(uint32_t M, uint32_t F, const uint32_t* rows, const uint32_t* dims, int sgd,
             float* const* w, float* const* v, uint8_t* const* dirty) {
  size_t woff = 0, voff = 0;
  std::vector<float*> ptr(M);
  for (uint32_t f = 0; f < F; ++f) {
    const uint32_t D = dims[f];
    for (uint32_t r = 0; r < rows[f]; ++r) {
      bool any = false;
      for (uint32_t g = 0; g < M; ++g) any |= dirty[g][voff + r] != 0;
      if (!any) continue;
      for (uint32_t g = 0; g < M; ++g) ptr[g] = w[g] + woff + (size_t)r * D;
      deterministic_mean_inplace(ptr, D);
      if (!sgd) {
        for (uint32_t g = 0; g < M; ++g) ptr[g] = v[g] + voff + r;
        deterministic_mean_inplace(ptr, 1);
      }
      for (uint32_t g = 0; g < M; ++g) dirty[g][voff + r] = 0;
    }
    woff += (size_t)rows[f] * D;
    voff += rows[f];
  }
  return 0;
}

// save_checkpoint / load_checkpoint (embedding.cpp:133-219) on the flat
// replica layout (table f = table_id f).  0 = ok, -1 = error (ref_last_error).
int ref_save_checkpoint(const char* path, uint32_t F, const uint32_t* rows, const uint32_t* dims, const float* w,
                        const float* v) {
  try {
    std::vector<EmbeddingTable> tables(F);
    std::vector<const EmbeddingTable*> ptrs(F);
    size_t woff = 0, voff = 0;
    for (uint32_t f = 0; f < F; ++f) {
      EmbeddingTable& t = tables[f];
      t.table_id = f;
      t.rows = rows[f];
      t.dim = dims[f];
      t.weights.assign(w + woff, w + woff + (size_t)rows[f] * dims[f]);
      t.moments.assign(v + voff, v + voff + rows[f]);
      woff += (size_t)rows[f] * dims[f];
      voff += rows[f];
      ptrs[f] = &t;
    }
    save_checkpoint(path, ptrs);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_load_checkpoint(const char* path, uint32_t F, const uint32_t* rows, const uint32_t* dims, float* w,
                        float* v) {
  try {
    const auto tables = load_checkpoint(path);
    if (tables.size() != F) throw std::runtime_error("checkpoint table count mismatch");
    size_t woff = 0, voff = 0;
    for (uint32_t f = 0; f < F; ++f) {
      const EmbeddingTable& t = tables[f];
      if (t.rows != rows[f] || t.dim != dims[f]) throw std::runtime_error("checkpoint shape mismatch");
      std::copy(t.weights.begin(), t.weights.end(), w + woff);
      std::copy(t.moments.begin(), t.moments.end(), v + voff);
      woff += (size_t)rows[f] * dims[f];
      voff += rows[f];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- the real Trainer, and the step restated on the public API --------------

// TrainerOptions subset (include/sparse2d/trainer.hpp:47-70) the pin needs.
struct RefTrainerOpts {
  uint32_t T, M, F, rows, dim, dense_hidden, over_hidden, dense_dim, ids_per_sample, B;
  int32_t strategy;  // 0 table-wise, 1 row-wise
  double zipf, eta, eps, c;
  int32_t sgd;
  uint32_t sync_interval;
  uint64_t data_seed, init_seed, eval_seed;
  uint32_t steps;
};

static TrainerOptions make_options(const RefTrainerOpts& o) {
  TrainerOptions t;
  t.topo = Topology(o.T, o.M);
  t.model.num_tables = o.F;
  t.model.rows_per_table = o.rows;
  t.model.dim = o.dim;
  t.model.dense_hidden = o.dense_hidden;
  t.model.over_hidden = o.over_hidden;
  t.data.dense_dim = o.dense_dim;
  t.opt = OptimizerConfig{o.eta, o.eps, o.c, o.sgd ? OptimizerVariant::Sgd : OptimizerVariant::RowWiseAdagrad};
  t.strategy = o.strategy ? ShardingStrategy::RowWise : ShardingStrategy::TableWise;
  t.zipf_exponent = o.zipf;
  t.ids_per_sample = o.ids_per_sample;
  t.per_rank_batch = o.B;
  t.steps = o.steps;
  t.sync_interval = o.sync_interval;
  t.data_seed = o.data_seed;
  t.init_seed = o.init_seed;
  t.eval_seed = o.eval_seed;
  t.eval_samples = 512;
  t.threads = 1;
  return t;
}

// Trainer(opts).step_n(steps) (trainer.hpp:106-132); replica_tables(g) into
// w_out[g] (F*rows*dim) / v_out[g] (F*rows); the plan into plan_out (4 u32
// per entry, *n_plan entries, cap >= F*N).
int ref_trainer_run(const RefTrainerOpts* o, float* const* w_out, float* const* v_out, uint32_t* plan_out,
                    uint32_t* n_plan) {
  try {
    Trainer tr(make_options(*o));
    tr.step_n(o->steps);
    for (uint32_t g = 0; g < o->M; ++g) {
      const auto tabs = tr.replica_tables(g);
      for (uint32_t f = 0; f < o->F; ++f) {
        std::memcpy(w_out[g] + (size_t)f * o->rows * o->dim, tabs[f]->weights.data(),
                    sizeof(float) * (size_t)o->rows * o->dim);
        std::memcpy(v_out[g] + (size_t)f * o->rows, tabs[f]->moments.data(), sizeof(float) * o->rows);
      }
    }
    const auto& pl = tr.plan();
    *n_plan = (uint32_t)pl.entries.size();
    for (size_t i = 0; i < pl.entries.size(); ++i) {
      plan_out[4 * i] = pl.entries[i].table_id;
      plan_out[4 * i + 1] = pl.entries[i].row_lo;
      plan_out[4 * i + 2] = pl.entries[i].row_hi;
      plan_out[4 * i + 3] = pl.entries[i].local_rank;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Trainer(opts with eval_cadence 1).step_n(steps) with the dense model's
// outputs as well: replicas as ref_trainer_run, rank_model(0)'s parameters
// concatenated into mlp_out (dense_arch w1 b1 w2 b2, over_arch w1 b1 w2 b2)
// and every step's MetricsRow into rows_out[steps][6] (step, loss, ne,
// eff_lr_p50, eff_lr_p99, v_mean).
int ref_trainer_run_model(const RefTrainerOpts* o, float* const* w_out, float* const* v_out, float* mlp_out,
                          double* loss_out) {
  try {
    TrainerOptions t = make_options(*o);
    t.eval_cadence = 1;
    Trainer tr(t);
    tr.step_n(o->steps);
    for (uint32_t g = 0; g < o->M; ++g) {
      const auto tabs = tr.replica_tables(g);
      for (uint32_t f = 0; f < o->F; ++f) {
        std::memcpy(w_out[g] + (size_t)f * o->rows * o->dim, tabs[f]->weights.data(),
                    sizeof(float) * (size_t)o->rows * o->dim);
        std::memcpy(v_out[g] + (size_t)f * o->rows, tabs[f]->moments.data(), sizeof(float) * o->rows);
      }
    }
    const RankModel& m = tr.rank_model(0);
    float* p = mlp_out;
    for (const Mlp* a : {&m.dense_arch, &m.over_arch})
      for (const std::vector<float>* v : {&a->w1, &a->b1, &a->w2, &a->b2}) {
        std::memcpy(p, v->data(), v->size() * sizeof(float));
        p += v->size();
      }
    const TrainResult res = tr.finalize();
    for (size_t i = 0; i < res.metrics.size() && i < o->steps; ++i) {
      const MetricsRow& m = res.metrics[i];
      const double row[6] = {(double)m.step, m.loss, m.ne, m.eff_lr_p50, m.eff_lr_p99, m.v_mean};
      std::memcpy(loss_out + 6 * i, row, sizeof(row));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference module's train_toy (bindings/module.cpp:148-163): run_train
// of ExperimentConfig + {keys[i]: vals[i]} overrides; final NE, baseline
// CTR and the 16-hex-digit config hash (hash_out, >= 17 bytes).
int ref_train_toy(uint32_t n, const char* const* keys, const char* const* vals, double* final_ne, double* baseline_ctr,
                  char* hash_out) {
  try {
    ExperimentConfig cfg;
    for (uint32_t i = 0; i < n; ++i) cfg.set(keys[i], vals[i]);
    const RunArtifact art = run_train(cfg);
    *final_ne = art.result.final_ne.ne;
    *baseline_ctr = art.result.final_ne.baseline_ctr;
    std::snprintf(hash_out, 17, "%s", art.config_hash.c_str());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The same training loop composed from the public API (run_step,
// trainer.cpp:615-663): DataGenerator batches, the embedding phases through
// ref_group_step (forward, then backward with the MLP's f32 wire gradient),
// the per-rank MLPs (init_rank_model, Mlp forward / backward_dx /
// accumulate_grads / apply_sgd: pool_and_forward 366-402, backward_rank
// 404-438, dense_sync_and_apply 507-545) and the replica sync (ref_sync,
// 547-596).  Records every step's per-rank inputs of the embedding path:
// rec_len[step][rank][B*F], rec_ids[step][rank][B*F*L],
// rec_up[step][rank][B][F*D], rec_pooled likewise (any may be NULL).
int ref_restated_run(const RefTrainerOpts* o, uint32_t* rec_len, uint32_t* rec_ids, float* rec_up,
                     float* rec_pooled, float* const* w_out, float* const* v_out) {
  try {
    const TrainerOptions t = make_options(*o);
    const uint32_t T = o->T, M = o->M, N = T / M, F = o->F, D = o->dim, B = o->B, L = o->ids_per_sample;
    DataGenerator gen(t.feature_specs(), t.data, t.data_seed, t.eval_seed);
    std::vector<TableLoadProfile> prof;
    for (const auto& s : gen.specs()) prof.push_back(profile_from_spec(s, D, N * B));
    const ShardingPlan plan = plan_greedy(prof, N, t.strategy);
    std::vector<uint32_t> pl;
    for (const auto& e : plan.entries) pl.insert(pl.end(), {e.table_id, e.row_lo, e.row_hi, e.local_rank});
    const uint32_t ne = (uint32_t)plan.entries.size();
    std::vector<uint32_t> rows(F, o->rows), dims(F, D);
    const size_t rf = (size_t)F * o->rows * D, rv = (size_t)F * o->rows;
    std::vector<std::vector<float>> ws(M, std::vector<float>(rf)), vs(M, std::vector<float>(rv, 0.0f));
    std::vector<std::vector<uint8_t>> dirty(M, std::vector<uint8_t>(rv, 0));
    for (uint32_t f = 0; f < F; ++f) {
      const EmbeddingTable tb = init_table(f, o->rows, D, t.init_seed);
      for (uint32_t g = 0; g < M; ++g) std::memcpy(ws[g].data() + (size_t)f * o->rows * D, tb.weights.data(), sizeof(float) * (size_t)o->rows * D);
    }
    std::vector<RankModel> models;
    for (uint32_t r = 0; r < T; ++r) models.push_back(init_rank_model(t.model, t.data.dense_dim, t.init_seed));
    const uint32_t oin = t.model.over_in(), dh = t.model.dense_hidden, oh = t.model.over_hidden;
    const size_t up_n = (size_t)B * F * D;
    MlpGrads dense_mean, over_mean;
    dense_mean.resize(models[0].dense_arch.dims());
    over_mean.resize(models[0].over_arch.dims());
    for (uint32_t step = 0; step < o->steps; ++step) {
      std::vector<MiniBatch> mb(T);
      std::vector<std::vector<uint32_t>> len(T, std::vector<uint32_t>((size_t)B * F)), ids(T);
      for (uint32_t r = 0; r < T; ++r) {
        gen.gen_batch_into(mb[r], step, r, B);
        for (uint32_t s = 0; s < B; ++s)
          for (uint32_t f = 0; f < F; ++f) {
            len[r][(size_t)s * F + f] = (uint32_t)mb[r].samples[s].ids[f].size();
            ids[r].insert(ids[r].end(), mb[r].samples[s].ids[f].begin(), mb[r].samples[s].ids[f].end());
          }
      }
      // forward of every group (pooled rows, pre-update replica)
      std::vector<std::vector<float>> pooled(T, std::vector<float>(up_n)), upstream(T, std::vector<float>(up_n));
      for (uint32_t g = 0; g < M; ++g) {
        std::vector<const uint32_t*> lp(N), ip(N);
        std::vector<float*> pp(N);
        for (uint32_t n = 0; n < N; ++n) {
          lp[n] = len[g * N + n].data();
          ip[n] = ids[g * N + n].data();
          pp[n] = pooled[g * N + n].data();
        }
        if (ref_group_step(F, N, B, rows.data(), dims.data(), ne, pl.data(), t.opt.eta, t.opt.eps, t.opt.c,
                           o->sgd, lp.data(), ip.data(), nullptr, pp.data(), ws[g].data(), vs[g].data(), nullptr, 1,
                           nullptr))
          return -1;
      }
      // per rank: MLP forward + backward -> f32 wire gradient
      struct Act {
        std::vector<float> over_in, dense_hidden, over_hidden;
        std::vector<double> probs, dh_over, dh_dense, ddense_out;
      };
      std::vector<Act> act(T);
      for (uint32_t r = 0; r < T; ++r) {
        Act& a = act[r];
        const RankModel& m = models[r];
        a.over_in.assign((size_t)B * oin, 0.f);
        a.dense_hidden.assign((size_t)B * dh, 0.f);
        a.over_hidden.assign((size_t)B * oh, 0.f);
        a.probs.assign(B, 0.0);
        a.dh_over.assign((size_t)B * oh, 0.0);
        a.dh_dense.assign((size_t)B * dh, 0.0);
        a.ddense_out.assign((size_t)B * D, 0.0);
        std::vector<double> dx(oin);
        for (uint32_t s = 0; s < B; ++s) {
          float* oi = &a.over_in[(size_t)s * oin];
          std::memcpy(oi, &pooled[r][(size_t)s * F * D], sizeof(float) * F * D);
          m.dense_arch.forward(mb[r].samples[s].dense.data(), &a.dense_hidden[(size_t)s * dh], oi + (size_t)F * D);
          float logit = 0.f;
          m.over_arch.forward(oi, &a.over_hidden[(size_t)s * oh], &logit);
          a.probs[s] = sigmoid((double)logit);
          const double y = (double)mb[r].samples[s].label;
          const double dlogit = a.probs[s] - y;
          m.over_arch.backward_dx(&a.over_hidden[(size_t)s * oh], &dlogit, &a.dh_over[(size_t)s * oh], dx.data());
          for (uint32_t k = 0; k < F * D; ++k) upstream[r][(size_t)s * F * D + k] = (float)dx[k];
          for (uint32_t j = 0; j < D; ++j) a.ddense_out[(size_t)s * D + j] = dx[(size_t)F * D + j];
          m.dense_arch.backward_dx(&a.dense_hidden[(size_t)s * dh], &a.ddense_out[(size_t)s * D],
                                   &a.dh_dense[(size_t)s * dh], nullptr);
        }
      }
      // backward of every group: embedding gradient + fused update
      for (uint32_t g = 0; g < M; ++g) {
        std::vector<const uint32_t*> lp(N), ip(N);
        std::vector<const float*> up(N);
        std::vector<float*> pp(N);
        std::vector<std::vector<float>> scratch(N, std::vector<float>(up_n));
        for (uint32_t n = 0; n < N; ++n) {
          lp[n] = len[g * N + n].data();
          ip[n] = ids[g * N + n].data();
          up[n] = upstream[g * N + n].data();
          pp[n] = scratch[n].data();
        }
        if (ref_group_step(F, N, B, rows.data(), dims.data(), ne, pl.data(), t.opt.eta, t.opt.eps, t.opt.c,
                           o->sgd, lp.data(), ip.data(), up.data(), pp.data(), ws[g].data(), vs[g].data(),
                           dirty[g].data(), 1, nullptr))
          return -1;
      }
      // dense_sync_and_apply: one left fold in (rank, sample) order
      dense_mean.reset();
      over_mean.reset();
      for (uint32_t r = 0; r < T; ++r) {
        const Act& a = act[r];
        const RankModel& m = models[r];
        for (uint32_t s = 0; s < B; ++s) {
          const double dlogit = a.probs[s] - (double)mb[r].samples[s].label;
          m.over_arch.accumulate_grads(&a.over_in[(size_t)s * oin], &a.over_hidden[(size_t)s * oh], &dlogit,
                                       &a.dh_over[(size_t)s * oh], over_mean);
          m.dense_arch.accumulate_grads(mb[r].samples[s].dense.data(), &a.dense_hidden[(size_t)s * dh],
                                        &a.ddense_out[(size_t)s * D], &a.dh_dense[(size_t)s * dh], dense_mean);
        }
      }
      const double inv_global = 1.0 / ((double)T * B);
      models[0].dense_arch.apply_sgd(dense_mean, t.opt.eta, inv_global);
      models[0].over_arch.apply_sgd(over_mean, t.opt.eta, inv_global);
      for (uint32_t r = 1; r < T; ++r) {
        models[r].dense_arch.copy_params_from(models[0].dense_arch);
        models[r].over_arch.copy_params_from(models[0].over_arch);
      }
      if (M > 1 && (step + 1) % t.sync_interval == 0) {
        std::vector<float*> wp(M), vp(M);
        std::vector<uint8_t*> dp(M);
        for (uint32_t g = 0; g < M; ++g) {
          wp[g] = ws[g].data();
          vp[g] = vs[g].data();
          dp[g] = dirty[g].data();
        }
        ref_sync(M, F, rows.data(), dims.data(), o->sgd, wp.data(), vp.data(), dp.data());
      }
      const size_t bf = (size_t)B * F, ni = bf * L;
      for (uint32_t r = 0; r < T; ++r) {
        const size_t at = (size_t)step * T + r;
        if (rec_len) std::memcpy(rec_len + at * bf, len[r].data(), bf * 4);
        if (rec_ids) std::memcpy(rec_ids + at * ni, ids[r].data(), ni * 4);
        if (rec_up) std::memcpy(rec_up + at * up_n, upstream[r].data(), up_n * 4);
        if (rec_pooled) std::memcpy(rec_pooled + at * up_n, pooled[r].data(), up_n * 4);
      }
    }
    for (uint32_t g = 0; g < M; ++g) {
      std::memcpy(w_out[g], ws[g].data(), rf * 4);
      std::memcpy(v_out[g], vs[g].data(), rv * 4);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ---- analytic helpers (cost_model.cpp, moment_analysis.cpp, trainer.cpp) ----
double ref_memory_overhead(double s, uint32_t g, uint32_t t) { return memory_overhead(s, g, t); }
double ref_sync_latency(double s, uint32_t g, uint32_t t, double bw) { return sync_latency(s, g, t, bw); }
double ref_qps_scaling_factor(double a, double b, double c, double d) { return qps_scaling_factor(a, b, c, d); }
double ref_closed_form_ratio(double mu, double sigma, uint32_t dim, uint32_t b, uint32_t g) {
  return closed_form_ratio(make_noise_model(mu, sigma, dim, b), g);
}
double ref_recommend_c(double mu, double sigma, uint32_t dim, uint32_t b, uint32_t g) {
  return recommend_c(make_noise_model(mu, sigma, dim, b), g);
}
void ref_estimate_increment_ratio(double mu, double sigma, uint32_t dim, uint32_t b, uint32_t g, uint64_t trials,
                                  uint64_t seed, double* out2) {
  const auto r = estimate_increment_ratio(make_noise_model(mu, sigma, dim, b), g, trials, seed);
  out2[0] = r.ratio_estimate;
  out2[1] = r.std_error;
}
double ref_evaluate_ne(const double* p, const float* y, uint64_t n) {
  return evaluate_ne(std::span<const double>(p, n), std::span<const float>(y, n)).ne;
}

}  // extern "C"
