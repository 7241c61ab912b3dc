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
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sparse2d/data.hpp"
#include "sparse2d/embedding.hpp"
#include "sparse2d/optimizer.hpp"
#include "sparse2d/planner.hpp"
#include "sparse2d/topology.hpp"

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

}  // extern "C"
