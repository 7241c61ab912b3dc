// Trainer facade (include/sparse2d/trainer.hpp:106-132): the reference's
// single-object training loop over the 2D mesh, with every rank a virtual
// rank of this process (LocalHub) on the GPUs given -- the shape of
// Trainer::Impl (src/trainer.cpp:164-257, run_step 615-663), minus the dense
// MLP.  Per step and rank: the reference DataGenerator's ids on the device
// (s2d_gen_batch), the lookup into the engine-owned pooled buffer, the
// upstream gradient (a caller callback -- the dense model's backward -- or
// the synthetic f32(1e-3 N(0,1)) of SURVEY.md 8(d)), the backward + fused
// update, and the replica sync every sync_interval steps (trainer.cpp:661).
// One host thread per rank runs each call; the calls of different ranks
// meet on the hub exactly like NCCL ranks do.
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <thread>

#include "ctx.h"

namespace s2d {

struct Trainer {
  s2d_trainer_options o{};
  uint32_t T = 1, M = 1, N = 1;
  std::vector<int> devices;
  std::shared_ptr<LocalHub> hub;
  std::vector<std::unique_ptr<Ctx>> ranks;
  std::vector<s2d_plan_entry> plan;
  std::vector<DevBuf> d_len, d_ids, d_up;
  std::vector<double> zipf;
  std::vector<uint32_t> per_sample;
  uint64_t steps_done = 0;
  s2d_upstream_fn upstream_fn = nullptr;
  void* upstream_user = nullptr;

  // fn(rank) on T threads; the first error is rethrown
  void run_all(const std::function<void(uint32_t)>& fn) {
    std::vector<std::exception_ptr> err(T);
    std::vector<std::thread> th;
    th.reserve(T);
    for (uint32_t r = 0; r < T; ++r)
      th.emplace_back([&, r] {
        try {
          fn(r);
        } catch (...) {
          err[r] = std::current_exception();
        }
      });
    for (auto& t : th) t.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
  }

  void create(const s2d_trainer_options& opts) {
    o = opts;
    const s2d_topology topo = make_topology(o.total_ranks, o.groups);
    T = topo.total_ranks;
    M = topo.groups;
    N = topo.ranks_per_group;
    if (o.num_tables < 1 || o.rows_per_table < 1 || o.dim < 1)
      throw Error(S2D_EINVAL, "model dimensions must all be >= 1");  // DlrmConfig::validate, model.cpp
    if (o.per_rank_batch < 1) throw Error(S2D_EINVAL, "per_rank_batch must be >= 1");
    if (o.sync_interval < 1) throw Error(S2D_EINVAL, "sync_interval must be >= 1");
    if (!(o.zipf_exponent >= 0)) throw Error(S2D_EINVAL, "zipf_exponent must be >= 0");
    if (o.ids_per_sample < 1) throw Error(S2D_EINVAL, "ids_per_sample must be >= 1");
    check_optimizer(o.opt);
    int ndev = 0;
    S2D_CUDA(cudaGetDeviceCount(&ndev));
    if (ndev < 1) throw Error(S2D_ECUDA, "no CUDA device");
    devices.assign(T, 0);
    for (uint32_t r = 0; r < T; ++r)
      devices[r] = o.n_devices && o.devices ? o.devices[r % o.n_devices] : (int)(r % (uint32_t)ndev);
    // plan_greedy over profile_from_spec (planner.cpp:181-190; trainer.cpp:187-191)
    std::vector<s2d_table_load_profile> prof(o.num_tables);
    for (uint32_t f = 0; f < o.num_tables; ++f)
      prof[f] = {f, (uint64_t)o.rows_per_table * o.dim * 4, (double)o.ids_per_sample * ((double)N * o.per_rank_batch),
                 o.rows_per_table};
    plan = plan_greedy(prof, N, o.strategy);
    validate_plan(plan, N, prof);
    std::vector<s2d_table_desc> tables(o.num_tables);
    for (uint32_t f = 0; f < o.num_tables; ++f) tables[f] = {f, o.rows_per_table, o.dim, S2D_POOL_SUM};
    zipf.assign(o.num_tables, o.zipf_exponent);
    per_sample.assign(o.num_tables, o.ids_per_sample);
    hub = std::make_shared<LocalHub>(T);
    ranks.resize(T);
    d_len.resize(T);
    d_ids.resize(T);
    d_up.resize(T);
    const uint64_t BF = (uint64_t)o.per_rank_batch * o.num_tables;
    run_all([&](uint32_t r) {
      auto c = std::make_unique<Ctx>();
      c->create(devices[r], T, M, r, nullptr, hub);
      c->register_tables(tables.data(), (uint32_t)tables.size(), plan.data(), (uint32_t)plan.size(),
                         o.weight_dtype);
      c->set_optimizer(o.opt);
      c->strict = false;  // faults surface at the end of each step (synchronize_and_check)
      c->init_tables(o.init_seed);
      d_len[r].ensure(BF * 4);
      d_ids[r].ensure(BF * o.ids_per_sample * 4);
      d_up[r].ensure(BF * o.dim * 4);
      ranks[r] = std::move(c);
    });
  }

  void step_n(uint64_t count) {
    const uint32_t B = o.per_rank_batch;
    const uint64_t nnz = (uint64_t)B * o.num_tables * o.ids_per_sample;
    const uint64_t first = steps_done;
    run_all([&](uint32_t r) {
      Ctx& c = *ranks[r];
      S2D_CUDA(cudaSetDevice(c.device));
      for (uint64_t k = first; k < first + count; ++k) {
        c.gen_batch(o.data_seed, k, r, B, zipf.data(), per_sample.data(), d_len[r].as<uint32_t>(),
                    d_ids[r].as<uint32_t>(), S2D_DEVICE);
        c.lookup_forward(B, d_len[r].as<uint32_t>(), d_ids[r].as<uint32_t>(), nnz, nullptr, S2D_DEVICE);
        if (upstream_fn) {
          S2D_CUDA(cudaStreamSynchronize(c.stream));
          const int rc = upstream_fn(upstream_user, r, k, B, d_len[r].as<uint32_t>(), c.pooled_buffer(),
                                     d_up[r].as<float>(), c.stream);
          if (rc) throw Error(S2D_ERUNTIME, "upstream callback failed with " + std::to_string(rc));
        } else {
          c.gen_upstream(o.data_seed ^ 0x5EEDull, k, r, B, d_up[r].as<float>(), S2D_DEVICE);
        }
        c.backward_update(d_up[r].as<float>(), S2D_DEVICE);
        if (M > 1 && (k + 1) % o.sync_interval == 0) c.replica_sync();  // trainer.cpp:661
        c.synchronize_and_check();
      }
    });
    steps_done += count;
  }

  // replica of `group`, table f: the full rows x dim table assembled from
  // the group's shards (Trainer::replica_tables, trainer.cpp:845-853)
  void replica_table(uint32_t group, uint32_t f, float* w, float* v) {
    if (group >= M) throw Error(S2D_ERANGE, "group out of range");
    if (f >= o.num_tables) throw Error(S2D_ERANGE, "table out of range");
    for (uint32_t l = 0; l < N; ++l) {
      Ctx& c = *ranks[group * N + l];
      const FeatDev& fd = c.feats[f];
      if (fd.hi <= fd.lo) continue;
      c.shard_io(f, fd.lo, fd.hi, w ? w + (size_t)fd.lo * o.dim : nullptr, v ? v + fd.lo : nullptr, false);
    }
  }
};

}  // namespace s2d

using s2d::Error;

namespace {
template <typename Fn>
int tguard(Fn&& fn) {
  try {
    fn();
    return S2D_OK;
  } catch (const Error& e) {
    s2d::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    s2d::set_last_error(e.what());
    return S2D_ERUNTIME;
  }
}
s2d::Trainer* as_trainer(s2d_trainer* t) {
  if (!t) throw Error(S2D_EINVAL, "null trainer");
  return reinterpret_cast<s2d::Trainer*>(t);
}
}  // namespace

extern "C" {

int s2d_trainer_create(const s2d_trainer_options* opts, s2d_trainer** out) {
  return tguard([&] {
    if (!opts || !out) throw Error(S2D_EINVAL, "null argument");
    auto t = std::make_unique<s2d::Trainer>();
    t->create(*opts);
    *out = reinterpret_cast<s2d_trainer*>(t.release());
  });
}

int s2d_trainer_destroy(s2d_trainer* t) {
  return tguard([&] { delete reinterpret_cast<s2d::Trainer*>(t); });
}

int s2d_trainer_set_upstream(s2d_trainer* t, s2d_upstream_fn fn, void* user) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    tr->upstream_fn = fn;
    tr->upstream_user = user;
  });
}

int s2d_trainer_step_n(s2d_trainer* t, uint64_t count) {
  return tguard([&] { as_trainer(t)->step_n(count); });
}

int s2d_trainer_run(s2d_trainer* t) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    if (tr->steps_done < tr->o.steps) tr->step_n(tr->o.steps - tr->steps_done);
  });
}

int s2d_trainer_steps_done(s2d_trainer* t, uint64_t* out) {
  return tguard([&] { *out = as_trainer(t)->steps_done; });
}

int s2d_trainer_plan(s2d_trainer* t, s2d_plan_entry* out, uint32_t cap, uint32_t* n) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    if (n) *n = (uint32_t)tr->plan.size();
    if (out && cap < tr->plan.size()) throw Error(S2D_EINVAL, "plan output capacity too small");
    if (out) std::memcpy(out, tr->plan.data(), tr->plan.size() * sizeof(s2d_plan_entry));
  });
}

int s2d_trainer_replica_table(s2d_trainer* t, uint32_t group, uint32_t table, float* w, float* v) {
  return tguard([&] { as_trainer(t)->replica_table(group, table, w, v); });
}

int s2d_trainer_save_tables(s2d_trainer* t, const char* path) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    tr->run_all([&](uint32_t r) { tr->ranks[r]->save_tables(path); });
  });
}

int s2d_trainer_load_tables(s2d_trainer* t, const char* path) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    tr->run_all([&](uint32_t r) { tr->ranks[r]->load_tables(path); });
  });
}

int s2d_trainer_metrics(s2d_trainer* t, s2d_metrics_row* out) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    std::vector<s2d_metrics_row> rows(tr->T);
    tr->run_all([&](uint32_t r) { tr->ranks[r]->metrics(&rows[r]); });
    *out = rows[0];  // group 0's replica (trainer.cpp:745-771 reads replicas[0])
  });
}

int s2d_trainer_rank_ctx(s2d_trainer* t, uint32_t rank, s2d_ctx** out) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    if (rank >= tr->T) throw Error(S2D_ERANGE, "rank out of range");
    *out = reinterpret_cast<s2d_ctx*>(tr->ranks[rank].get());
  });
}

}  // extern "C"
