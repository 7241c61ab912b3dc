// Trainer facade (include/sparse2d/trainer.hpp:106-132): the reference's
// single-object training loop over the 2D mesh, with every rank a virtual
// rank of this process (LocalHub) on the GPUs given -- the shape of
// Trainer::Impl (src/trainer.cpp:164-257, run_step 615-663).  Per step and
// rank: the reference DataGenerator's ids on the device (s2d_gen_batch), the
// lookup into the engine-owned pooled buffer, the upstream gradient (a caller
// callback; else the device MLPs of dense.h -- the reference's own dense
// model -- or the synthetic f32(1e-3 N(0,1)) of SURVEY.md 8(d)), the
// backward + fused update, and the replica sync every sync_interval steps
// (trainer.cpp:661); then, with the MLPs, the dense DP step on rank 0's GPU
// (trainer.cpp:507-545) and its parameters copied to every rank.  One host
// thread per rank runs each call; the calls of different ranks meet on the
// hub exactly like NCCL ranks do.
#include <cmath>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <thread>

#include "ctx.h"
#include "dense.h"

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

  // ---- dense model (dense.h) ----
  // per-rank parameter block: f32 [dense w1 b1 w2 b2 | over w1 b1 w2 b2]
  // then the f64 mirrors [dense w1d w2d | over w1d w2d]
  struct MlpLayout {
    uint32_t in = 0, hidden = 0, out = 0;
    size_t w1 = 0, b1 = 0, w2 = 0, b2 = 0, w1d = 0, w2d = 0;  // byte offsets
  };
  struct DenseRank {
    DevBuf params, gt_ids, gt_dense;
    DevBuf dense, labels, dense_out, dhid, ohid, logit, probs, dlogit, loss, lsum, dh_over, ddense, dh_dense;
    double lsum_host[2] = {0.0, -1.0};
  };
  bool dense_on = false;
  MlpLayout lay[2];  // 0 dense_arch, 1 over_arch
  size_t param_bytes = 0;
  std::vector<DenseRank> dn;
  DevBuf fold_ptrs;  // rank 0: per-rank pointer tables of the fold
  double last_loss = 0.0;
  bool have_loss = false;
  // evaluation (trainer.cpp:687-771), on rank 0's GPU
  DevBuf ev_ids, ev_len, ev_dense, ev_labels, ev_pooled, ev_dout, ev_dhid, ev_ohid, ev_logit, ev_probs, ev_shards;
  std::vector<float> ev_labels_host;
  bool ev_ready = false;
  std::vector<s2d_train_metrics_row> metrics_rows;
  s2d_ne_report final_ne{};
  bool final_done = false;

  MlpView view(uint32_t r, int a) {
    const MlpLayout& l = lay[a];
    char* b = dn[r].params.as<char>();
    return MlpView{l.in, l.hidden, l.out, reinterpret_cast<float*>(b + l.w1), reinterpret_cast<float*>(b + l.b1),
                   reinterpret_cast<float*>(b + l.w2), reinterpret_cast<float*>(b + l.b2),
                   reinterpret_cast<double*>(b + l.w1d), reinterpret_cast<double*>(b + l.w2d)};
  }

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
    if (o.dense_model) dense_create();
  }

  // init_rank_model (model.cpp:193-199): Mlp(dims, init_seed, tag) draws w1
  // then w2 from CounterRng({seed, tag}) as f32(lo + (hi - lo) * u) with
  // bound 1/sqrt(fan-in), biases 0 (model.cpp:46-66); every rank identical.
  static void mlp_init(const MlpLayout& l, uint64_t seed, uint64_t tag, char* host) {
    const uint64_t f[2] = {seed, tag};
    const uint64_t key = rng_make_key(f, 2);
    uint64_t ctr = 0;
    auto uni = [&](double lo, double hi) {
      const uint64_t z = key + (++ctr) * 0x9E3779B97F4A7C15ULL;
      uint64_t x = z;
      x ^= x >> 30;
      x *= 0xBF58476D1CE4E5B9ULL;
      x ^= x >> 27;
      x *= 0x94D049BB133111EBULL;
      x ^= x >> 31;
      return lo + (hi - lo) * (static_cast<double>(x >> 11) * 0x1.0p-53);
    };
    const double bound1 = 1.0 / std::sqrt(static_cast<double>(l.in));
    const double bound2 = 1.0 / std::sqrt(static_cast<double>(l.hidden));
    float* w1 = reinterpret_cast<float*>(host + l.w1);
    float* w2 = reinterpret_cast<float*>(host + l.w2);
    double* w1d = reinterpret_cast<double*>(host + l.w1d);
    double* w2d = reinterpret_cast<double*>(host + l.w2d);
    for (size_t i = 0; i < (size_t)l.hidden * l.in; ++i) w1[i] = static_cast<float>(uni(-bound1, bound1));
    for (size_t i = 0; i < (size_t)l.out * l.hidden; ++i) w2[i] = static_cast<float>(uni(-bound2, bound2));
    std::memset(host + l.b1, 0, (size_t)l.hidden * 4);
    std::memset(host + l.b2, 0, (size_t)l.out * 4);
    for (size_t i = 0; i < (size_t)l.hidden * l.in; ++i) w1d[i] = static_cast<double>(w1[i]);
    for (size_t i = 0; i < (size_t)l.out * l.hidden; ++i) w2d[i] = static_cast<double>(w2[i]);
  }

  void dense_create() {
    if (o.dense_dim < 1 || o.dense_hidden < 1 || o.over_hidden < 1)
      throw Error(S2D_EINVAL, "model dimensions must all be >= 1");  // DlrmConfig::validate (model.cpp:188-192)
    if (o.eval_samples < 1) throw Error(S2D_EINVAL, "eval_samples must be >= 1");  // trainer.cpp:56-58
    const uint32_t FD = o.num_tables * o.dim;
    lay[0].in = o.dense_dim, lay[0].hidden = o.dense_hidden, lay[0].out = o.dim;
    lay[1].in = FD + o.dim, lay[1].hidden = o.over_hidden, lay[1].out = 1;  // DlrmConfig::over_in
    size_t off = 0;
    auto take = [&](size_t bytes, size_t align) {
      off = (off + align - 1) / align * align;
      const size_t at = off;
      off += bytes;
      return at;
    };
    for (auto& l : lay) {
      l.w1 = take((size_t)l.hidden * l.in * 4, 16);
      l.b1 = take((size_t)l.hidden * 4, 16);
      l.w2 = take((size_t)l.out * l.hidden * 4, 16);
      l.b2 = take((size_t)l.out * 4, 16);
    }
    for (auto& l : lay) {
      l.w1d = take((size_t)l.hidden * l.in * 8, 16);
      l.w2d = take((size_t)l.out * l.hidden * 8, 16);
    }
    param_bytes = off;
    std::vector<char> host(param_bytes, 0);
    mlp_init(lay[0], o.init_seed, 101, host.data());
    mlp_init(lay[1], o.init_seed, 102, host.data());
    dn.resize(T);
    const uint32_t B = o.per_rank_batch;
    run_all([&](uint32_t r) {
      Ctx& c = *ranks[r];
      S2D_CUDA(cudaSetDevice(c.device));
      DenseRank& d = dn[r];
      d.params.ensure(param_bytes);
      S2D_CUDA(cudaMemcpy(d.params.p, host.data(), param_bytes, cudaMemcpyHostToDevice));
      // GroundTruthModel(data_seed, ...) (data.cpp:37-55) on this rank's GPU
      d.gt_ids.ensure((size_t)o.num_tables * o.rows_per_table * 4);
      d.gt_dense.ensure((size_t)o.dense_dim * 4);
      for (uint32_t f = 0; f < o.num_tables; ++f) {
        const uint64_t kf[3] = {o.data_seed, 10, f};
        launch_gt_normals(rng_make_key(kf, 3), o.rows_per_table, o.gt_id_scale,
                          d.gt_ids.as<float>() + (size_t)f * o.rows_per_table, c.stream);
      }
      const uint64_t kd[2] = {o.data_seed, 11};
      launch_gt_normals(rng_make_key(kd, 2), o.dense_dim, o.gt_dense_scale, d.gt_dense.as<float>(), c.stream);
      d.dense.ensure((size_t)B * o.dense_dim * 4);
      d.labels.ensure((size_t)B * 4);
      d.dense_out.ensure((size_t)B * o.dim * 4);
      d.dhid.ensure((size_t)B * o.dense_hidden * 4);
      d.ohid.ensure((size_t)B * o.over_hidden * 4);
      d.logit.ensure((size_t)B * 4);
      d.probs.ensure((size_t)B * 8);
      d.dlogit.ensure((size_t)B * 8);
      d.loss.ensure((size_t)B * 8);
      d.lsum.ensure(16);
      d.dh_over.ensure((size_t)B * o.over_hidden * 8);
      d.ddense.ensure((size_t)B * o.dim * 8);
      d.dh_dense.ensure((size_t)B * o.dense_hidden * 8);
      S2D_CUDA(cudaStreamSynchronize(c.stream));
    });
    fold_ptrs.release();
    S2D_CUDA(cudaSetDevice(ranks[0]->device));
    // the dense DP fold and the evaluation read every rank's buffers from
    // rank 0's GPU
    for (uint32_t r = 1; r < T; ++r) {
      const int d = ranks[r]->device;
      if (d == ranks[0]->device) continue;
      const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        (void)cudaGetLastError();
      else
        S2D_CUDA(e);
    }
    fold_ptrs.ensure((size_t)9 * T * sizeof(void*));
    dense_on = true;
  }

  // pool_and_forward's MLP part + backward_rank (trainer.cpp:391-438) on
  // rank r's stream: dense features and labels, dense_arch -> over_in tail,
  // over_arch -> logit -> prob, loss, over_arch.backward_dx -> the f32 wire
  // gradient (upstream) and the dense arch's f64 upstream, dense_arch's
  // hidden gradient, the rank's loss_sum.
  void dense_forward_backward(uint32_t r, uint64_t k) {
    Ctx& c = *ranks[r];
    DenseRank& d = dn[r];
    const uint32_t B = o.per_rank_batch, FD = o.num_tables * o.dim;
    launch_gen_dense(o.data_seed, 0, k, r, B, o.dense_dim, d.dense.as<float>(), c.stream);
    launch_gen_labels(o.data_seed, 0, k, r, B, o.num_tables, o.ids_per_sample, d_ids[r].as<uint32_t>(),
                      d.gt_ids.as<float>(), o.rows_per_table, d.dense.as<float>(), d.gt_dense.as<float>(), o.dense_dim,
                      o.gt_bias, d.labels.as<float>(), c.stream);
    const MlpView da = view(r, 0), oa = view(r, 1);
    launch_mlp_hidden(da, MlpInput{d.dense.as<float>(), o.dense_dim, nullptr, 0}, B, d.dhid.as<float>(), c.stream);
    launch_mlp_out(da, d.dhid.as<float>(), B, d.dense_out.as<float>(), nullptr, c.stream);
    launch_mlp_hidden(oa, MlpInput{c.pooled_buffer(), FD, d.dense_out.as<float>(), o.dim}, B, d.ohid.as<float>(),
                      c.stream);
    launch_mlp_out(oa, d.ohid.as<float>(), B, d.logit.as<float>(), d.probs.as<double>(), c.stream);
    launch_over_backward(oa, d.ohid.as<float>(), d.probs.as<double>(), d.labels.as<float>(), B,
                         d.dlogit.as<double>(), d.dh_over.as<double>(), d.loss.as<double>(), c.stream);
    launch_mlp_dx(oa, d.dh_over.as<double>(), B, FD, d_up[r].as<float>(), d.ddense.as<double>(), c.stream);
    launch_mlp_dhidden(da, d.dhid.as<float>(), d.ddense.as<double>(), B, d.dh_dense.as<double>(), c.stream);
    launch_loss_sum(d.loss.as<double>(), B, d.lsum.as<double>(), c.stream);
  }

  // dense_sync_and_apply (trainer.cpp:507-545) on rank 0's GPU: each layer's
  // gradient folded over (rank, sample) from every rank's activations (peer
  // reads when the ranks span GPUs), one SGD step with eta * 1/(T*B), the
  // parameters copied to every other rank; last_loss = (sum over ranks of
  // loss_sum) / (T*B).
  void dense_sync_and_apply(uint64_t k) {
    const uint32_t B = o.per_rank_batch, FD = o.num_tables * o.dim;
    for (uint32_t r = 0; r < T; ++r)
      if (dn[r].lsum_host[1] >= 0.0)
        throw Error(S2D_ERUNTIME, "nonfinite loss at step " + std::to_string(k) + " rank " + std::to_string(r) +
                                      " sample " + std::to_string((uint64_t)dn[r].lsum_host[1]));
    double loss_total = 0.0;
    for (uint32_t r = 0; r < T; ++r) loss_total += dn[r].lsum_host[0];
    const double inv_global = 1.0 / (static_cast<double>(T) * B);
    last_loss = loss_total * inv_global;
    have_loss = true;
    Ctx& c0 = *ranks[0];
    S2D_CUDA(cudaSetDevice(c0.device));
    // pointer tables: 0 dh_over, 1 pooled, 2 dense_out, 3 dlogit, 4 ohid,
    // 5 dh_dense, 6 dense, 7 ddense, 8 dhid
    std::vector<const void*> tab((size_t)9 * T);
    for (uint32_t r = 0; r < T; ++r) {
      DenseRank& d = dn[r];
      const void* p[9] = {d.dh_over.p, ranks[r]->pooled_buffer(), d.dense_out.p, d.dlogit.p, d.ohid.p,
                          d.dh_dense.p, d.dense.p, d.ddense.p, d.dhid.p};
      for (int q = 0; q < 9; ++q) tab[(size_t)q * T + r] = p[q];
    }
    S2D_CUDA(cudaMemcpyAsync(fold_ptrs.p, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice, c0.stream));
    auto tp = [&](int q) { return fold_ptrs.as<const void*>() + (size_t)q * T; };
    const double f = o.opt.eta * inv_global;  // Mlp::apply_sgd(g, eta, inv_global): lr * scale
    const MlpView oa = view(0, 1), da = view(0, 0);
    auto fold = [&](const MlpView& m, int layer, int qd, int skip, int qx0, uint32_t n0, int qx1, uint32_t n1) {
      FoldArgs a{};
      a.T = T;
      a.B = B;
      a.P = layer == 1 ? m.hidden : m.out;
      a.Q = layer == 1 ? m.in : m.hidden;
      a.d = reinterpret_cast<const double* const*>(tp(qd));
      a.skip_zero = skip;
      a.x0 = reinterpret_cast<const float* const*>(tp(qx0));
      a.n0 = n0;
      a.x1 = qx1 >= 0 ? reinterpret_cast<const float* const*>(tp(qx1)) : nullptr;
      a.n1 = n1;
      a.w = layer == 1 ? m.w1 : m.w2;
      a.wd = layer == 1 ? m.w1d : m.w2d;
      a.b = layer == 1 ? m.b1 : m.b2;
      a.f = f;
      launch_fold_sgd(a, c0.stream);
    };
    fold(oa, 2, 3, 0, 4, o.over_hidden, -1, 0);       // over w2 / b2: dlogit x over hidden
    fold(oa, 1, 0, 1, 1, FD, 2, o.dim);               // over w1 / b1: dh_over x [pooled | dense out]
    fold(da, 2, 7, 0, 8, o.dense_hidden, -1, 0);      // dense w2 / b2: ddense x dense hidden
    fold(da, 1, 5, 1, 6, o.dense_dim, -1, 0);         // dense w1 / b1: dh_dense x dense features
    S2D_CUDA(cudaStreamSynchronize(c0.stream));
    for (uint32_t r = 1; r < T; ++r) {  // ranks 1+ adopt rank 0's result (trainer.cpp:540-543)
      S2D_CUDA(cudaMemcpyPeer(dn[r].params.p, ranks[r]->device, dn[0].params.p, c0.device, param_bytes));
    }
  }

  void step_n(uint64_t count) {
    const uint32_t B = o.per_rank_batch;
    const uint64_t nnz = (uint64_t)B * o.num_tables * o.ids_per_sample;
    const bool mlp = dense_on && !upstream_fn;
    auto one_step = [&](uint32_t r, uint64_t k) {
      Ctx& c = *ranks[r];
      c.gen_batch(o.data_seed, k, r, B, zipf.data(), per_sample.data(), d_len[r].as<uint32_t>(),
                  d_ids[r].as<uint32_t>(), S2D_DEVICE);
      c.lookup_forward(B, d_len[r].as<uint32_t>(), d_ids[r].as<uint32_t>(), nnz, nullptr, S2D_DEVICE);
      if (upstream_fn) {
        S2D_CUDA(cudaStreamSynchronize(c.stream));
        const int rc = upstream_fn(upstream_user, r, k, B, d_len[r].as<uint32_t>(), c.pooled_buffer(),
                                   d_up[r].as<float>(), c.stream);
        if (rc) throw Error(S2D_ERUNTIME, "upstream callback failed with " + std::to_string(rc));
      } else if (mlp) {
        dense_forward_backward(r, k);
      } else {
        c.gen_upstream(o.data_seed ^ 0x5EEDull, k, r, B, d_up[r].as<float>(), S2D_DEVICE);
      }
      c.backward_update(d_up[r].as<float>(), S2D_DEVICE);
      if (M > 1 && (k + 1) % o.sync_interval == 0) c.replica_sync();  // trainer.cpp:661
      c.synchronize_and_check();
      if (mlp) S2D_CUDA(cudaMemcpy(dn[r].lsum_host, dn[r].lsum.p, 16, cudaMemcpyDeviceToHost));
    };
    if (mlp) {
      // the dense DP step joins every rank between steps
      for (uint64_t i = 0; i < count; ++i) {
        const uint64_t k = steps_done;
        run_all([&](uint32_t r) {
          S2D_CUDA(cudaSetDevice(ranks[r]->device));
          one_step(r, k);
        });
        dense_sync_and_apply(k);
        ++steps_done;
        after_step();
      }
      return;
    }
    const uint64_t first = steps_done;
    run_all([&](uint32_t r) {
      S2D_CUDA(cudaSetDevice(ranks[r]->device));
      for (uint64_t k = first; k < first + count; ++k) one_step(r, k);
    });
    steps_done += count;
  }

  // ensure_eval_set (trainer.cpp:689-705): eval_samples samples in chunks of
  // 1024, chunk c = DataGenerator::gen_batch_into(step c, rank 0, lane kEval)
  // with eval_seed; ids, dense features and labels stay on rank 0's GPU
  void ensure_eval_set() {
    if (ev_ready) return;
    Ctx& c = *ranks[0];
    S2D_CUDA(cudaSetDevice(c.device));
    const uint32_t S = o.eval_samples, F = o.num_tables, L = o.ids_per_sample, dd = o.dense_dim;
    ev_ids.ensure((size_t)S * F * L * 4);
    ev_len.ensure((size_t)std::min<uint32_t>(S, 1024) * F * 4);
    ev_dense.ensure((size_t)S * dd * 4);
    ev_labels.ensure((size_t)S * 4);
    uint64_t idx = 0;
    for (uint32_t c0 = 0; c0 < S; ++idx) {
      const uint32_t take = std::min<uint32_t>(1024, S - c0);
      c.gen_batch(o.eval_seed, idx, 0, take, zipf.data(), per_sample.data(), ev_len.as<uint32_t>(),
                  ev_ids.as<uint32_t>() + (size_t)c0 * F * L, S2D_DEVICE, 1);
      launch_gen_dense(o.eval_seed, 1, idx, 0, take, dd, ev_dense.as<float>() + (size_t)c0 * dd, c.stream);
      launch_gen_labels(o.eval_seed, 1, idx, 0, take, F, L, ev_ids.as<uint32_t>() + (size_t)c0 * F * L,
                        dn[0].gt_ids.as<float>(), o.rows_per_table, ev_dense.as<float>() + (size_t)c0 * dd,
                        dn[0].gt_dense.as<float>(), dd, o.gt_bias, ev_labels.as<float>() + c0, c.stream);
      c0 += take;
    }
    ev_labels_host.resize(S);
    S2D_CUDA(cudaStreamSynchronize(c.stream));
    S2D_CUDA(cudaMemcpy(ev_labels_host.data(), ev_labels.p, (size_t)S * 4, cudaMemcpyDeviceToHost));
    const uint32_t FD = F * o.dim;
    ev_pooled.ensure((size_t)S * FD * 4);
    ev_dout.ensure((size_t)S * o.dim * 4);
    ev_dhid.ensure((size_t)S * o.dense_hidden * 4);
    ev_ohid.ensure((size_t)S * o.over_hidden * 4);
    ev_logit.ensure((size_t)S * 4);
    ev_probs.ensure((size_t)S * 8);
    ev_shards.ensure((size_t)F * N * sizeof(EvalShard));
    ev_ready = true;
  }

  // eval_probs (trainer.cpp:714-743): pool_ids over group 0's shards (peer
  // reads when its ranks span GPUs), rank 0's dense_arch + over_arch, sigmoid
  std::vector<double> eval_probs() {
    ensure_eval_set();
    const uint32_t S = o.eval_samples, F = o.num_tables, FD = F * o.dim;
    std::vector<EvalShard> sh((size_t)F * N);
    for (uint32_t f = 0; f < F; ++f)
      for (uint32_t l = 0; l < N; ++l) {
        Ctx& cl = *ranks[l];
        const FeatDev& fd = cl.feats[f];
        sh[(size_t)f * N + l] = {fd.lo, fd.hi, cl.weights.as<char>() + fd.wbase * (cl.bf16 ? 2 : 4)};
      }
    Ctx& c = *ranks[0];
    S2D_CUDA(cudaSetDevice(c.device));
    S2D_CUDA(cudaMemcpyAsync(ev_shards.p, sh.data(), sh.size() * sizeof(EvalShard), cudaMemcpyHostToDevice, c.stream));
    launch_eval_pool(S, F, o.ids_per_sample, N, ev_ids.as<uint32_t>(), ev_shards.as<EvalShard>(), o.dim, c.bf16,
                     ev_pooled.as<float>(), c.stream);
    const MlpView da = view(0, 0), oa = view(0, 1);
    launch_mlp_hidden(da, MlpInput{ev_dense.as<float>(), o.dense_dim, nullptr, 0}, S, ev_dhid.as<float>(), c.stream);
    launch_mlp_out(da, ev_dhid.as<float>(), S, ev_dout.as<float>(), nullptr, c.stream);
    launch_mlp_hidden(oa, MlpInput{ev_pooled.as<float>(), FD, ev_dout.as<float>(), o.dim}, S, ev_ohid.as<float>(),
                      c.stream);
    launch_mlp_out(oa, ev_ohid.as<float>(), S, ev_logit.as<float>(), ev_probs.as<double>(), c.stream);
    std::vector<double> probs(S);
    S2D_CUDA(cudaStreamSynchronize(c.stream));
    S2D_CUDA(cudaMemcpy(probs.data(), ev_probs.p, (size_t)S * 8, cudaMemcpyDeviceToHost));
    return probs;
  }

  s2d_ne_report evaluate(const std::vector<double>& probs) {
    s2d_ne_report rep{};
    const int rc = s2d_evaluate_ne(probs.data(), ev_labels_host.data(), probs.size(), &rep.ne, &rep.baseline_ctr);
    if (rc) throw Error(rc, "evaluate_ne: all labels identical, baseline entropy is zero");
    rep.eval_samples = probs.size();
    return rep;
  }

  // make_metrics_row (trainer.cpp:745-771) + the step_n cadence (773-787)
  void after_step() {
    const bool last = steps_done == o.steps;
    const bool cadence = o.eval_cadence > 0 && steps_done % o.eval_cadence == 0;
    if (!cadence && !last) return;
    const auto probs = eval_probs();
    const s2d_ne_report rep = evaluate(probs);
    std::vector<s2d_metrics_row> mr(T);
    run_all([&](uint32_t r) { ranks[r]->metrics(&mr[r]); });
    s2d_train_metrics_row row{};
    row.step = steps_done;
    row.loss = last_loss;
    row.ne = rep.ne;
    row.eff_lr_p50 = mr[0].eff_lr_p50;
    row.eff_lr_p99 = mr[0].eff_lr_p99;
    row.v_mean = mr[0].v_mean;
    metrics_rows.push_back(row);
    if (last) {
      final_ne = rep;
      final_done = true;
    }
  }

  s2d_ne_report finalize_ne() {
    if (!dense_on) throw Error(S2D_EINVAL, "the trainer has no dense model");
    if (!final_done) {
      final_ne = evaluate(eval_probs());
      final_done = true;
    }
    return final_ne;
  }

  // Trainer::rank_model(rank) (trainer.hpp:125)
  void rank_model(uint32_t rank, int arch, float* w1, float* b1, float* w2, float* b2) {
    if (!dense_on) throw Error(S2D_EINVAL, "the trainer has no dense model");
    if (rank >= T) throw Error(S2D_ERANGE, "rank out of range");
    if (arch != 0 && arch != 1) throw Error(S2D_EINVAL, "arch must be 0 (dense_arch) or 1 (over_arch)");
    const MlpLayout& l = lay[arch];
    S2D_CUDA(cudaSetDevice(ranks[rank]->device));
    const char* b = dn[rank].params.as<char>();
    if (w1) S2D_CUDA(cudaMemcpy(w1, b + l.w1, (size_t)l.hidden * l.in * 4, cudaMemcpyDeviceToHost));
    if (b1) S2D_CUDA(cudaMemcpy(b1, b + l.b1, (size_t)l.hidden * 4, cudaMemcpyDeviceToHost));
    if (w2) S2D_CUDA(cudaMemcpy(w2, b + l.w2, (size_t)l.out * l.hidden * 4, cudaMemcpyDeviceToHost));
    if (b2) S2D_CUDA(cudaMemcpy(b2, b + l.b2, (size_t)l.out * 4, cudaMemcpyDeviceToHost));
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

int s2d_trainer_rank_model(s2d_trainer* t, uint32_t rank, int32_t arch, float* w1, float* b1, float* w2, float* b2) {
  return tguard([&] { as_trainer(t)->rank_model(rank, arch, w1, b1, w2, b2); });
}

int s2d_trainer_last_loss(s2d_trainer* t, double* out) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    if (!out) throw Error(S2D_EINVAL, "null argument");
    if (!tr->dense_on) throw Error(S2D_EINVAL, "the trainer has no dense model");
    if (!tr->have_loss) throw Error(S2D_EINVAL, "no step has run");
    *out = tr->last_loss;
  });
}

int s2d_trainer_metrics_rows(s2d_trainer* t, s2d_train_metrics_row* out, uint32_t cap, uint32_t* n) {
  return tguard([&] {
    auto* tr = as_trainer(t);
    if (n) *n = (uint32_t)tr->metrics_rows.size();
    if (out && cap < tr->metrics_rows.size()) throw Error(S2D_EINVAL, "metrics output capacity too small");
    if (out) std::memcpy(out, tr->metrics_rows.data(), tr->metrics_rows.size() * sizeof(s2d_train_metrics_row));
  });
}

int s2d_trainer_final_ne(s2d_trainer* t, s2d_ne_report* out) {
  return tguard([&] {
    if (!out) throw Error(S2D_EINVAL, "null argument");
    *out = as_trainer(t)->finalize_ne();
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
