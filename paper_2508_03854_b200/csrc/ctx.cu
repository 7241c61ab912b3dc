// Step driver of one rank.  Sequence per step (src/trainer.cpp:615-663,
// embedding phases only):
//
//   N == 1:  lengths -> id offsets (scan) -> K2 lookup writes pooled rows and
//            (slot, upstream-row) pairs -> [backward] radix sort -> K3b/K4
//            range partials + fused segment reduce / AdaGrad straight from the
//            upstream gradient.
//   N  > 1:  K1 count (lengths stored into the owners' receive buffers over
//            peer memory) + scans -> count matrix published to every peer ->
//            barrier -> one host read of the matrix (buffer sizes) -> K1
//            permute (ids stored into the owners' buffers) -> barrier -> owner
//            K2 lookup storing partials / final pooled rows into the
//            requesters' buffers (C1 fused) -> barrier -> requester combine;
//            the sort of the owner's pairs starts on a side stream right after
//            the lookup.  [backward] gradient gather storing each (bag, owner)
//            upstream row into the owner's buffer (C2 fused) -> barrier ->
//            fused update.
//   M  > 1:  replica_sync(): dirty-flag lists all-gathered into one ascending
//            union; over peer memory each replica owns a slice of the union,
//            receives every replica's copy of its rows, forms the f64
//            ascending-group mean and stores it into every replica (C3);
//            NCCL all-gather + mean is the fallback when the DP group cannot
//            map each other's memory.
// Barriers are device flags (st.release / ld.acquire, system scope) across
// processes, host rendezvous between virtual ranks of one process (comm.h).
//
// Every buffer on the wire has the reference's layout: demand ids per owner
// in (requester, sample, feature, occurrence) order, one partial / gradient
// row per non-empty (bag, owner) entry in (sample, feature) order
// (trainer.cpp:283-313, 331-335, 446-453).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "ctx.h"

#include <cmath>

namespace s2d {

void Ctx::phase_begin(int ph) {
  if (!profile) return;
  if (open_phase >= 0) phase_end();
  // every event pair drains the stream between two kernels (and breaks their
  // PDL overlap), so the light mode brackets only the dominant update kernels
  if (profile_hot_only && ph != kPhUpdate) return;
  while (ev_pool.size() < ev_used + 2) {
    cudaEvent_t e;
    S2D_CUDA(cudaEventCreate(&e));
    ev_pool.push_back(e);
  }
  S2D_CUDA(cudaEventRecord(ev_pool[ev_used], stream));
  ev_marks.push_back({ph, ev_used});
  ev_used += 2;
  open_phase = ph;
}

void Ctx::phase_end() {
  if (!profile || open_phase < 0) return;
  S2D_CUDA(cudaEventRecord(ev_pool[ev_marks.back().second + 1], stream));
  open_phase = -1;
}

void Ctx::phase_times(double* ms, uint32_t* counts) {
  for (int i = 0; i < kNumPhases; ++i) {
    ms[i] = 0.0;
    if (counts) counts[i] = 0;
  }
  phase_end();
  S2D_CUDA(cudaStreamSynchronize(stream));
  for (const auto& m : ev_marks) {
    float t = 0.f;
    S2D_CUDA(cudaEventElapsedTime(&t, ev_pool[m.second], ev_pool[m.second + 1]));
    ms[m.first] += t;
    if (counts) counts[m.first] += 1;
  }
  ev_marks.clear();
  ev_used = 0;
}

namespace {

int bit_width(uint32_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace

Ctx::~Ctx() {
  if (device >= 0) cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (PeerBuf* pb : {&p_flags, &p_xcnt, &p_len, &p_ids, &p_part, &p_grad, &p_pooled, &dp_flags, &dp_stage})
    for (void* q : pb->opened) cudaIpcCloseMemHandle(q);
  for (void* q : dp_opened) cudaIpcCloseMemHandle(q);
  for (auto e : ev_pool) cudaEventDestroy(e);
  for (cudaStream_t q : {h2d_stream, d2h_stream, sort_stream, sync_stream})
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (cudaEvent_t e : {ev_fwd, ev_d2h, ev_up, ev_keys, ev_sorted, ev_union, ev_sync_done, ev_in_ready, ev_in_used[0],
                        ev_in_used[1], ev_up_used[0], ev_up_used[1], ev_d2h_done[0], ev_d2h_done[1]})
    if (e) cudaEventDestroy(e);
  dp.destroy();
  mp.destroy();
  world.destroy();
  if (own_stream) cudaStreamDestroy(own_stream);
  if (hub) {
    hub->release_rank(rank);
    hub.reset();
    // buffers released by the member destructors after this body go to the
    // deferred-free list while other virtual ranks live (local_guard)
  }
}

void Ctx::create(int dev, uint32_t total, uint32_t groups, uint32_t r, const uint8_t* nccl_id,
                 std::shared_ptr<LocalHub> local_hub) {
  if (total == 0 || groups == 0 || total % groups)
    throw Error(S2D_EINVAL, "groups must divide total_ranks (both >= 1)");
  if (r >= total) throw Error(S2D_EINVAL, "rank out of range");
  T = total;
  M = groups;
  N = total / groups;
  if (N > (uint32_t)kMaxRanksPerGroup)
    throw Error(S2D_EINVAL, "owner bitmask limits ranks per group to 32");
  rank = r;
  group = r / N;
  local = r % N;
  device = dev;
  S2D_CUDA(cudaSetDevice(dev));
  S2D_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
  stream = own_stream;
  S2D_CUDA(cudaStreamCreateWithFlags(&h2d_stream, cudaStreamNonBlocking));
  S2D_CUDA(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking));
  S2D_CUDA(cudaStreamCreateWithFlags(&sort_stream, cudaStreamNonBlocking));
  S2D_CUDA(cudaStreamCreateWithFlags(&sync_stream, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&ev_fwd, &ev_d2h, &ev_up, &ev_keys, &ev_sorted, &ev_union, &ev_sync_done, &ev_in_ready,
                         &ev_in_used[0], &ev_in_used[1], &ev_up_used[0], &ev_up_used[1], &ev_d2h_done[0],
                         &ev_d2h_done[1]})
    S2D_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  err.ensure(4);
  S2D_CUDA(cudaMemsetAsync(err.p, 0, 4, stream));
  err_host.ensure(16);
  *err_host.as<uint32_t>() = 0;
  h_counts.ensure(4096);
  if (local_hub) {
    // virtual ranks of one process: collectives rendezvous on the hub,
    // peer buffers are plain device pointers
    if (local_hub->T != T) throw Error(S2D_EINVAL, "hub size differs from total_ranks");
    local_hub->claim_rank(rank);
    hub = local_hub;
    local_ctx_enter();
    local_guard.armed = true;
    world.hub = mp.hub = dp.hub = hub;
    world.key = 1ull << 40;
    mp.key = (2ull << 40) | group;
    dp.key = (3ull << 40) | local;
  } else if (T > 1) {
    if (!nccl_id) throw Error(S2D_EINVAL, "nccl_id required when total_ranks > 1");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    S2D_NCCL(ncclCommInitRank(&world.nccl, (int)T, id, (int)rank));
    // MP group: contiguous ranks {g*N .. g*N+N-1}; DP group: {l, l+N, ...}
    S2D_NCCL(ncclCommSplit(world.nccl, (int)group, (int)local, &mp.nccl, nullptr));
    S2D_NCCL(ncclCommSplit(world.nccl, (int)local, (int)group, &dp.nccl, nullptr));
  }
  world.n = T;
  world.me = rank;
  mp.n = N;
  mp.me = local;
  dp.n = M;
  dp.me = group;
}

void Ctx::register_tables(const s2d_table_desc* t, uint32_t n, const s2d_plan_entry* p, uint32_t np,
                          int dtype) {
  if (n == 0) throw Error(S2D_EINVAL, "at least one table required");
  if (dtype != S2D_F32 && dtype != S2D_BF16) throw Error(S2D_EINVAL, "weight dtype must be F32 or BF16");
  S2D_CUDA(cudaSetDevice(device));
  tables.assign(t, t + n);
  plan.assign(p, p + np);
  F = n;
  bf16 = dtype == S2D_BF16;
  feats.assign(F, FeatDev{});
  ranges.clear();
  sum_dims = 0;
  max_dim = 0;
  any_mean = false;
  for (uint32_t f = 0; f < F; ++f) {
    const auto& d = tables[f];
    if (d.table_id != f) throw Error(S2D_EINVAL, "table_id must equal its index");
    if (d.rows < 1 || d.dim < 1) throw Error(S2D_EINVAL, "table needs rows >= 1 and dim >= 1");
    if (d.dim % 4 || d.dim > (uint32_t)kMaxDim)
      throw Error(S2D_EINVAL, "dim must be a multiple of 4 and <= 512 (table " + std::to_string(f) + ")");
    if (d.pooling != S2D_POOL_SUM && d.pooling != S2D_POOL_MEAN)
      throw Error(S2D_EINVAL, "pooling must be S2D_POOL_SUM or S2D_POOL_MEAN (table " + std::to_string(f) + ")");
    feats[f].dim = d.dim;
    feats[f].mean = d.pooling == S2D_POOL_MEAN ? 1u : 0u;
    any_mean = any_mean || feats[f].mean;
    feats[f].rows = d.rows;
    feats[f].coff = sum_dims;
    sum_dims += d.dim;
    max_dim = std::max(max_dim, d.dim);
  }
  // plan: coverage + ownership (validate_plan semantics)
  std::vector<s2d_table_load_profile> prof(F);
  for (uint32_t f = 0; f < F; ++f) prof[f] = {f, (uint64_t)tables[f].rows * tables[f].dim * 4, 0.0, tables[f].rows};
  validate_plan(plan, N, prof);
  n_slots = 0;
  n_weight_elems = 0;
  for (uint32_t f = 0; f < F; ++f) {
    std::vector<s2d_plan_entry> mine;
    for (const auto& e : plan)
      if (e.table_id == f) mine.push_back(e);
    std::sort(mine.begin(), mine.end(), [](const s2d_plan_entry& a, const s2d_plan_entry& b) { return a.row_lo < b.row_lo; });
    feats[f].rbeg = (uint32_t)ranges.size();
    bool owned = false;
    for (const auto& e : mine) {
      ranges.push_back({e.row_lo, e.row_hi, e.local_rank, 0});
      if (e.local_rank == local) {
        if (owned) throw Error(S2D_EINVAL, "a local rank may own at most one range per table");
        owned = true;
        feats[f].lo = e.row_lo;
        feats[f].hi = e.row_hi;
      }
    }
    feats[f].rend = (uint32_t)ranges.size();
    feats[f].single = mine.size() == 1 ? 1u : 0u;
    feats[f].vbase = n_slots;
    feats[f].wbase = n_weight_elems;
    const uint64_t own = feats[f].hi - feats[f].lo;
    if ((uint64_t)n_slots + own >= 0xffffffffull) throw Error(S2D_EINVAL, "too many rows on one rank (>= 2^32-1)");
    n_slots += (uint32_t)own;
    n_weight_elems += own * feats[f].dim;
  }
  all_same_dim = true;
  for (uint32_t f = 0; f < F; ++f) all_same_dim = all_same_dim && feats[f].dim == max_dim;
  uni_dim = 0;
  for (uint32_t f = 0; f < F; ++f)
    if (feats[f].hi > feats[f].lo) {
      if (uni_dim == 0) uni_dim = feats[f].dim;
      else if (uni_dim != feats[f].dim) uni_dim = 0xffffffffu;
    }
  if (uni_dim == 0xffffffffu) uni_dim = 0;
  vbase_sorted.clear();
  feat_of_vbase.clear();
  for (uint32_t f = 0; f < F; ++f)
    if (feats[f].hi > feats[f].lo) {
      vbase_sorted.push_back(feats[f].vbase);
      feat_of_vbase.push_back(f);
    }
  if (vbase_sorted.empty()) {
    vbase_sorted.push_back(0);
    feat_of_vbase.push_back(0);
  }
  vbase_sorted.push_back(n_slots);
  d_feats.ensure(sizeof(FeatDev) * F);
  d_ranges.ensure(sizeof(RangeDev) * std::max<size_t>(1, ranges.size()));
  d_vbase_sorted.ensure(4 * vbase_sorted.size());
  d_feat_of_vbase.ensure(4 * feat_of_vbase.size());
  S2D_CUDA(cudaMemcpy(d_feats.p, feats.data(), sizeof(FeatDev) * F, cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d_ranges.p, ranges.data(), sizeof(RangeDev) * ranges.size(), cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d_vbase_sorted.p, vbase_sorted.data(), 4 * vbase_sorted.size(), cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d_feat_of_vbase.p, feat_of_vbase.data(), 4 * feat_of_vbase.size(), cudaMemcpyHostToDevice));
  // shard + padding: a zero row at slot n_slots (slot-indexed lookups of
  // invalid ids) and room for whole-warp row chunks past a short row
  const size_t pad_elems = 2 * (size_t)max_dim + 512;
  const size_t wbytes = (n_weight_elems + pad_elems) * (bf16 ? 2 : 4);
  slot_rows = all_same_dim;
  for (uint32_t f = 0; f < F && slot_rows; ++f) slot_rows = feats[f].wbase == (uint64_t)feats[f].vbase * max_dim;
  for (void* q : dp_opened) cudaIpcCloseMemHandle(q);  // mappings of the old replicas
  dp_opened.clear();
  dp_p2p = -1;
  weights.release();
  moments.release();
  dirty.release();
  weights.ensure(wbytes);
  moments.ensure(std::max<size_t>((size_t)n_slots * 4, 16));
  S2D_CUDA(cudaMemsetAsync(weights.p, 0, wbytes, stream));
  S2D_CUDA(cudaMemsetAsync(moments.p, 0, (size_t)n_slots * 4, stream));
  if (M > 1) {
    dirty.ensure(std::max<size_t>(n_slots, 16));
    S2D_CUDA(cudaMemsetAsync(dirty.p, 0, n_slots, stream));
  }
  S2D_CUDA(cudaStreamSynchronize(stream));
  if (N > 1) {  // collective: barrier flags and the count matrix
    peer_alloc(p_flags, (size_t)N * 8);
    peer_alloc(p_xcnt, (size_t)N * N * 3 * 8);
  }
  fwd_done = false;
}

void Ctx::set_optimizer(const s2d_optimizer_config& c) {
  check_optimizer(c);
  opt = c;
  have_opt = true;
}

void Ctx::init_tables(uint64_t seed) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  launch_init_rows(weights.p, bf16, feats.data(), F, seed, stream);
  S2D_CUDA(cudaMemsetAsync(moments.p, 0, (size_t)n_slots * 4, stream));
  if (M > 1) S2D_CUDA(cudaMemsetAsync(dirty.p, 0, n_slots, stream));
  finish_call();
}

void Ctx::shard_io(uint32_t table, uint32_t lo, uint32_t hi, float* w, float* v, bool write) {
  if (table >= F) throw Error(S2D_EINVAL, "table out of range");
  const FeatDev& fd = feats[table];
  if (lo > hi || lo < fd.lo || hi > fd.hi)
    throw Error(S2D_ERANGE, "rows [" + std::to_string(lo) + "," + std::to_string(hi) + ") outside owned range [" +
                                std::to_string(fd.lo) + "," + std::to_string(fd.hi) + ") of table " +
                                std::to_string(table));
  if (hi == lo) return;
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  S2D_CUDA(cudaStreamSynchronize(stream));
  const uint64_t n = (uint64_t)(hi - lo) * fd.dim;
  const uint64_t off = fd.wbase + (uint64_t)(lo - fd.lo) * fd.dim;
  if (w) {
    if (!bf16) {
      float* dst = weights.as<float>() + off;
      if (write)
        S2D_CUDA(cudaMemcpy(dst, w, n * 4, cudaMemcpyHostToDevice));
      else
        S2D_CUDA(cudaMemcpy(w, dst, n * 4, cudaMemcpyDeviceToHost));
    } else {
      std::vector<uint16_t> tmp(n);
      uint16_t* dst = weights.as<uint16_t>() + off;
      if (write) {
        for (uint64_t i = 0; i < n; ++i) {  // round-to-nearest-even f32 -> bf16
          uint32_t x;
          std::memcpy(&x, &w[i], 4);
          if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x7fffffu))
            tmp[i] = (uint16_t)((x >> 16) | 0x40);
          else
            tmp[i] = (uint16_t)((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
        }
        S2D_CUDA(cudaMemcpy(dst, tmp.data(), n * 2, cudaMemcpyHostToDevice));
      } else {
        S2D_CUDA(cudaMemcpy(tmp.data(), dst, n * 2, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < n; ++i) {
          const uint32_t x = (uint32_t)tmp[i] << 16;
          std::memcpy(&w[i], &x, 4);
        }
      }
    }
  }
  if (write && M > 1) {  // written rows join the next replica sync's dirty union
    S2D_CUDA(cudaMemset(dirty.as<uint8_t>() + fd.vbase + (lo - fd.lo), 1, hi - lo));
    snap_broken = true;  // not in the snapshot log: the next sync exchanges every union row
    dirty_clean = false;
    list_ready = false;
  }
  if (v) {
    float* dst = moments.as<float>() + fd.vbase + (lo - fd.lo);
    if (write)
      S2D_CUDA(cudaMemcpy(dst, v, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice));
    else
      S2D_CUDA(cudaMemcpy(v, dst, (size_t)(hi - lo) * 4, cudaMemcpyDeviceToHost));
  }
}

void Ctx::apply_row_updates(uint32_t table, uint32_t n, const uint32_t* rows, const double* delta,
                            const double* new_moment) {
  if (table >= F) throw Error(S2D_EINVAL, "table out of range");
  if (!n) return;
  if (!rows || !delta || !new_moment) throw Error(S2D_EINVAL, "null rows / delta / new_moment");
  const FeatDev& fd = feats[table];
  // every row validated before any write (the reference throws per call,
  // embedding.cpp:110-121; a batch is all-or-nothing)
  for (uint32_t i = 0; i < n; ++i) {
    if (rows[i] < fd.lo || rows[i] >= fd.hi)
      throw Error(S2D_ERANGE, "row " + std::to_string(rows[i]) + " outside shard range [" + std::to_string(fd.lo) +
                                  "," + std::to_string(fd.hi) + ")");
    if (!(new_moment[i] >= 0.0) || !std::isfinite(new_moment[i]))
      throw Error(S2D_EINVAL, "new_moment must be finite and >= 0 (got " + std::to_string(new_moment[i]) + ")");
  }
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return rows[a] < rows[b]; });
  std::vector<uint32_t> seg, seg_row;
  for (uint32_t k = 0; k < n; ++k)
    if (k == 0 || rows[order[k]] != rows[order[k - 1]]) {
      seg.push_back(k);
      seg_row.push_back(rows[order[k]] - fd.lo);
    }
  const uint32_t nseg = (uint32_t)seg.size();
  seg.push_back(n);
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  S2D_CUDA(cudaStreamSynchronize(stream));
  const size_t b_order = (size_t)n * 4, b_seg = seg.size() * 4, b_row = (size_t)nseg * 4;
  const size_t b_delta = (size_t)n * fd.dim * 8, b_mom = (size_t)n * 8;
  const size_t o_seg = b_order, o_row = o_seg + b_seg, o_delta = (o_row + b_row + 7) / 8 * 8,
               o_mom = o_delta + b_delta;
  row_upd_scratch.ensure(o_mom + b_mom);
  char* d = row_upd_scratch.as<char>();
  S2D_CUDA(cudaMemcpy(d, order.data(), b_order, cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d + o_seg, seg.data(), b_seg, cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d + o_row, seg_row.data(), b_row, cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d + o_delta, delta, b_delta, cudaMemcpyHostToDevice));
  S2D_CUDA(cudaMemcpy(d + o_mom, new_moment, b_mom, cudaMemcpyHostToDevice));
  void* wbase = bf16 ? (void*)(weights.as<uint16_t>() + fd.wbase) : (void*)(weights.as<float>() + fd.wbase);
  // M > 1: the rows written here join the next replica sync's dirty union
  // (the sync averages only dirty rows, so an unflagged write would leave
  // the replicas different)
  launch_apply_rows(wbase, bf16, moments.as<float>() + fd.vbase, reinterpret_cast<uint32_t*>(d),
                    reinterpret_cast<uint32_t*>(d + o_seg), reinterpret_cast<uint32_t*>(d + o_row),
                    reinterpret_cast<double*>(d + o_delta), reinterpret_cast<double*>(d + o_mom), nseg, fd.dim,
                    M > 1 ? dirty.as<uint8_t>() + fd.vbase : nullptr, stream);
  if (M > 1) {
    snap_broken = true;  // not in the snapshot log (see shard_io)
    dirty_clean = false;
    list_ready = false;
  }
  S2D_CUDA(cudaStreamSynchronize(stream));
}

// Rows `rows` (global ids of `table`, owned here) -> f32 weights + moments
// (bf16 widened exactly); S2D_ERANGE for a row outside the owned range.
void Ctx::gather_rows(uint32_t table, uint32_t n, const uint32_t* rows, float* w, float* v) {
  if (table >= F) throw Error(S2D_EINVAL, "table out of range");
  if (!n) return;
  if (!rows) throw Error(S2D_EINVAL, "null rows");
  const FeatDev& fd = feats[table];
  std::vector<uint32_t> loc(n);
  for (uint32_t i = 0; i < n; ++i) {
    if (rows[i] < fd.lo || rows[i] >= fd.hi)
      throw Error(S2D_ERANGE, "row " + std::to_string(rows[i]) + " outside owned range [" + std::to_string(fd.lo) +
                                  "," + std::to_string(fd.hi) + ")");
    loc[i] = rows[i] - fd.lo;
  }
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  S2D_CUDA(cudaStreamSynchronize(stream));
  const size_t bw = (size_t)n * fd.dim * 4, bv = (size_t)n * 4;
  gather_scratch.ensure(bw + bv + (size_t)n * 4 + 64);
  char* d = gather_scratch.as<char>();
  float* dw = reinterpret_cast<float*>(d);
  float* dv = reinterpret_cast<float*>(d + bw);
  uint32_t* dr = reinterpret_cast<uint32_t*>(d + bw + bv);
  S2D_CUDA(cudaMemcpy(dr, loc.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
  const void* wb = bf16 ? (const void*)(weights.as<uint16_t>() + fd.wbase) : (const void*)(weights.as<float>() + fd.wbase);
  launch_gather_rows(wb, bf16, moments.as<float>() + fd.vbase, dr, n, fd.dim, dw, dv, stream);
  S2D_CUDA(cudaStreamSynchronize(stream));
  if (w) S2D_CUDA(cudaMemcpy(w, dw, bw, cudaMemcpyDeviceToHost));
  if (v) S2D_CUDA(cudaMemcpy(v, dv, bv, cudaMemcpyDeviceToHost));
}

void Ctx::check_faults() {
  const uint32_t e = *err_host.as<uint32_t>();
  if (!e) return;
  *err_host.as<uint32_t>() = 0;
  S2D_CUDA(cudaMemsetAsync(err.p, 0, 4, stream));
  stats.error_flags = e;
  if (e & kErrIdRange) throw Error(S2D_ERANGE, "lookup id outside the table's rows / shard ranges");
  if (e & kErrNonfinite) throw Error(S2D_ENONFINITE, "nonfinite row gradient");
  if (e & kErrPeerTimeout) throw Error(S2D_ENCCL, "peer barrier timed out (a rank of the MP group stopped)");
}

void Ctx::finish_call() {
  // strict: wait and raise now; otherwise faults surface at s2d_synchronize
  // (no copy node here: it would break the kernels' PDL chain across calls)
  if (strict) synchronize_and_check();
}

void Ctx::synchronize_and_check() {
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  S2D_CUDA(cudaStreamSynchronize(h2d_stream));
  S2D_CUDA(cudaStreamSynchronize(d2h_stream));
  S2D_CUDA(cudaStreamSynchronize(sort_stream));
  S2D_CUDA(cudaMemcpyAsync(err_host.p, err.p, 4, cudaMemcpyDeviceToHost, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  check_faults();
}

// ---- forward -------------------------------------------------------------

void Ctx::lookup_forward(uint32_t batch, const uint32_t* lengths, const uint32_t* ids, uint64_t nnz,
                         float* pooled, int mem) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (batch == 0) throw Error(S2D_EINVAL, "batch must be >= 1");
  if (nnz >= 0xffffffffull) throw Error(S2D_EINVAL, "nnz must be < 2^32-1 per rank");
  if (mem != S2D_HOST && mem != S2D_DEVICE) throw Error(S2D_EINVAL, "mem must be S2D_HOST or S2D_DEVICE");
  S2D_CUDA(cudaSetDevice(device));
  B = batch;
  nnz_local = nnz;
  const uint64_t BF = (uint64_t)B * F;
  stats = s2d_step_stats{};
  stats_counters_valid = false;
  sync_stats_pending = false;  // the counters describe this step from here on
  stats.nnz_local = nnz;
  if (sort_pending) {  // a forward without its backward: its sort still reads the keys
    S2D_CUDA(cudaStreamWaitEvent(stream, ev_sorted, 0));
    sort_pending = false;
  }
  if (N == 1) join_sync();  // the lookup below reads the weights (N > 1: after the id exchange)
  // stage inputs
  phase_begin(kPhInput);
  const uint32_t* d_len = lengths;
  const uint32_t* d_ids = ids;
  float* d_pooled = pooled;
  // zero-copy output: pooled == NULL (device mode) selects the engine-owned,
  // peer-mapped pooled buffer (s2d_pooled_buffer); owners of single-owner
  // tables then store pooled rows straight into it over NVLink
  const bool engine_out = (mem == S2D_DEVICE && pooled == nullptr) || mem == S2D_HOST;
  // N > 1: the peer-mapped pooled buffer is (re)allocated by every rank
  // whatever its own output mode, so the collective growth decisions of the
  // group never depend on a per-rank choice (B itself must agree across the
  // MP group; read_counts checks it every step)
  if (N > 1) peer_alloc(p_pooled, (uint64_t)B * sum_dims * 4);
  // N == 1 host mode: the read-back alternates between two staging buffers,
  // so this step's lookup runs while the previous step's rows still travel
  // to the host (the buffer written now was last read back two steps ago)
  const bool host_pair = mem == S2D_HOST && N == 1;
  if (host_pair) {
    out_sel ^= 1;
    if (d2h_done_rec[out_sel]) S2D_CUDA(cudaStreamWaitEvent(stream, ev_d2h_done[out_sel], 0));
    p_pooled_host[out_sel].ensure((uint64_t)B * sum_dims * 4);
    d_pooled = p_pooled_host[out_sel].as<float>();
  } else if (engine_out) {
    if (d2h_pending) S2D_CUDA(cudaStreamWaitEvent(stream, ev_d2h, 0));  // last read-back of the buffer
    if (N == 1) p_pooled_local.ensure((uint64_t)B * sum_dims * 4);
    d_pooled = N > 1 ? p_pooled.buf.as<float>() : p_pooled_local.as<float>();
  }
  if (mem == S2D_HOST) {
    // ids + lengths go up on the H2D copy stream into one of two staging
    // pairs (the one this forward's predecessor-but-one read), so the upload
    // overlaps the previous step's update; the compute stream waits here
    in_sel ^= 1;
    DevBuf& bl = in_len2[in_sel];
    DevBuf& bi = in_ids2[in_sel];
    bl.ensure(BF * 4);
    bi.ensure(std::max<uint64_t>(nnz, 1) * 4);
    if (in_used_rec[in_sel]) S2D_CUDA(cudaStreamWaitEvent(h2d_stream, ev_in_used[in_sel], 0));
    S2D_CUDA(cudaMemcpyAsync(bl.p, lengths, BF * 4, cudaMemcpyHostToDevice, h2d_stream));
    if (nnz) S2D_CUDA(cudaMemcpyAsync(bi.p, ids, nnz * 4, cudaMemcpyHostToDevice, h2d_stream));
    S2D_CUDA(cudaEventRecord(ev_in_ready, h2d_stream));
    S2D_CUDA(cudaStreamWaitEvent(stream, ev_in_ready, 0));
    d_len = bl.as<uint32_t>();
    d_ids = bi.as<uint32_t>();
  }
  scan_tmp.ensure(scan_tmp_bytes(std::max<uint64_t>((uint64_t)N * BF, nnz) + 1));
  in_off.ensure((BF + 1) * 4);
  scan_u32_to_u32(d_len, in_off.as<uint32_t>(), BF, stream, scan_tmp.p, scan_tmp.cap);
  const FeatDev* dfe = d_feats.as<FeatDev>();

  if (N == 1) {
    phase_begin(kPhLookup);
    nnz_own = nnz;
    keys_a.ensure(std::max<uint64_t>(nnz, 1) * 4);
    vals_a.ensure(std::max<uint64_t>(nnz, 1) * 4);
    LookupArgs a{};
    a.feats = dfe;
    a.F = F;
    a.B = B;
    a.n_req = 1;
    a.sum_dims = sum_dims;
    a.lengths = d_len;
    a.id_off = in_off.as<uint32_t>();
    a.ids = d_ids;
    a.weights = weights.p;
    a.out = d_pooled;
    a.eoff = nullptr;
    a.keys = keys_a.as<uint32_t>();
    a.vals = vals_a.as<uint32_t>();
    a.err = err.as<uint32_t>();
    a.direct = 1;
    // S2D_SORT_BESIDE=1: the sort pairs come from a pass over the ids and
    // the sort runs on the side stream beside the lookup (experiment)
    static const bool beside = [] {
      const char* e = std::getenv("S2D_SORT_BESIDE");
      return e && e[0] == '1';
    }();
    static const uint32_t lookup_bps = [] {
      const char* e = std::getenv("S2D_LOOKUP_BPS");
      return e ? (uint32_t)std::atoi(e) : 0u;
    }();
    a.emit_keys = beside ? 0 : 1;
    a.blocks_per_sm = lookup_bps;
    a.uni_d4 = all_same_dim ? max_dim / 4 : 0;
    a.uni_rows = slot_rows ? 1 : 0;
    a.zero_row = n_slots;
    counters.ensure(64);
    a.ticket = counters.as<uint32_t>() + 8;
    if (beside && nnz) {
      launch_emit_pairs(dfe, F, B, sum_dims, in_off.as<uint32_t>(), d_ids, keys_a.as<uint32_t>(),
                        vals_a.as<uint32_t>(), stream);
      S2D_CUDA(cudaEventRecord(ev_keys, stream));
      S2D_CUDA(cudaStreamWaitEvent(sort_stream, ev_keys, 0));
      launch_sort(sort_stream);
      S2D_CUDA(cudaEventRecord(ev_sorted, sort_stream));
      sort_pending = true;
    }
    launch_lookup_stream(a, bf16, (int)max_dim, stream);
    stats.nnz_owned = nnz;
    stats.entries_owned = BF;
  } else {
    // ---- K1 fused with the id all-to-all over NVLink peer memory ----
    phase_begin(kPhBucket);
    peer_alloc(p_len, (uint64_t)N * BF * 4);  // collective; B is uniform across ranks
    cnt.ensure((uint64_t)N * BF * 4);
    send_off.ensure(((uint64_t)N * BF + 1) * 4);
    eoff_req.ensure(((uint64_t)N * BF + 1) * 8);
    BucketArgs ba{};
    ba.feats = dfe;
    ba.ranges = d_ranges.as<RangeDev>();
    ba.F = F;
    ba.BF = (uint32_t)BF;
    ba.N = N;
    ba.lengths = d_len;
    ba.id_off = in_off.as<uint32_t>();
    ba.ids = d_ids;
    ba.cnt = cnt.as<uint32_t>();
    ba.send_off = send_off.as<uint32_t>();
    ba.err = err.as<uint32_t>();
    ba.me = local;
    ba.peer_len = ptrs(p_len);
    launch_bucket_count(ba, stream);  // also stores cnt[o][:] into owner o's receive lengths
    scan_count_pair(cnt.as<uint32_t>(), send_off.as<uint32_t>(), eoff_req.as<uint64_t>(), (uint64_t)N * BF, F, dfe,
                    stream, scan_tmp.p, scan_tmp.cap);
    // the batch word carries this requester's output mode: owners store
    // single-owner pooled rows straight into a requester's pooled buffer
    // only when that requester asked for the engine-owned output
    launch_publish_counts(send_off.as<uint32_t>(), eoff_req.as<uint64_t>(), N, BF,
                          (uint64_t)B | (engine_out ? kEngineOutFlag : 0ull), ptrs(p_xcnt), local, stream);
    peer_barrier();
    phase_begin(kPhCountSync);
    read_counts();  // count matrix -> offsets; grows the peer buffers collectively
    phase_begin(kPhA2AIds);
    ba.peer_ids = ptrs(p_ids);
    for (uint32_t o = 0; o < N; ++o) ba.ids_adj[o] = (int64_t)ids_base_at_owner[o] - (int64_t)send_bound[o];
    launch_bucket_permute(ba, stream);  // ids straight into the owners' receive buffers
    peer_barrier();
    // ---- owner side: partial pools written into the requesters' buffers ----
    own_idoff.ensure(((uint64_t)N * BF + 1) * 4);
    own_eoff.ensure(((uint64_t)N * BF + 1) * 8);
    scan_count_pair(p_len.buf.as<uint32_t>(), own_idoff.as<uint32_t>(), own_eoff.as<uint64_t>(), (uint64_t)N * BF, F,
                    dfe, stream, scan_tmp.p, scan_tmp.cap);
    keys_a.ensure(std::max<uint64_t>(nnz_own, 1) * 4);
    vals_a.ensure(std::max<uint64_t>(nnz_own, 1) * 4);
    LookupArgs a{};
    a.feats = dfe;
    a.F = F;
    a.B = B;
    a.n_req = N;
    a.sum_dims = sum_dims;
    a.lengths = p_len.buf.as<uint32_t>();
    a.id_off = own_idoff.as<uint32_t>();
    a.ids = p_ids.buf.as<uint32_t>();
    a.weights = weights.p;
    a.out = nullptr;
    a.eoff = own_eoff.as<uint64_t>();
    a.keys = keys_a.as<uint32_t>();
    a.vals = vals_a.as<uint32_t>();
    a.err = err.as<uint32_t>();
    a.direct = 0;
    a.emit_keys = 1;
    a.uni_d4 = all_same_dim ? max_dim / 4 : 0;
    a.uni_rows = slot_rows ? 1 : 0;
    a.zero_row = n_slots;
    a.peer_out = ptrs(p_part);
    a.use_peer_pooled = (int)engine_mask;  // per requester (bit n), from the count matrix
    a.peer_pooled = ptrs(p_pooled);
    for (uint32_t n = 0; n < N; ++n) a.peer_adj[n] = (int64_t)part_base_at_req[n] - (int64_t)own_eoff_bound[n];
    counters.ensure(64);
    a.ticket = counters.as<uint32_t>() + 8;
    a.unit_rot = ((uint64_t)((local + 1) % N) * BF) / 32;  // start at the next requester
    join_sync();  // the bucketing and id exchange above overlapped the last replica sync's tail
    phase_begin(kPhLookup);
    launch_lookup_stream(a, bf16, (int)max_dim, stream);
    // the gradient rows' (slot, offset) pairs are final: sort them now
    S2D_CUDA(cudaEventRecord(ev_keys, stream));
    S2D_CUDA(cudaStreamWaitEvent(sort_stream, ev_keys, 0));
    launch_sort(sort_stream);
    S2D_CUDA(cudaEventRecord(ev_sorted, sort_stream));
    sort_pending = true;
    phase_begin(kPhA2ALookup);
    peer_barrier();  // every owner's partials have landed in p_part
    phase_begin(kPhCombine);
    CombineArgs ca{};
    ca.feats = dfe;
    ca.F = F;
    ca.B = B;
    ca.N = N;
    ca.sum_dims = sum_dims;
    ca.cnt = cnt.as<uint32_t>();
    ca.eoff = eoff_req.as<uint64_t>();
    ca.recv = p_part.buf.as<float>();
    ca.pooled = d_pooled;
    ca.skip_single = engine_out ? 1 : 0;
    ca.bag_off = in_off.as<uint32_t>();
    launch_combine(ca, (int)max_dim, stream);
    phase_end();  // the gap until the backward call is no phase
    uint64_t ef_own = 0, sent = 0, recv = 0;
    for (uint32_t q = 0; q < N; ++q) {
      ef_own += ef_from[q];
      if (q == local) continue;
      sent += nnz_to[q] * 4 + BF * 4 + ef_from[q] * 4;
      recv += nnz_from[q] * 4 + BF * 4 + ef_to[q] * 4;
      stats.ids_bytes_sent += nnz_to[q] * 4 + BF * 4;
      stats.lookup_bytes_sent += ef_from[q] * 4;
    }
    stats.nnz_owned = nnz_own;
    stats.entries_owned = ef_own / std::max<uint32_t>(1, max_dim);
    stats.a2a_bytes_sent = sent;
    stats.a2a_bytes_recv = recv;
  }
  if (mem == S2D_HOST) {
    // every reader of this forward's input staging is queued: the next
    // upload into it waits for this point
    S2D_CUDA(cudaEventRecord(ev_in_used[in_sel], stream));
    in_used_rec[in_sel] = true;
    // read-back on the D2H stream: overlaps the upstream upload, the sort and
    // the update (and, N == 1, the next step's lookup)
    S2D_CUDA(cudaEventRecord(ev_fwd, stream));
    S2D_CUDA(cudaStreamWaitEvent(d2h_stream, ev_fwd, 0));
    S2D_CUDA(cudaMemcpyAsync(pooled, d_pooled, (uint64_t)B * sum_dims * 4, cudaMemcpyDeviceToHost, d2h_stream));
    if (host_pair) {
      S2D_CUDA(cudaEventRecord(ev_d2h_done[out_sel], d2h_stream));
      d2h_done_rec[out_sel] = true;
    } else {
      S2D_CUDA(cudaEventRecord(ev_d2h, d2h_stream));
      d2h_pending = true;
    }
    if (!async_host) S2D_CUDA(cudaStreamSynchronize(d2h_stream));
  }
  phase_end();
  fwd_done = true;
  finish_call();
}

// ---- MP-group peer memory -------------------------------------------------

PeerPtrs Ctx::ptrs(const PeerBuf& pb) const {
  PeerPtrs pp{};
  for (uint32_t q = 0; q < pb.ptr.size() && q < (uint32_t)kMaxPeers; ++q) pp.p[q] = pb.ptr[q];
  return pp;
}

// Collective over the MP group: every rank calls it with the same `bytes`
// (derived from data all ranks share), so growth decisions agree.
void Ctx::peer_alloc(PeerBuf& pb, size_t bytes) { peer_alloc_in(pb, bytes, mp); }

// Collective over `comm`: (re)allocate pb and map every member's copy
// (CUDA IPC across processes, plain pointers between virtual ranks).
void Ctx::peer_alloc_in(PeerBuf& pb, size_t bytes, Comm& comm) {
  if (pb.buf.p && bytes <= pb.cap) return;
  const size_t want = std::max<size_t>(bytes + bytes / 4, 4096);
  S2D_CUDA(cudaStreamSynchronize(stream));
  for (void* q : pb.opened) cudaIpcCloseMemHandle(q);
  pb.opened.clear();
  // everyone has unmapped the old buffers before anyone frees them
  comm.barrier(stream, hbuf);
  pb.buf.release();
  S2D_CUDA(cudaMalloc(&pb.buf.p, want));
  pb.buf.cap = want;
  pb.cap = want;
  S2D_CUDA(cudaMemsetAsync(pb.buf.p, 0, want, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  // every member must have asked for the same size (sizes derive from data
  // the group shares, e.g. the per-rank batch); a mismatch is a caller error
  std::vector<uint64_t> sizes(comm.n);
  const uint64_t mine = bytes;
  comm.host_allgather(&mine, 8, sizes.data(), stream, hbuf);
  for (uint64_t s : sizes)
    if (s != mine)
      throw Error(S2D_EINVAL, "MP group members disagree on a shared buffer size (per-rank batch / table set must "
                              "be identical in the group)");
  pb.ptr = map_peer_buffers(comm, pb.buf.p, device, stream, hbuf, pb.opened);
}

float* Ctx::pooled_buffer() {
  return N > 1 ? p_pooled.buf.as<float>() : p_pooled_local.as<float>();
}

// DP group over NVLink: map every replica's weights and moments (identical
// shard layout in every group) once; every member must agree, else the sync
// stays on the NCCL all-gather path (S2D_SYNC_NCCL=1 forces that path).
void Ctx::dp_setup() {
  if (dp_p2p >= 0) return;
  dp_p2p = 0;
  if (M <= 1) return;
  const char* e = std::getenv("S2D_SYNC_NCCL");
  if (e && e[0] == '1') return;
  S2D_CUDA(cudaStreamSynchronize(stream));
  dp_w.assign(M, nullptr);
  dp_v.assign(M, nullptr);
  int ok = 1;
  if (dp.local()) {
    dp_w = map_peer_buffers(dp, weights.p, device, stream, hbuf, dp_opened);
    dp_v = map_peer_buffers(dp, moments.p, device, stream, hbuf, dp_opened);
  } else {
    cudaIpcMemHandle_t h[2];
    S2D_CUDA(cudaIpcGetMemHandle(&h[0], weights.p));
    S2D_CUDA(cudaIpcGetMemHandle(&h[1], moments.p));
    std::vector<cudaIpcMemHandle_t> all((size_t)M * 2);
    dp.host_allgather(h, sizeof(h), all.data(), stream, hbuf);
    for (uint32_t g = 0; g < M && ok; ++g) {
      if (g == group) {
        dp_w[g] = weights.p;
        dp_v[g] = moments.p;
        continue;
      }
      for (int k = 0; k < 2 && ok; ++k) {
        void* m = nullptr;
        if (cudaIpcOpenMemHandle(&m, all[(size_t)g * 2 + k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          (void)cudaGetLastError();
          ok = 0;
          break;
        }
        dp_opened.push_back(m);
        (k == 0 ? dp_w : dp_v)[g] = m;
      }
    }
  }
  // agree across the group (min over members)
  std::vector<int32_t> oks(M);
  dp.host_allgather(&ok, 4, oks.data(), stream, hbuf);
  if (*std::min_element(oks.begin(), oks.end()) == 0) {
    for (void* q : dp_opened) cudaIpcCloseMemHandle(q);
    dp_opened.clear();
    return;
  }
  peer_alloc_in(dp_flags, (size_t)M * 8, dp);
  dp_p2p = 1;
}

// Virtual ranks of one process synchronise on the host (drain the stream,
// rendezvous on the hub): a kernel spinning on a peer that shares the GPU
// could wait behind that peer's host thread, which an implicitly
// device-synchronising runtime call (first-touch cudaMalloc / cudaMallocHost)
// can stall.  Across processes the barrier stays on the device.
void Ctx::dp_barrier(cudaStream_t st) {
  if (dp.local()) {
    dp.barrier(st, hbuf);
    return;
  }
  ++dp_epoch;
  launch_peer_barrier(ptrs(dp_flags), dp_flags.buf.as<uint64_t>(), group, M, dp_epoch, err.as<uint32_t>(), st);
}

void Ctx::peer_barrier() {
  if (mp.local()) {
    mp.barrier(stream, hbuf);
    return;
  }
  ++epoch;
  launch_peer_barrier(ptrs(p_flags), p_flags.buf.as<uint64_t>(), local, N, epoch, err.as<uint32_t>(), stream);
}

// Count matrix xcnt[n][o] = (ids n sends to o, partial floats of those
// entries, n's batch), published by every requester into every peer.
void Ctx::read_counts() {
  const size_t nx = (size_t)N * N * 3;
  h_xcnt.ensure(nx * 8);  // pinned: a pageable D2H would stage synchronously
  S2D_CUDA(cudaMemcpyAsync(h_xcnt.p, p_xcnt.buf.p, nx * 8, cudaMemcpyDeviceToHost, stream));
  const auto t0 = std::chrono::steady_clock::now();
  S2D_CUDA(cudaStreamSynchronize(stream));
  host_wait_total_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                            std::chrono::steady_clock::now() - t0).count();
  const uint64_t* x = h_xcnt.as<uint64_t>();
  auto at = [&](uint32_t n, uint32_t o, int k) { return x[((size_t)n * N + o) * 3 + k]; };
  engine_mask = 0;
  for (uint32_t n = 0; n < N; ++n) {
    const uint64_t bw = at(n, 0, 2);
    if ((bw & ~kEngineOutFlag) != B)
      throw Error(S2D_EINVAL, "per-rank batch must be identical in the MP group (" +
                                  std::to_string(bw & ~kEngineOutFlag) + " vs " + std::to_string(B) + ")");
    if (bw & kEngineOutFlag) engine_mask |= 1u << n;
  }
  nnz_to.assign(N, 0);
  ef_to.assign(N, 0);
  nnz_from.assign(N, 0);
  ef_from.assign(N, 0);
  send_bound.assign(N, 0);
  eoff_req_bound.assign(N, 0);
  own_eoff_bound.assign(N, 0);
  ids_base_at_owner.assign(N, 0);
  part_base_at_req.assign(N, 0);
  grad_base_at_owner.assign(N, 0);
  uint64_t need_ids = 0, need_part = 0, need_grad = 0;
  for (uint32_t r = 0; r < N; ++r) {
    uint64_t ids_in = 0, ef_in = 0, ef_out = 0;
    for (uint32_t q = 0; q < N; ++q) {
      ids_in += at(q, r, 0);
      ef_in += at(q, r, 1);
      ef_out += at(r, q, 1);
    }
    need_ids = std::max(need_ids, ids_in);
    need_grad = std::max(need_grad, ef_in);
    need_part = std::max(need_part, ef_out);
  }
  nnz_own = 0;
  uint64_t sb = 0, eb = 0, ob = 0;
  for (uint32_t q = 0; q < N; ++q) {
    nnz_to[q] = at(local, q, 0);
    ef_to[q] = at(local, q, 1);
    nnz_from[q] = at(q, local, 0);
    ef_from[q] = at(q, local, 1);
    send_bound[q] = sb;
    eoff_req_bound[q] = eb;
    own_eoff_bound[q] = ob;
    sb += nnz_to[q];
    eb += ef_to[q];
    ob += ef_from[q];
    nnz_own += nnz_from[q];
    for (uint32_t n = 0; n < local; ++n) {
      ids_base_at_owner[q] += at(n, q, 0);   // my block in owner q's id buffer
      grad_base_at_owner[q] += at(n, q, 1);  // ... and in its gradient buffer
    }
    for (uint32_t o = 0; o < local; ++o) part_base_at_req[q] += at(q, o, 1);  // my block in requester q's partials
  }
  if (nnz_own >= 0xffffffffull) throw Error(S2D_EINVAL, "owner demand exceeds 2^32-1 ids");
  peer_alloc(p_ids, std::max<uint64_t>(need_ids, 1) * 4);
  peer_alloc(p_part, std::max<uint64_t>(need_part, 4) * 4);
  peer_alloc(p_grad, std::max<uint64_t>(need_grad, 4) * 4);
}

// ---- backward + fused update ---------------------------------------------------

// K3a on `st`: stable radix sort of this rank's (slot, gradient offset)
// pairs; the sorted pairs land in (keys_c, vals_c).  (A dense-rank variant
// -- touched-slot bitmap, 2 passes of 10 bits -- measured no faster; see
// DESIGN.md section 5.)
void Ctx::launch_sort(cudaStream_t st) {
  const uint64_t n = nnz_own;
  if (n == 0) return;
  keys_b.ensure(n * 4);
  vals_b.ensure(n * 4);
  const int bits = std::max(1, bit_width(n_slots));
  sort_tmp.ensure(radix_tmp_bytes(n, bits));
  const bool in_b = radix_sort_pairs(keys_a.as<uint32_t>(), vals_a.as<uint32_t>(), keys_b.as<uint32_t>(),
                                     vals_b.as<uint32_t>(), n, bits, sort_tmp.p, sort_tmp.cap, st);
  sorted_k = in_b ? keys_b.as<uint32_t>() : keys_a.as<uint32_t>();
  sorted_v = in_b ? vals_b.as<uint32_t>() : vals_a.as<uint32_t>();
}

void Ctx::backward_update(const float* upstream, int mem) {
  if (!fwd_done) throw Error(S2D_EINVAL, "backward_update needs a preceding lookup_forward");
  if (!have_opt) throw Error(S2D_EINVAL, "set_optimizer first");
  if (mem != S2D_HOST && mem != S2D_DEVICE) throw Error(S2D_EINVAL, "mem must be S2D_HOST or S2D_DEVICE");
  S2D_CUDA(cudaSetDevice(device));
  if (M > 1) dp_setup();  // DP-group collective: every replica calls backward_update every step
  const uint64_t BF = (uint64_t)B * F;
  const float* d_up = upstream;
  phase_begin(kPhInput);
  bool up_wait = false;  // the compute stream still has to wait for the upload
  if (mem == S2D_HOST) {
    // upload on the H2D stream once the previous update stopped reading the
    // staging buffer; the compute stream waits only where rows are read
    up_sel ^= 1;  // two staging buffers: the upload overlaps the update that reads the other one
    up_stage2[up_sel].ensure((uint64_t)B * sum_dims * 4);
    if (up_used_rec[up_sel]) S2D_CUDA(cudaStreamWaitEvent(h2d_stream, ev_up_used[up_sel], 0));
    S2D_CUDA(cudaMemcpyAsync(up_stage2[up_sel].p, upstream, (uint64_t)B * sum_dims * 4, cudaMemcpyHostToDevice,
                             h2d_stream));
    S2D_CUDA(cudaEventRecord(ev_up, h2d_stream));
    d_up = up_stage2[up_sel].as<float>();
    up_wait = true;
  }
  const float* grad = d_up;
  if (N == 1 && any_mean && nnz_own > 0) {
    // mean-pooled tables: the bag's gradient row is f32(f64(up) * (1/L))
    // (the N > 1 gradient gather applies the same scale on its way out)
    if (up_wait) S2D_CUDA(cudaStreamWaitEvent(stream, ev_up, 0));
    up_wait = false;
    mean_stage.ensure((uint64_t)B * sum_dims * 4);
    launch_mean_prescale(d_feats.as<FeatDev>(), F, B, sum_dims, in_off.as<uint32_t>(), d_up, mean_stage.as<float>(),
                         stream);
    grad = mean_stage.as<float>();
  }
  if (N > 1) {
    if (up_wait) S2D_CUDA(cudaStreamWaitEvent(stream, ev_up, 0));
    up_wait = false;
    // C2 fused: gradient rows stored straight into the owners' buffers; the
    // owner's receive layout equals its partial send layout, so the
    // lookup's (slot, val) pairs index it.
    phase_begin(kPhGradGather);
    GradGatherArgs ga{};
    ga.feats = d_feats.as<FeatDev>();
    ga.ranges = d_ranges.as<RangeDev>();
    ga.F = F;
    ga.B = B;
    ga.N = N;
    ga.sum_dims = sum_dims;
    ga.cnt = cnt.as<uint32_t>();
    ga.eoff = eoff_req.as<uint64_t>();
    ga.upstream = d_up;
    ga.bag_off = in_off.as<uint32_t>();
    ga.peer_dst = ptrs(p_grad);
    for (uint32_t o = 0; o < N; ++o) ga.peer_adj[o] = (int64_t)grad_base_at_owner[o] - (int64_t)eoff_req_bound[o];
    launch_grad_gather(ga, (int)max_dim, stream);
    phase_begin(kPhA2AGrad);
    peer_barrier();
    grad = p_grad.buf.as<float>();
    uint64_t sent = 0, recv = 0;
    for (uint32_t q = 0; q < N; ++q) {
      if (q == local) continue;
      sent += ef_to[q] * 4;
      recv += ef_from[q] * 4;
    }
    stats.a2a_bytes_sent += sent;
    stats.grad_bytes_sent = sent;
    stats.a2a_bytes_recv += recv;
  }
  (void)BF;
  const uint64_t n = nnz_own;
  uint64_t uniq = 0;
  if (n > 0) {
    phase_begin(kPhSort);
    if (sort_pending)
      S2D_CUDA(cudaStreamWaitEvent(stream, ev_sorted, 0));
    else
      launch_sort(stream);
    sort_pending = false;
    const uint32_t* sk = sorted_k;
    const uint32_t* sv = sorted_v;
    phase_begin(kPhUpdate);
    if (up_wait) S2D_CUDA(cudaStreamWaitEvent(stream, ev_up, 0));
    up_wait = false;
    counters.ensure(64);
    chunk_part.ensure(stream_partial_bytes(n, max_dim));
    StreamUpdateArgs ua{};
    ua.keys = sk;
    ua.vals = sv;
    ua.n = n;
    ua.n_slots = n_slots;
    ua.feats = d_feats.as<FeatDev>();
    ua.vbase_sorted = d_vbase_sorted.as<uint32_t>();
    ua.feat_of_vbase = d_feat_of_vbase.as<uint32_t>();
    ua.n_feat_owned = (uint32_t)feat_of_vbase.size();
    ua.uni_dim = uni_dim;
    ua.max_d4 = max_dim / 4;
    ua.grad = grad;
    ua.weights = weights.p;
    ua.moments = moments.as<float>();
    ua.dirty = M > 1 ? dirty.as<uint8_t>() : nullptr;
    const uint64_t nparts1 = stream_partial1_rows(n);
    ua.part1 = chunk_part.as<double>();
    ua.part2 = chunk_part.as<double>() + nparts1 * max_dim;
    ua.part3 = ua.part2 + stream_partial2_rows(n) * max_dim;
    ua.inv_batch = 1.0 / (double)((uint64_t)N * B);  // group batch (trainer.cpp:462)
    ua.eta = opt.eta;
    ua.eps = opt.eps;
    ua.c = opt.c;
    {
      int ex = 0;
      const double mant = std::frexp(opt.c, &ex);
      ua.c_pow2 = std::isfinite(opt.c) && mant == 0.5 && ex > -1000 && ex < 1000;
      ua.inv_c = ua.c_pow2 ? std::ldexp(1.0, 1 - ex) : 0.0;
    }
    ua.sgd = opt.variant == S2D_SGD;
    ua.err = err.as<uint32_t>();
    ua.counters = counters.as<uint32_t>();
    if (debug_grad) {  // debug view of the row gradients (s2d_debug_read 7): head ordinals, one host read of U
      dbg_head.ensure((n + 1) * 4);
      scan_tmp.ensure(scan_tmp_bytes(n + 1));
      scan_heads_u32(sk, dbg_head.as<uint32_t>(), n, n_slots, stream, scan_tmp.p, scan_tmp.cap);
      uint32_t U = 0;
      S2D_CUDA(cudaMemcpyAsync(&U, dbg_head.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, stream));
      S2D_CUDA(cudaStreamSynchronize(stream));
      dbg_rows = U;
      dbg_grad.ensure(std::max<uint64_t>(U, 1) * max_dim * 8);
      S2D_CUDA(cudaMemsetAsync(dbg_grad.p, 0, std::max<uint64_t>(U, 1) * max_dim * 8, stream));
      ua.grad_dbg = dbg_grad.as<double>();
      ua.head_ord = dbg_head.as<uint32_t>();
    }
    // head ordinals (heads before each sorted position), scanned at most once
    bool have_ord = false;
    auto ensure_ord = [&] {
      if (have_ord) return;
      head_ord_buf.ensure((n + 1) * 4);
      scan_tmp.ensure(scan_tmp_bytes(n + 1));
      scan_heads_u32(sk, head_ord_buf.as<uint32_t>(), n, n_slots, stream, scan_tmp.p, scan_tmp.cap);
      have_ord = true;
    };
    if (!dev_total) {
      size_t fr = 0;
      S2D_CUDA(cudaMemGetInfo(&fr, &dev_total));
    }
    static const bool force_dense = [] {  // S2D_SNAP_DENSE=1: always the dense log (tests)
      const char* e = std::getenv("S2D_SNAP_DENSE");
      return e && e[0] == '1';
    }();
    // the snapshot log: indexed by a head's sorted position (it spans the
    // update's n items) while that fits a quarter of the device, else dense
    // (by the head's ordinal)
    const bool snap_path = snapshot_enabled() && !snap_broken;
    const bool dense = snap_path && (force_dense || (snap_ub + n) * (uint64_t)(max_dim + 4) * 4 > (uint64_t)dev_total / 4);
    // M = 2: the first update after a sync also writes this replica's
    // ascending dirty list, so the sync scans no dirty flags -- worth it when
    // the flags (one byte per owned row) outweigh the scan of the sorted keys
    // (measured: config 4 2x2 1.875 -> 1.713 ms; config 3 2x2 1.777 -> 1.849)
    // or when the dense log scans the keys anyway
    static const bool force_list = [] {  // S2D_SYNC_LIST=1: always (tests)
      const char* e = std::getenv("S2D_SYNC_LIST");
      return e && e[0] == '1';
    }();
    const bool want_list = M == 2 && dirty_clean && sync_list_mode_enabled() &&
                           (force_list || dense || (uint64_t)n_slots > 8 * n);
    if (want_list) {
      ensure_ord();
      dlist.ensure(std::max<uint64_t>(std::min<uint64_t>(n, n_slots), 1) * 4);
      ua.head_ord = head_ord_buf.as<uint32_t>();
      ua.dirty_list = dlist.as<uint32_t>();
    }
    if (snap_path) {
      uint64_t rows = n;
      if (dense) {  // one host read of the update's row count
        ensure_ord();
        uint32_t U = 0;
        S2D_CUDA(cudaMemcpyAsync(&U, head_ord_buf.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, stream));
        S2D_CUDA(cudaStreamSynchronize(stream));
        rows = U;
      }
      const uint64_t base = snap_reserve(rows);
      if (!snap_broken) {
        if (dense) ua.head_ord = head_ord_buf.as<uint32_t>();
        ua.snap_dense = dense ? 1 : 0;
        ua.snap = snap.as<float>();
        ua.snap_pos = snap_pos.as<uint32_t>();
        ua.snap_base = base;
        ua.snap_cap = snap_cap_rows;
        ua.snap_rf = max_dim + 4;
      }
    }
    launch_update_stream(ua, bf16, stream);
    if (M > 1) {
      list_ready = want_list;  // a second update before the sync dirties rows this list lacks
      list_n = n;
      dirty_clean = false;
    }
    uniq = 1;
  }
  (void)uniq;
  if (up_wait) S2D_CUDA(cudaStreamWaitEvent(stream, ev_up, 0));  // n == 0: nothing read it
  if (mem == S2D_HOST) {
    S2D_CUDA(cudaEventRecord(ev_up_used[up_sel], stream));
    up_used_rec[up_sel] = true;
  }
  // N > 1: the step is complete when its update and its pooled read-back are
  // (the peer-mapped pooled buffer is written by the owners of the next step)
  if (d2h_pending) S2D_CUDA(cudaStreamWaitEvent(stream, ev_d2h, 0));
  phase_end();
  fwd_done = false;
  stats_counters_valid = n > 0;
  finish_call();
}

void Ctx::refresh_stats() {
  S2D_CUDA(cudaSetDevice(device));
  if (sync_stats_pending) {  // the last replica sync's union length (device-side count)
    join_sync();
    S2D_CUDA(cudaStreamSynchronize(stream));
    uint32_t cw[5] = {0, 0, 0, 0, 0};
    S2D_CUDA(cudaMemcpy(cw, sync_count.p, 20, cudaMemcpyDeviceToHost));
    // the union: counted on the device, or (pair sync) both lists less the rows both hold
    const uint32_t count = sync_snapshot_used ? (uint32_t)(sync_pair_rows - cw[4]) : cw[0];
    const uint64_t rf = max_dim + 4;
    const uint64_t lo = (uint64_t)count * group / M, hi = (uint64_t)count * (group + 1) / M;
    stats.dirty_rows = count;
    stats.sync_bytes = sync_snapshot_used ? sync_sent_rows * (M - 1) * rf * 4 + (uint64_t)sync_cmax * 4 * (M - 1)
                                          : 2 * (hi - lo) * (M - 1) * rf * 4 + (uint64_t)sync_cmax * 4 * (M - 1);
    sync_stats_pending = false;
  }
  if (!stats_counters_valid) return;
  S2D_CUDA(cudaStreamSynchronize(stream));
  uint32_t c[4];
  S2D_CUDA(cudaMemcpy(c, counters.p, 16, cudaMemcpyDeviceToHost));
  stats.unique_rows = c[0];
  stats.long_segments = c[1];
}

// ---- K5 replica sync ---------------------------------------------------------

// The weights / moments / dirty flags are final only once the previous
// replica sync's tail (on sync_stream) has run: every reader and writer of
// them on the main stream joins it first.
void Ctx::join_sync() {
  if (!sync_pending) return;
  S2D_CUDA(cudaStreamWaitEvent(stream, ev_sync_done, 0));
  sync_pending = false;
}

// S2D_SYNC_LIST=0 keeps the dirty-flag scans at M = 2 (A/B switch; =1 forces the list)
bool Ctx::sync_list_mode_enabled() const {
  static const bool off = [] {
    const char* e = std::getenv("S2D_SYNC_LIST");
    return e && e[0] == '0';
  }();
  return !off;
}

// S2D_SYNC_OVERLAP=0 keeps the sync tail on the main stream (A/B switch)
static bool sync_overlap_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("S2D_SYNC_OVERLAP");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool Ctx::snapshot_enabled() const {
  if (M != 2 || dp_p2p != 1) return false;  // the pair sync (M > 2: slice push / mean / scatter)
  static const bool off = [] {
    const char* e = std::getenv("S2D_SYNC_SNAPSHOT");
    return e && e[0] == '0';
  }();
  return !off;
}

// Room in the snapshot log for an update of at most `items` rows: its heads
// save at log row base + their ordinal (no atomics), so the interval's log
// spans every row its updates write (config 2: 0.45M rows, 0.23 GB per
// step; config 5 at B = 16384 on 2x2: 17.6M rows, 18 GB).  The log is held to a quarter of the device's memory and
// leaves the sync's staging plus a quarter of the device (at least 4 GB)
// free for the other buffers' growth; when it cannot grow the interval is
// marked broken (the sync then exchanges every union row, which needs no
// snapshot).  Returns base.
uint64_t Ctx::snap_reserve(uint64_t items) {
  if (snap_broken) return 0;
  const uint64_t rf = max_dim + 4;
  if (!snap_pos.p) snap_pos.ensure((size_t)n_slots * 4);
  const uint64_t base = snap_ub;
  const uint64_t need = snap_ub + items;
  if (need >= 0xffffffffull) {  // log positions are 32-bit
    snap_broken = true;
    return 0;
  }
  snap_ub = need;
  if (need <= snap_cap_rows) return base;
  size_t fr = 0, tot = 0;
  S2D_CUDA(cudaMemGetInfo(&fr, &tot));
  const uint64_t cap_rows = (uint64_t)tot / 4 / (rf * 4);  // a quarter of the device
  const uint64_t want = std::min<uint64_t>(std::min<uint64_t>(need + need / 4, 0xfffffffeull), cap_rows);
  void* p = nullptr;
  const uint64_t keep = std::max<uint64_t>(4ull << 30, (uint64_t)tot / 4);
  if (need > want ||
      (uint64_t)fr < (want + std::min<uint64_t>(items, n_slots)) * rf * 4 + keep ||
      cudaMalloc(&p, want * rf * 4) != cudaSuccess) {
    (void)cudaGetLastError();
    snap_broken = true;
    return 0;
  }
  if (base) S2D_CUDA(cudaMemcpyAsync(p, snap.p, base * rf * 4, cudaMemcpyDeviceToDevice, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  snap.release();
  snap.p = p;
  snap.cap = want * rf * 4;
  snap_cap_rows = want;
  return base;
}

void Ctx::replica_sync() {
  if (M <= 1 || !F) return;
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  phase_begin(kPhSync);
  // Union of the dirty rows across the DP group in O(dirty rows) wire bytes:
  // each replica compacts its own flags into an ascending slot list, the
  // lists are all-gathered, every replica flags the others' slots and
  // compacts again -> the same ascending union list everywhere.
  sync_tmp.ensure(flag_tmp_bytes(n_slots));
  sync_count.ensure(64 + (size_t)M * 20);
  uint32_t* d_count = sync_count.as<uint32_t>();
  uint32_t* d_counts = d_count + 16;      // [M] list lengths of the group
  uint32_t* d_gath = d_counts + M;        // [M][4] (list length, snapshot log complete, 0, 0)
  // this replica's (count, log complete): the snapshot sync runs only if
  // every replica's log saw every write of the interval
  const bool snap_on = snapshot_enabled();
  const uint32_t ok_word[3] = {(snap_on && !snap_broken && snap_pos.p) ? 1u : 0u, 0u, 0u};
  // this replica's dirty count: its update's row count when that update's
  // list is the whole dirty set, else a scan of the flags
  const bool use_list = list_ready;
  if (use_list)
    S2D_CUDA(cudaMemcpyAsync(d_count, head_ord_buf.as<uint32_t>() + list_n, 4, cudaMemcpyDeviceToDevice, stream));
  else
    launch_flag_count(dirty.as<uint8_t>(), n_slots, d_count, sync_tmp.p, sync_tmp.cap, stream);
  list_ready = false;
  dirty_clean = true;  // (after this sync; the early returns below included)
  S2D_CUDA(cudaMemcpyAsync(d_count + 1, ok_word, 12, cudaMemcpyHostToDevice, stream));
  dp.allgather(d_count, d_gath, 16, stream);
  S2D_CUDA(cudaMemcpyAsync(h_counts.p, d_gath, (size_t)M * 16, cudaMemcpyDeviceToHost, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  const uint32_t* hg = h_counts.as<uint32_t>();
  std::vector<uint32_t> hc(M);
  bool use_snap = snap_on;
  for (uint32_t g = 0; g < M; ++g) {
    hc[g] = hg[4 * g];
    use_snap = use_snap && hg[4 * g + 1] == 1;
  }
  const uint32_t mine = hc[group];
  uint32_t cmax = 0;
  for (uint32_t g = 0; g < M; ++g) cmax = std::max(cmax, hc[g]);
  // the next interval's log starts empty
  snap_ub = 0;
  snap_broken = false;
  if (cmax == 0) {
    stats.dirty_rows = 0;
    stats.sync_mode = 0;
    phase_end();
    finish_call();
    return;
  }
  sync_list.ensure((uint64_t)cmax * 4);
  if (use_list) {
    if (mine) S2D_CUDA(cudaMemcpyAsync(sync_list.p, dlist.p, (size_t)mine * 4, cudaMemcpyDeviceToDevice, stream));
  } else {
    launch_flag_write(dirty.as<uint8_t>(), n_slots, sync_list.as<uint32_t>(), sync_tmp.p, stream);
  }
  if (cmax > mine)  // pad to the longest list (0xffffffff is not a slot)
    S2D_CUDA(cudaMemsetAsync(sync_list.as<uint32_t>() + mine, 0xff, (size_t)(cmax - mine) * 4, stream));
  sync_lists.ensure((uint64_t)cmax * M * 4);
  dp.allgather(sync_list.p, sync_lists.p, (size_t)cmax * 4, stream);
  const uint32_t row_floats = max_dim + 4;  // row + moment, 16-byte pitch
  dp_setup();
  sync_snapshot_used = false;
  if (use_snap) {
    // Pair sync (M = 2, k_sync.cu): each replica sends the rows it dirtied
    // once -- the final mean of a row only it dirtied, its copy of a row
    // both dirtied -- into the peer's staging (its list order); after a
    // group barrier each replica stores / averages the peer's entries.
    const uint32_t peer = group ^ 1u;
    S2D_CUDA(cudaMemcpyAsync(d_counts, hc.data(), (size_t)M * 4, cudaMemcpyHostToDevice, stream));
    S2D_CUDA(cudaMemsetAsync(d_count + 4, 0, 4, stream));  // rows both replicas dirtied
    peer_alloc_in(dp_stage, (uint64_t)cmax * row_floats * 4, dp);  // same size everywhere
    const int sgd = opt.variant == S2D_SGD;
    const bool overlap = sync_overlap_enabled() && !dp.local() && !profile;
    cudaStream_t ts = stream;
    if (overlap) {
      S2D_CUDA(cudaEventRecord(ev_union, stream));
      S2D_CUDA(cudaStreamWaitEvent(sync_stream, ev_union, 0));
      ts = sync_stream;
    }
    const uint32_t* lists = sync_lists.as<uint32_t>();
    phase_begin(kPhSyncPush);
    launch_pair_push(reinterpret_cast<float*>(ptrs(dp_stage).p[peer]), group, lists + (uint64_t)group * cmax, d_counts,
                     lists + (uint64_t)peer * cmax, mine, d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(),
                     d_feat_of_vbase.as<uint32_t>(), (uint32_t)feat_of_vbase.size(), snap.as<float>(),
                     snap_pos.as<uint32_t>(), row_floats, weights.p, bf16, moments.as<float>(), sgd, d_count + 4, ts);
    dp_barrier(ts);  // the peer's entries have landed here
    phase_begin(kPhSyncMean);
    launch_pair_recv(dp_stage.buf.as<float>(), group, lists + (uint64_t)peer * cmax, d_counts, hc[peer],
                     d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(), d_feat_of_vbase.as<uint32_t>(),
                     (uint32_t)feat_of_vbase.size(), row_floats, weights.p, bf16, moments.as<float>(), sgd, ts);
    phase_begin(kPhSyncScatter);
    if (use_list)  // only this replica's rows carry a flag
      launch_clear_listed(dirty.as<uint8_t>(), dlist.as<uint32_t>(), d_counts + group, mine, ts);
    else
      launch_zero(dirty.p, n_slots, ts);
    if (overlap) {
      S2D_CUDA(cudaEventRecord(ev_sync_done, ts));
      sync_pending = true;
    }
    sync_stats_pending = true;
    sync_snapshot_used = true;
    stats.sync_mode = 1;
    sync_sent_rows = mine;
    sync_pair_rows = (uint64_t)hc[0] + hc[1];
    sync_cmax = cmax;
    phase_end();
    finish_call();
    return;
  }
  launch_mark_slots(sync_lists.as<uint32_t>(), (uint64_t)cmax * M, n_slots, dirty.as<uint8_t>(), stream);
  launch_flag_count(dirty.as<uint8_t>(), n_slots, d_count, sync_tmp.p, sync_tmp.cap, stream);
  if (dp_p2p == 1) {
    // The union's length stays on the device: every size below uses the
    // bound count_ub = min(M * cmax, n_slots), identical on every replica,
    // and the kernels read the count itself.  Every replica's update of this
    // step is complete (the list all-gather above ran after each replica's
    // update on its stream, and the host read its counts).  Slice s of the
    // union list is averaged by replica s.  Staging per replica:
    // [M][slice_cap] copies of its slice | [count_ub] means.
    const uint32_t count_ub = (uint32_t)std::min<uint64_t>((uint64_t)M * cmax, n_slots);
    sync_list.ensure((uint64_t)count_ub * 4);
    launch_flag_write(dirty.as<uint8_t>(), n_slots, sync_list.as<uint32_t>(), sync_tmp.p, stream);
    const uint64_t slice_cap = (uint64_t)count_ub / M + 1;
    const uint64_t copies = slice_cap * M * row_floats;
    peer_alloc_in(dp_stage, (copies + (uint64_t)count_ub * row_floats) * 4, dp);  // same size everywhere
    PeerPtrs means{};
    for (uint32_t g = 0; g < M; ++g) means.p[g] = reinterpret_cast<float*>(dp_stage.ptr[g]) + copies;
    const int sgd = opt.variant == S2D_SGD;
    // Across processes the push / mean / scatter tail runs on its own stream:
    // the next forward's bucketing and id exchange (which touch no weights)
    // overlap it, and its lookup waits for it (join_sync).  Virtual ranks
    // synchronise on the host, so their tail stays on the main stream, as
    // does a profiled one (its phases are timed on the main stream).
    const bool overlap = sync_overlap_enabled() && !dp.local() && !profile;
    cudaStream_t ts = stream;
    if (overlap) {
      S2D_CUDA(cudaEventRecord(ev_union, stream));
      S2D_CUDA(cudaStreamWaitEvent(sync_stream, ev_union, 0));
      ts = sync_stream;
    }
    phase_begin(kPhSyncPush);
    launch_p2p_push(ptrs(dp_stage), group, M, d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(),
                    d_feat_of_vbase.as<uint32_t>(), (uint32_t)feat_of_vbase.size(), sync_list.as<uint32_t>(), d_count,
                    count_ub, weights.p, bf16, moments.as<float>(), row_floats, slice_cap, ts);
    dp_barrier(ts);  // every copy of every slice is staged at its owner
    phase_begin(kPhSyncMean);
    launch_p2p_mean(dp_stage.buf.as<float>(), means, M, group, d_count, count_ub, row_floats, slice_cap, sgd, ts);
    dp_barrier(ts);  // every replica's staging holds every mean
    phase_begin(kPhSyncScatter);
    launch_p2p_scatter(d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(), d_feat_of_vbase.as<uint32_t>(),
                       (uint32_t)feat_of_vbase.size(), sync_list.as<uint32_t>(), d_count, count_ub,
                       dp_stage.buf.as<float>() + copies, row_floats, weights.p, bf16, moments.as<float>(), sgd, ts);
    launch_zero(dirty.p, n_slots, ts);
    if (overlap) {
      S2D_CUDA(cudaEventRecord(ev_sync_done, ts));
      sync_pending = true;
    }
    sync_stats_pending = true;  // dirty_rows / sync_bytes from the device count (refresh_stats)
    stats.sync_mode = 2;
    sync_cmax = cmax;
    phase_end();
    finish_call();
    return;
  }
  S2D_CUDA(cudaMemcpyAsync(h_counts.p, d_count, 4, cudaMemcpyDeviceToHost, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  const uint32_t count = *h_counts.as<uint32_t>();
  stats.dirty_rows = count;
  sync_list.ensure((uint64_t)count * 4);
  launch_flag_write(dirty.as<uint8_t>(), n_slots, sync_list.as<uint32_t>(), sync_tmp.p, stream);
  sync_packed.ensure((uint64_t)count * row_floats * 4);
  sync_gathered.ensure((uint64_t)count * row_floats * 4 * M);
  launch_pack_rows(d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(), d_feat_of_vbase.as<uint32_t>(),
                   (uint32_t)feat_of_vbase.size(), sync_list.as<uint32_t>(), d_count, weights.p, bf16,
                   moments.as<float>(), row_floats, sync_packed.as<float>(), count, stream);
  dp.allgather(sync_packed.p, sync_gathered.p, (size_t)count * row_floats * 4, stream);
  launch_mean_rows(d_feats.as<FeatDev>(), d_vbase_sorted.as<uint32_t>(), d_feat_of_vbase.as<uint32_t>(),
                   (uint32_t)feat_of_vbase.size(), sync_list.as<uint32_t>(), d_count, sync_gathered.as<float>(), M,
                   row_floats, count, weights.p, bf16, moments.as<float>(), opt.variant == S2D_SGD,
                   dirty.as<uint8_t>(), stream);
  stats.sync_bytes = (uint64_t)count * row_floats * 4 * (M - 1) + (uint64_t)cmax * 4 * (M - 1);
  stats.sync_mode = 3;
  phase_end();
  finish_call();
}

// ---- MetricsRow (trainer.cpp:745-771) ----------------------------------------

// Collective over the MP group: the moment statistics of this group's
// replica (group 0's is the reference's MetricsRow, which reads
// replicas[0]).  Exact k-th largest moment by a 4-round radix select over
// the group's shards (histograms all-gathered), then the reference's
// effective_lr and percentile index on the host.
void Ctx::metrics(s2d_metrics_row* out) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (!have_opt) throw Error(S2D_EINVAL, "set_optimizer first");
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  uint64_t n_total = 0;
  for (uint32_t f = 0; f < F; ++f) n_total += tables[f].rows;
  const uint32_t nb = moment_sum_blocks();
  metric_buf.ensure((size_t)(N + 1) * 256 * 4 + (size_t)nb * 8 + 64);
  uint32_t* d_hist = metric_buf.as<uint32_t>();
  uint32_t* d_all = d_hist + 256;
  double* d_part = reinterpret_cast<double*>(metric_buf.as<char>() + (size_t)(N + 1) * 256 * 4);
  // v_mean: per-rank block sums in index order, gathered and added in
  // (rank, block) order
  launch_moment_sum(moments.as<float>(), n_slots, d_part, stream);
  std::vector<double> parts((size_t)N * nb);
  {
    std::vector<double> mine(nb);
    S2D_CUDA(cudaMemcpyAsync(mine.data(), d_part, (size_t)nb * 8, cudaMemcpyDeviceToHost, stream));
    S2D_CUDA(cudaStreamSynchronize(stream));
    if (N > 1)
      mp.host_allgather(mine.data(), (size_t)nb * 8, parts.data(), stream, hbuf);
    else
      parts = mine;
  }
  double v_sum = 0.0;
  for (double p : parts) v_sum += p;
  // descending index k of the moments -> ascending rank n_total - 1 - k
  auto select = [&](uint64_t asc) -> float {
    uint32_t prefix = 0, mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      launch_moment_hist(moments.as<float>(), n_slots, shift, mask, prefix, d_hist, stream);
      std::vector<uint32_t> all((size_t)N * 256);
      if (N > 1) {
        mp.allgather(d_hist, d_all, 256 * 4, stream);
        S2D_CUDA(cudaMemcpyAsync(all.data(), d_all, all.size() * 4, cudaMemcpyDeviceToHost, stream));
      } else {
        S2D_CUDA(cudaMemcpyAsync(all.data(), d_hist, 256 * 4, cudaMemcpyDeviceToHost, stream));
      }
      S2D_CUDA(cudaStreamSynchronize(stream));
      uint64_t cum = 0;
      uint32_t digit = 255;
      for (uint32_t d = 0; d < 256; ++d) {
        uint64_t c = 0;
        for (uint32_t q = 0; q < N; ++q) c += all[(size_t)q * 256 + d];
        if (asc < cum + c) {
          digit = d;
          break;
        }
        cum += c;
      }
      asc -= cum;
      prefix |= digit << shift;
      mask |= 255u << shift;
    }
    float x;
    std::memcpy(&x, &prefix, 4);
    return x;
  };
  auto pct = [&](double q) {  // trainer.cpp:759-764 on the lr values
    const uint64_t idx = (uint64_t)std::ceil(q * (double)n_total) - 1;
    const float v = select(n_total - 1 - idx);
    return effective_lr((double)v, opt);
  };
  out->eff_lr_p50 = pct(0.50);
  out->eff_lr_p99 = pct(0.99);
  out->v_mean = v_sum / (double)n_total;
  out->rows = n_total;
}

// ---- debug views ------------------------------------------------------------

void Ctx::debug_read(int which, void* out, uint64_t cap, uint64_t* n) {
  S2D_CUDA(cudaSetDevice(device));
  join_sync();
  S2D_CUDA(cudaStreamSynchronize(stream));
  const uint64_t BF = (uint64_t)B * F;
  auto copy = [&](const void* src, uint64_t elems, size_t esz) {
    *n = elems;
    const uint64_t k = std::min(cap, elems);
    if (k && out) S2D_CUDA(cudaMemcpy(out, src, k * esz, cudaMemcpyDeviceToHost));
  };
  switch (which) {
    case 0:
      copy(p_len.buf.p, N == 1 ? 0 : (uint64_t)N * BF, 4);
      break;
    case 1:
      copy(p_ids.buf.p, N == 1 ? 0 : nnz_own, 4);
      break;
    case 2: {  // partials received from the owners, concatenated by owner
      uint64_t t = 0;
      for (auto q : ef_to) t += q;
      copy(p_part.buf.p, N == 1 ? 0 : t, 4);
      break;
    }
    case 3: {  // gradient rows received from the requesters, by requester
      uint64_t t = 0;
      for (auto q : ef_from) t += q;
      copy(p_grad.buf.p, N == 1 ? 0 : t, 4);
      break;
    }
    case 4: {
      std::vector<uint32_t> c((uint64_t)N * BF, 0), mask(BF, 0);
      if (N > 1) S2D_CUDA(cudaMemcpy(c.data(), cnt.p, c.size() * 4, cudaMemcpyDeviceToHost));
      for (uint64_t b = 0; b < BF; ++b)
        for (uint32_t o = 0; o < N; ++o)
          if (N == 1 || c[(uint64_t)o * BF + b]) mask[b] |= 1u << o;
      *n = BF;
      if (out) std::memcpy(out, mask.data(), std::min(cap, BF) * 4);
      break;
    }
    case 5:
    case 8: {  // unique rows updated (5: global row ids, 8: their table ids)
      std::vector<uint32_t> k(nnz_own);
      const void* src = sorted_k;
      if (nnz_own) S2D_CUDA(cudaMemcpy(k.data(), src, nnz_own * 4, cudaMemcpyDeviceToHost));
      std::vector<uint32_t> rows;
      for (uint64_t i = 0; i < nnz_own; ++i) {
        if (k[i] >= n_slots) break;
        if (i && k[i] == k[i - 1]) continue;
        const size_t j = std::upper_bound(vbase_sorted.begin(), vbase_sorted.end() - 1, k[i]) - vbase_sorted.begin() - 1;
        const FeatDev& fd = feats[feat_of_vbase[j]];
        rows.push_back(which == 5 ? k[i] - fd.vbase + fd.lo : feat_of_vbase[j]);
      }
      *n = rows.size();
      if (out) std::memcpy(out, rows.data(), std::min<uint64_t>(cap, rows.size()) * 4);
      break;
    }
    case 6:  // engine-owned pooled output of the last forward
      copy(pooled_buffer(), pooled_buffer() ? (uint64_t)B * sum_dims : 0, 4);
      break;
    case 7:  // f64 row gradients of the last update (debug_grad on), rows as in view 5, max_dim columns
      copy(dbg_grad.p, debug_grad ? dbg_rows * max_dim : 0, 8);
      break;
    default:
      throw Error(S2D_EINVAL, "unknown debug buffer");
  }
}

}  // namespace s2d
