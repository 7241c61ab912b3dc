// K5 replica sync (sync_replicas, src/trainer.cpp:547-596):
//   flag_count /   ascending list of this replica's dirty slots; the
//   flag_write     replicas all-gather their lists, mark each other's slots
//   mark_slots     dirty and compact again, so every replica holds the same
//                  ascending union list and the all-gathered rows line up
//   pack_rows      (w row, v) of each listed slot -> fp32 wire rows
//   mean_rows      x = f32((sum_{g ascending} f64(x_g)) * (1/M)) per element
//                  (deterministic_mean_inplace, src/topology.cpp:150-163),
//                  weights then moments (moments skipped for SGD); clears
//                  the dirty flag.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "device.cuh"

namespace s2d {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kSyncRows = 4;  // rows per warp and iteration in the P2P sync kernels

// 16 flags per thread, one 16-byte load when the tile is full
__device__ __forceinline__ void load_flags(const uint8_t* __restrict__ flags, uint64_t base, uint32_t n,
                                           uint32_t (&f)[kItems]) {
  if (base + kItems <= n) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(flags + base));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < kItems; ++i) f[i] = ((w[i / 4] >> (8 * (i % 4))) & 0xffu) != 0;
  } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) f[i] = (base + i < n) ? (flags[base + i] != 0) : 0u;
  }
}

__global__ void __launch_bounds__(kThreads) k_flag_count(const uint8_t* __restrict__ flags, uint32_t n,
                                                         uint32_t* __restrict__ tile_sum) {
  using BR = cub::BlockReduce<uint32_t, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  uint32_t f[kItems];
  load_flags(flags, (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems, n, f);
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) c += f[i];
  const uint32_t s = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_flag_write(const uint8_t* __restrict__ flags, uint32_t n,
                                                         const uint32_t* __restrict__ tile_sum,
                                                         uint32_t* __restrict__ list) {
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kItems;
  uint32_t f[kItems];
  load_flags(flags, base, n, f);
  uint32_t ex[kItems];
  BS(tmp).ExclusiveSum(f, ex);
  const uint32_t off = tile_sum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if (f[i]) list[off + ex[i]] = (uint32_t)(base + i);
}

// union: flag every slot another replica listed (0xffffffff = padding)
__global__ void k_mark_slots(const uint32_t* __restrict__ lists, uint64_t n, uint32_t n_slots,
                             uint8_t* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = __ldg(lists + i);
    if (s < n_slots) flags[s] = 1;
  }
}

template <typename WT>
__global__ void k_pack_rows(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                            uint32_t n_feat, const uint32_t* __restrict__ list, const uint32_t* count,
                            const WT* __restrict__ w, const float* __restrict__ moments, uint32_t row_floats,
                            float* __restrict__ packed) {
  const uint32_t n = *count;
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const uint32_t slot = list[i];
    const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, slot);
    const uint32_t dim = feats[f].dim;
    const WT* row = w + feats[f].wbase + (uint64_t)(slot - feats[f].vbase) * dim;
    float* out = packed + (uint64_t)i * row_floats;
    for (uint32_t c4 = lane; c4 < dim / 4; c4 += 32) {
      double d[4];
      Vec4<WT>::load_rw(row + c4 * 4, d);
      *reinterpret_cast<float4*>(out + c4 * 4) = make_float4((float)d[0], (float)d[1], (float)d[2], (float)d[3]);
    }
    if (lane == 0) out[row_floats - 1] = moments[slot];
  }
}

template <typename WT>
__global__ void k_mean_rows(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                            uint32_t n_feat, const uint32_t* __restrict__ list, const uint32_t* count,
                            const float* __restrict__ gathered, uint32_t M, uint32_t row_floats,
                            uint32_t rows_cap, WT* __restrict__ w, float* __restrict__ moments, int sgd,
                            uint8_t* __restrict__ dirty) {
  const uint32_t n = *count;
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  const double inv_m = 1.0 / (double)M;
  const uint64_t rstride = (uint64_t)rows_cap * row_floats;  // replica stride in `gathered`
  for (uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const uint32_t slot = list[i];
    const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, slot);
    const uint32_t dim = feats[f].dim;
    WT* row = w + feats[f].wbase + (uint64_t)(slot - feats[f].vbase) * dim;
    for (uint32_t c4 = lane; c4 < dim / 4; c4 += 32) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (uint32_t g = 0; g < M; ++g) {  // ascending group order
        const float4 x = *reinterpret_cast<const float4*>(gathered + g * rstride + (uint64_t)i * row_floats + c4 * 4);
        acc[0] += (double)x.x;
        acc[1] += (double)x.y;
        acc[2] += (double)x.z;
        acc[3] += (double)x.w;
      }
      double d[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = (double)(float)(acc[j] * inv_m);
      Vec4<WT>::store(row + c4 * 4, d);
    }
    if (lane == 0) {
      if (!sgd) {
        double acc = 0.0;
        for (uint32_t g = 0; g < M; ++g) acc += (double)gathered[g * rstride + (uint64_t)i * row_floats + row_floats - 1];
        moments[slot] = (float)(acc * inv_m);
      }
      dirty[slot] = 0;
    }
  }
}

// ---- P2P replica mean (DP group on one NVLink domain) --------------------
// Replica s averages slice s = [count*s/M, count*(s+1)/M) of the union list.
// Phase 1 (push): every replica stores its copy of each union row (f32 row +
// moment) into the slice owner's staging area, slot [g][i - lo_s], over
// NVLink.  Phase 2, after a group barrier: the owner reads the M copies of
// its slice locally, forms f32((sum_{g asc} f64 x_g) * (1/M))
// (deterministic_mean_inplace, topology.cpp:150-163; moments likewise unless
// SGD) and stores the mean into every replica.  All NVLink traffic is posted
// stores: 2(M-1)/M rows per union row per replica, vs M-1 for an all-gather.
// 4 stored elements widened to f32 (exact for fp32 and bf16)
__device__ __forceinline__ float4 load4_f32(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 load4_f32(const __nv_bfloat16* p) {
  const uint2 x = *reinterpret_cast<const uint2*>(p);
  return make_float4(__uint_as_float(x.x << 16), __uint_as_float(x.x & 0xffff0000u), __uint_as_float(x.y << 16),
                     __uint_as_float(x.y & 0xffff0000u));
}

template <typename WT, int kSyncV>  // kSyncV: 16-byte chunks per lane (rows up to kSyncV * 128 floats)
__global__ void k_p2p_push(PeerPtrs stage, uint32_t me, uint32_t M, const FeatDev* feats,
                           const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase, uint32_t n_feat,
                           const uint32_t* __restrict__ list, const uint32_t* __restrict__ count_ptr,
                           const WT* __restrict__ w, const float* __restrict__ moments, uint32_t row_floats,
                           uint64_t slice_cap) {
  pdl_wait();
  const uint32_t count = *count_ptr;  // the union's length (device-side)
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  // kSyncRows rows per warp and iteration: their loads are all in flight
  // before the first peer store (the loop is latency-bound otherwise)
  for (uint32_t i0 = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * kSyncRows; i0 < count;
       i0 += warps * kSyncRows) {
    float4 d[kSyncRows][kSyncV];
    float mom[kSyncRows];
    float* out[kSyncRows];
    uint32_t dim[kSyncRows];
#pragma unroll
    for (int r = 0; r < kSyncRows; ++r) {
      const uint32_t i = i0 + r;
      dim[r] = 0;
      out[r] = nullptr;
      if (i >= count) continue;
      // slice owner s of row i: largest s with count*s/M <= i
      uint32_t s = (uint32_t)(((uint64_t)i * M) / count);
      while (s + 1 < M && (uint64_t)count * (s + 1) / M <= i) ++s;
      while (s > 0 && (uint64_t)count * s / M > i) --s;
      const uint32_t lo = (uint32_t)((uint64_t)count * s / M);
      const uint32_t slot = list[i];
      const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, slot);
      dim[r] = feats[f].dim;
      const WT* row = w + feats[f].wbase + (uint64_t)(slot - feats[f].vbase) * dim[r];
      out[r] = reinterpret_cast<float*>(stage.p[s]) + ((uint64_t)me * slice_cap + (i - lo)) * row_floats;
#pragma unroll
      for (int v = 0; v < kSyncV; ++v)
        if (lane + v * 32 < dim[r] / 4) d[r][v] = load4_f32(row + (lane + v * 32) * 4);
      mom[r] = lane == 0 ? moments[slot] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < kSyncRows; ++r) {
      if (!out[r]) continue;
#pragma unroll
      for (int v = 0; v < kSyncV; ++v)
        if (lane + v * 32 < dim[r] / 4) *reinterpret_cast<float4*>(out[r] + (lane + v * 32) * 4) = d[r][v];
      if (lane == 0) out[r][row_floats - 1] = mom[r];
    }
  }
}

// Phase 2: the owner averages its slice (M staged copies, local reads) and
// stores each mean row into every replica's staging "means" area at its
// union index -- contiguous NVLink stores (storing into the peers' weight
// rows directly would scatter over their whole shard and thrash the
// peer-mapping TLB: measured 3x slower).
__global__ void k_p2p_mean(const float* __restrict__ local, PeerPtrs means, uint32_t M, uint32_t me,
                           const uint32_t* __restrict__ count_ptr, uint32_t row_floats, uint64_t slice_cap, int sgd) {
  pdl_wait();
  const uint32_t count = *count_ptr;  // this replica's slice [lo, hi) of the union
  const uint32_t lo = (uint32_t)((uint64_t)count * me / M), hi = (uint32_t)((uint64_t)count * (me + 1) / M);
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  const double inv_m = 1.0 / (double)M;
  const uint64_t gstride = slice_cap * row_floats;
  const uint32_t n4 = (row_floats - 4) / 4;  // row chunks (the last chunk holds the moment)
  for (uint32_t i = lo + blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < hi; i += warps) {
    const float* in = local + (uint64_t)(i - lo) * row_floats;
    for (uint32_t c4 = lane; c4 < n4; c4 += 32) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (uint32_t g = 0; g < M; ++g) {  // ascending group order
        const float4 x = *reinterpret_cast<const float4*>(in + g * gstride + c4 * 4);
        acc[0] += (double)x.x;
        acc[1] += (double)x.y;
        acc[2] += (double)x.z;
        acc[3] += (double)x.w;
      }
      const float4 m = make_float4((float)(acc[0] * inv_m), (float)(acc[1] * inv_m), (float)(acc[2] * inv_m),
                                   (float)(acc[3] * inv_m));
      for (uint32_t g = 0; g < M; ++g)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(means.p[g]) + (uint64_t)i * row_floats + c4 * 4) = m;
    }
    if (lane == 0 && !sgd) {
      double acc = 0.0;
      for (uint32_t g = 0; g < M; ++g) acc += (double)in[g * gstride + row_floats - 1];
      const float m = (float)(acc * inv_m);
      for (uint32_t g = 0; g < M; ++g)
        reinterpret_cast<float*>(means.p[g])[(uint64_t)i * row_floats + row_floats - 1] = m;
    }
  }
}

// Phase 3 (local): every replica scatters the count mean rows into its
// weights (one rounding to the storage type) and moments.
template <typename WT, int kSyncV>
__global__ void k_p2p_scatter(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                              uint32_t n_feat, const uint32_t* __restrict__ list,
                              const uint32_t* __restrict__ count_ptr, const float* __restrict__ means,
                              uint32_t row_floats, WT* __restrict__ w, float* __restrict__ moments, int sgd) {
  pdl_wait();
  const uint32_t count = *count_ptr;
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t i0 = (blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * kSyncRows; i0 < count;
       i0 += warps * kSyncRows) {
    float4 x[kSyncRows][kSyncV];
    float mom[kSyncRows];
    WT* row[kSyncRows];
    uint32_t dim[kSyncRows], slot[kSyncRows];
#pragma unroll
    for (int r = 0; r < kSyncRows; ++r) {
      const uint32_t i = i0 + r;
      row[r] = nullptr;
      dim[r] = 0;
      if (i >= count) continue;
      slot[r] = list[i];
      const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, slot[r]);
      dim[r] = feats[f].dim;
      row[r] = w + feats[f].wbase + (uint64_t)(slot[r] - feats[f].vbase) * dim[r];
      const float* in = means + (uint64_t)i * row_floats;
#pragma unroll
      for (int v = 0; v < kSyncV; ++v)
        if (lane + v * 32 < dim[r] / 4) x[r][v] = *reinterpret_cast<const float4*>(in + (lane + v * 32) * 4);
      mom[r] = in[row_floats - 1];
    }
#pragma unroll
    for (int r = 0; r < kSyncRows; ++r) {
      if (!row[r]) continue;
#pragma unroll
      for (int v = 0; v < kSyncV; ++v)
        if (lane + v * 32 < dim[r] / 4) {
          const double d[4] = {(double)x[r][v].x, (double)x[r][v].y, (double)x[r][v].z, (double)x[r][v].w};
          Vec4<WT>::store(row[r] + (lane + v * 32) * 4, d);
        }
      if (lane == 0 && !sgd) moments[slot[r]] = mom[r];
    }
  }
}

// ---- pair (M = 2) snapshot replica sync -----------------------------------
// Row x's replicas x_0, x_1: replica g's current row if g dirtied it this
// interval, else the row's value at the last sync (x_0 of the interval).
// The update saved that value (snapshot log) before a replica's first write
// to the row, so for a row only replica g dirtied, g alone forms the mean
// f32((f64 x_0 + f64 x_1) * 0.5) (deterministic_mean_inplace,
// topology.cpp:150-163, ascending group order) from its row and its
// snapshot, stores it, and sends the mean; a row both dirtied is sent as
// g's copy and both replicas average it on receipt.  Each replica sends its
// dirty rows once (no union list, no slice round trip); the receiver streams
// the peer's entries in the peer's list order.
//
// Staging entry j of the peer's list: f32 row | flag at rf - 2 (1 = final
// mean, 0 = copy) | moment at rf - 1.
constexpr int kPairWarps = 8;
template <typename WT, int kSyncV>
__global__ void __launch_bounds__(kPairWarps * 32) k_pair_push(
    float* __restrict__ peer_stage, uint32_t me, const uint32_t* __restrict__ mine, const uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ theirs, const FeatDev* feats, const uint32_t* vbase_sorted,
    const uint32_t* feat_of_vbase, uint32_t n_feat, const float* __restrict__ snap, const uint32_t* __restrict__ snap_pos,
    uint32_t row_floats, WT* __restrict__ w, float* __restrict__ moments, int sgd, uint32_t* __restrict__ n_both) {
  pdl_wait();
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  const uint32_t count = counts[me], their_n = counts[me ^ 1u];
  const uint64_t nwarps = (uint64_t)gridDim.x * kPairWarps;
  const uint64_t chunks = (count + 31) / 32, per_warp = (chunks + nwarps - 1) / nwarps;
  const uint64_t gw = (uint64_t)blockIdx.x * kPairWarps + wib;
  const uint64_t r0 = gw * per_warp * 32, r1 = min((uint64_t)count, r0 + per_warp * 32);
  uint32_t both_n = 0;
  for (uint64_t c0 = r0; c0 < r1; c0 += 32) {
    const uint32_t rows = r1 - c0 < 32 ? (uint32_t)(r1 - c0) : 32u;
    const uint32_t my_slot = lane < rows ? mine[c0 + lane] : 0xffffffffu;
    // is the row in the peer's list too?  (per lane binary search; the
    // lists are a few MB, L2-resident)
    uint32_t lo = 0, hi = their_n;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (theirs[mid] < my_slot) lo = mid + 1;
      else hi = mid;
    }
    const bool both = lane < rows && lo < their_n && theirs[lo] == my_slot;
    both_n += __popc(__ballot_sync(0xffffffffu, both));
    // per lane (row): weight row, dim, snapshot (a row only this replica dirtied)
    uint32_t my_dim = 0, my_snap = 0xffffffffu;
    uint64_t my_wofs = 0;
    if (lane < rows) {
      const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, my_slot);
      my_dim = feats[f].dim;
      my_wofs = feats[f].wbase + (uint64_t)(my_slot - feats[f].vbase) * my_dim;
      if (!both) my_snap = snap_pos[my_slot];
    }
    constexpr int R = kSyncV == 1 ? 4 : kSyncV == 2 ? 2 : 1;  // rows in flight
    for (uint32_t j = 0; j < rows; j += R) {
      float4 own[R][kSyncV], old[R][kSyncV];
      float own_m[R], old_m[R];
      uint32_t dim[R], slot[R];
      WT* row[R];
      const float* sp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t i = (j + r) & 31;
        slot[r] = __shfl_sync(0xffffffffu, my_slot, i);
        dim[r] = j + r < rows ? __shfl_sync(0xffffffffu, my_dim, i) : 0u;
        row[r] = w + shfl64(my_wofs, i);
        const uint32_t sn = __shfl_sync(0xffffffffu, my_snap, i);
        sp[r] = sn != 0xffffffffu ? snap + (uint64_t)sn * row_floats : nullptr;
        own_m[r] = old_m[r] = 0.f;
        if (!dim[r]) continue;
#pragma unroll
        for (int v = 0; v < kSyncV; ++v)
          if (lane + v * 32 < dim[r] / 4) {
            own[r][v] = load4_f32(row[r] + (lane + v * 32) * 4);
            if (sp[r]) old[r][v] = *reinterpret_cast<const float4*>(sp[r] + (lane + v * 32) * 4);
          }
        own_m[r] = moments[slot[r]];
        if (sp[r]) old_m[r] = sp[r][row_floats - 1];
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!dim[r]) continue;
        float* out = peer_stage + (c0 + j + r) * (uint64_t)row_floats;
        if (sp[r]) {  // only this replica dirtied the row: the mean, here and at the peer
#pragma unroll
          for (int v = 0; v < kSyncV; ++v)
            if (lane + v * 32 < dim[r] / 4) {
              const float4 a = me == 0 ? own[r][v] : old[r][v], b = me == 0 ? old[r][v] : own[r][v];
              const float4 m = make_float4((float)(((double)a.x + (double)b.x) * 0.5),
                                           (float)(((double)a.y + (double)b.y) * 0.5),
                                           (float)(((double)a.z + (double)b.z) * 0.5),
                                           (float)(((double)a.w + (double)b.w) * 0.5));
              const double d[4] = {(double)m.x, (double)m.y, (double)m.z, (double)m.w};
              Vec4<WT>::store(row[r] + (lane + v * 32) * 4, d);
              *reinterpret_cast<float4*>(out + (lane + v * 32) * 4) = m;
            }
          if (lane == 0) {
            const float am = me == 0 ? own_m[r] : old_m[r], bm2 = me == 0 ? old_m[r] : own_m[r];
            const float mm = (float)(((double)am + (double)bm2) * 0.5);
            if (!sgd) moments[slot[r]] = mm;
            out[row_floats - 2] = 1.f;
            out[row_floats - 1] = mm;
          }
        } else {  // both replicas dirtied it: send this replica's copy
#pragma unroll
          for (int v = 0; v < kSyncV; ++v)
            if (lane + v * 32 < dim[r] / 4) *reinterpret_cast<float4*>(out + (lane + v * 32) * 4) = own[r][v];
          if (lane == 0) {
            out[row_floats - 2] = 0.f;
            out[row_floats - 1] = own_m[r];
          }
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0 && both_n) atomicAdd(n_both, both_n);
}

// The peer's entries (its list order): a final mean is stored as is; a copy
// is averaged with this replica's row in ascending group order.  Each warp
// takes 32-entry chunks of the peer's list: lane i resolves entry i's row,
// flag and moments (one parallel feature lookup per chunk), then the warp
// streams the rows R at a time.
template <typename WT, int kSyncV>
__global__ void __launch_bounds__(256) k_pair_recv(const float* __restrict__ stage, uint32_t me,
                                                   const uint32_t* __restrict__ theirs,
                                                   const uint32_t* __restrict__ counts, const FeatDev* feats,
                                                   const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                                                   uint32_t n_feat, uint32_t row_floats, WT* __restrict__ w,
                                                   float* __restrict__ moments, int sgd) {
  pdl_wait();
  const uint32_t count = counts[me ^ 1u];
  const uint32_t lane = lane_id();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  constexpr int R = kSyncV == 1 ? 4 : kSyncV == 2 ? 2 : 1;
  for (uint64_t c0 = gw * 32; c0 < count; c0 += warps * 32) {
    const uint32_t rows = count - c0 < 32 ? (uint32_t)(count - c0) : 32u;
    uint32_t my_slot = 0, my_dim = 0;
    uint64_t my_wofs = 0;
    float my_flag = 1.f, my_xm = 0.f, my_own_m = 0.f;
    if (lane < rows) {
      my_slot = theirs[c0 + lane];
      const uint32_t f = feature_of_slot(vbase_sorted, feat_of_vbase, n_feat, my_slot);
      my_dim = feats[f].dim;
      my_wofs = feats[f].wbase + (uint64_t)(my_slot - feats[f].vbase) * my_dim;
      const float* in = stage + (c0 + lane) * (uint64_t)row_floats;
      my_flag = in[row_floats - 2];
      my_xm = in[row_floats - 1];
      if (my_flag == 0.f) my_own_m = moments[my_slot];
    }
    for (uint32_t j = 0; j < rows; j += R) {
      float4 x[R][kSyncV], own[R][kSyncV];
      uint32_t dim[R];
      bool fin[R];
      WT* row[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t i = (j + r) & 31;
        dim[r] = j + r < rows ? __shfl_sync(0xffffffffu, my_dim, i) : 0u;
        row[r] = w + shfl64(my_wofs, i);
        fin[r] = __shfl_sync(0xffffffffu, my_flag, i) != 0.f;
        if (!dim[r]) continue;
        const float* in = stage + (c0 + j + r) * (uint64_t)row_floats;
#pragma unroll
        for (int v = 0; v < kSyncV; ++v)
          if (lane + v * 32 < dim[r] / 4) {
            x[r][v] = *reinterpret_cast<const float4*>(in + (lane + v * 32) * 4);
            if (!fin[r]) own[r][v] = load4_f32(row[r] + (lane + v * 32) * 4);
          }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!dim[r]) continue;
#pragma unroll
        for (int v = 0; v < kSyncV; ++v)
          if (lane + v * 32 < dim[r] / 4) {
            float4 m = x[r][v];
            if (!fin[r]) {
              const float4 a = me == 0 ? own[r][v] : x[r][v], b = me == 0 ? x[r][v] : own[r][v];
              m = make_float4((float)(((double)a.x + (double)b.x) * 0.5), (float)(((double)a.y + (double)b.y) * 0.5),
                              (float)(((double)a.z + (double)b.z) * 0.5), (float)(((double)a.w + (double)b.w) * 0.5));
            }
            const double d[4] = {(double)m.x, (double)m.y, (double)m.z, (double)m.w};
            Vec4<WT>::store(row[r] + (lane + v * 32) * 4, d);
          }
      }
    }
    if (!sgd && lane < rows) {  // moments: entry `lane` of the chunk
      float mm = my_xm;
      if (my_flag == 0.f) {
        const float am = me == 0 ? my_own_m : my_xm, bm = me == 0 ? my_xm : my_own_m;
        mm = (float)(((double)am + (double)bm) * 0.5);
      }
      moments[my_slot] = mm;
    }
  }
}

}  // namespace

// tmp layout: tile counts [ntiles] | their exclusive scan [ntiles + 1] | scan workspace
static uint32_t flag_tiles(uint32_t n_slots) { return (n_slots + kTile - 1) / kTile; }

size_t flag_tmp_bytes(uint32_t n_slots) {
  const uint32_t nt = flag_tiles(n_slots);
  return ((size_t)2 * nt + 2) * 4 + scan_tmp_bytes((uint64_t)nt + 1) + 16;
}

void launch_flag_count(const uint8_t* dirty, uint32_t n_slots, uint32_t* count, void* tmp, size_t tmp_bytes,
                       cudaStream_t st) {
  const uint32_t ntiles = flag_tiles(n_slots);
  if (flag_tmp_bytes(n_slots) > tmp_bytes) throw Error(S2D_ECUDA, "compaction workspace too small");
  if (ntiles == 0) {
    S2D_CUDA(cudaMemsetAsync(count, 0, 4, st));
    return;
  }
  uint32_t* ts = reinterpret_cast<uint32_t*>(tmp);
  uint32_t* tx = ts + ntiles;
  char* sw = reinterpret_cast<char*>(tx + ntiles + 2);
  sw += (16 - reinterpret_cast<uintptr_t>(sw) % 16) % 16;
  k_flag_count<<<ntiles, kThreads, 0, st>>>(dirty, n_slots, ts);
  S2D_LAUNCH_CHECK();
  scan_u32_to_u32(ts, tx, ntiles, st, sw, scan_tmp_bytes((uint64_t)ntiles + 1));
  S2D_CUDA(cudaMemcpyAsync(count, tx + ntiles, 4, cudaMemcpyDeviceToDevice, st));
}

__global__ void k_clear_listed(uint8_t* __restrict__ dirty, const uint32_t* __restrict__ list,
                               const uint32_t* __restrict__ count) {
  const uint32_t n = *count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dirty[list[i]] = 0;
}

void launch_clear_listed(uint8_t* dirty, const uint32_t* list, const uint32_t* count, uint32_t n, cudaStream_t st) {
  if (!n) return;
  k_clear_listed<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(dirty, list, count);
  S2D_LAUNCH_CHECK();
}

void launch_flag_write(const uint8_t* dirty, uint32_t n_slots, uint32_t* list, const void* tmp, cudaStream_t st) {
  const uint32_t ntiles = flag_tiles(n_slots);
  if (ntiles == 0) return;
  k_flag_write<<<ntiles, kThreads, 0, st>>>(dirty, n_slots, reinterpret_cast<const uint32_t*>(tmp) + ntiles, list);
  S2D_LAUNCH_CHECK();
}

void launch_mark_slots(const uint32_t* lists, uint64_t n, uint32_t n_slots, uint8_t* dirty, cudaStream_t st) {
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  k_mark_slots<<<grid, 256, 0, st>>>(lists, n, n_slots, dirty);
  S2D_LAUNCH_CHECK();
}

void launch_pack_rows(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                      uint32_t n_feat_owned, const uint32_t* list, const uint32_t* count, const void* weights,
                      int bf16, const float* moments, uint32_t row_floats, float* packed, uint32_t max_rows,
                      cudaStream_t st) {
  if (!max_rows) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((max_rows + 7) / 8, 148ull * 8);
  if (bf16)
    k_pack_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(feats, vbase_sorted, feat_of_vbase, n_feat_owned, list, count,
                                                     reinterpret_cast<const __nv_bfloat16*>(weights), moments,
                                                     row_floats, packed);
  else
    k_pack_rows<float><<<grid, 256, 0, st>>>(feats, vbase_sorted, feat_of_vbase, n_feat_owned, list, count,
                                             reinterpret_cast<const float*>(weights), moments, row_floats, packed);
  S2D_LAUNCH_CHECK();
}

void launch_mean_rows(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                      uint32_t n_feat_owned, const uint32_t* list, const uint32_t* count, const float* gathered,
                      uint32_t M, uint32_t row_floats, uint32_t rows_cap, void* weights, int bf16, float* moments,
                      int sgd, uint8_t* dirty, cudaStream_t st) {
  if (!rows_cap) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((rows_cap + 7) / 8, 148ull * 8);
  if (bf16)
    k_mean_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(feats, vbase_sorted, feat_of_vbase, n_feat_owned, list, count,
                                                     gathered, M, row_floats, rows_cap,
                                                     reinterpret_cast<__nv_bfloat16*>(weights), moments, sgd, dirty);
  else
    k_mean_rows<float><<<grid, 256, 0, st>>>(feats, vbase_sorted, feat_of_vbase, n_feat_owned, list, count, gathered,
                                             M, row_floats, rows_cap, reinterpret_cast<float*>(weights), moments, sgd,
                                             dirty);
  S2D_LAUNCH_CHECK();
}


template <int V>
void p2p_push_v(const PeerPtrs& stage, uint32_t me, uint32_t M, const FeatDev* feats, const uint32_t* vbase_sorted,
                const uint32_t* feat_of_vbase, uint32_t n_feat, const uint32_t* list, const uint32_t* count,
                unsigned grid, const void* weights, int bf16, const float* moments, uint32_t row_floats,
                uint64_t slice_cap, cudaStream_t st) {
  if (bf16)
    pdl_launch(k_p2p_push<__nv_bfloat16, V>, dim3(grid), dim3(256), 0, st, stage, me, M, feats, vbase_sorted,
               feat_of_vbase, n_feat, list, count, reinterpret_cast<const __nv_bfloat16*>(weights), moments,
               row_floats, slice_cap);
  else
    pdl_launch(k_p2p_push<float, V>, dim3(grid), dim3(256), 0, st, stage, me, M, feats, vbase_sorted, feat_of_vbase,
               n_feat, list, count, reinterpret_cast<const float*>(weights), moments, row_floats, slice_cap);
}

void launch_p2p_push(const PeerPtrs& stage, uint32_t me, uint32_t M, const FeatDev* feats,
                     const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase, uint32_t n_feat,
                     const uint32_t* list, const uint32_t* count, uint32_t count_ub, const void* weights, int bf16,
                     const float* moments, uint32_t row_floats, uint64_t slice_cap, cudaStream_t st) {
  if (!count_ub) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((count_ub + 8 * kSyncRows - 1) / (8 * kSyncRows), 148ull * 16);
  const uint32_t d4 = (row_floats - 4) / 4;
  if (d4 <= 32)
    p2p_push_v<1>(stage, me, M, feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, weights, bf16, moments,
                  row_floats, slice_cap, st);
  else if (d4 <= 64)
    p2p_push_v<2>(stage, me, M, feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, weights, bf16, moments,
                  row_floats, slice_cap, st);
  else
    p2p_push_v<4>(stage, me, M, feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, weights, bf16, moments,
                  row_floats, slice_cap, st);
}

void launch_p2p_mean(const float* local, const PeerPtrs& means, uint32_t M, uint32_t me, const uint32_t* count,
                     uint32_t count_ub, uint32_t row_floats, uint64_t slice_cap, int sgd, cudaStream_t st) {
  if (!count_ub) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((count_ub / M + 8) / 8, 148ull * 16);
  pdl_launch(k_p2p_mean, dim3(grid), dim3(256), 0, st, local, means, M, me, count, row_floats, slice_cap, sgd);
}

template <int V>
void p2p_scatter_v(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase, uint32_t n_feat,
                   const uint32_t* list, const uint32_t* count, unsigned grid, const float* means, uint32_t row_floats,
                   void* weights, int bf16, float* moments, int sgd, cudaStream_t st) {
  if (bf16)
    pdl_launch(k_p2p_scatter<__nv_bfloat16, V>, dim3(grid), dim3(256), 0, st, feats, vbase_sorted, feat_of_vbase,
               n_feat, list, count, means, row_floats, reinterpret_cast<__nv_bfloat16*>(weights), moments, sgd);
  else
    pdl_launch(k_p2p_scatter<float, V>, dim3(grid), dim3(256), 0, st, feats, vbase_sorted, feat_of_vbase, n_feat,
               list, count, means, row_floats, reinterpret_cast<float*>(weights), moments, sgd);
}

void launch_p2p_scatter(const FeatDev* feats, const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase,
                        uint32_t n_feat, const uint32_t* list, const uint32_t* count, uint32_t count_ub,
                        const float* means, uint32_t row_floats, void* weights, int bf16, float* moments, int sgd,
                        cudaStream_t st) {
  if (!count_ub) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((count_ub + 8 * kSyncRows - 1) / (8 * kSyncRows), 148ull * 16);
  const uint32_t d4 = (row_floats - 4) / 4;
  if (d4 <= 32)
    p2p_scatter_v<1>(feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, means, row_floats, weights, bf16,
                     moments, sgd, st);
  else if (d4 <= 64)
    p2p_scatter_v<2>(feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, means, row_floats, weights, bf16,
                     moments, sgd, st);
  else
    p2p_scatter_v<4>(feats, vbase_sorted, feat_of_vbase, n_feat, list, count, grid, means, row_floats, weights, bf16,
                     moments, sgd, st);
}

template <int V>
void pair_v(bool push, unsigned grid, float* peer_stage, const float* stage, uint32_t me, const uint32_t* mine,
            const uint32_t* counts, const uint32_t* theirs, const FeatDev* feats, const uint32_t* vbase_sorted,
            const uint32_t* feat_of_vbase, uint32_t n_feat, const float* snap, const uint32_t* snap_pos,
            uint32_t row_floats, void* weights, int bf16, float* moments, int sgd, uint32_t* n_both, cudaStream_t st) {
  if (push) {
    if (bf16)
      pdl_launch(k_pair_push<__nv_bfloat16, V>, dim3(grid), dim3(kPairWarps * 32), 0, st, peer_stage, me, mine, counts,
                 theirs, feats, vbase_sorted, feat_of_vbase, n_feat, snap, snap_pos, row_floats,
                 reinterpret_cast<__nv_bfloat16*>(weights), moments, sgd, n_both);
    else
      pdl_launch(k_pair_push<float, V>, dim3(grid), dim3(kPairWarps * 32), 0, st, peer_stage, me, mine, counts, theirs,
                 feats, vbase_sorted, feat_of_vbase, n_feat, snap, snap_pos, row_floats, reinterpret_cast<float*>(weights),
                 moments, sgd, n_both);
  } else {
    if (bf16)
      pdl_launch(k_pair_recv<__nv_bfloat16, V>, dim3(grid), dim3(256), 0, st, stage, me, theirs, counts, feats,
                 vbase_sorted, feat_of_vbase, n_feat, row_floats, reinterpret_cast<__nv_bfloat16*>(weights), moments,
                 sgd);
    else
      pdl_launch(k_pair_recv<float, V>, dim3(grid), dim3(256), 0, st, stage, me, theirs, counts, feats, vbase_sorted,
                 feat_of_vbase, n_feat, row_floats, reinterpret_cast<float*>(weights), moments, sgd);
  }
}

static void pair_dispatch(bool push, unsigned grid, float* peer_stage, const float* stage, uint32_t me,
                          const uint32_t* mine, const uint32_t* counts, const uint32_t* theirs, const FeatDev* feats,
                          const uint32_t* vbase_sorted, const uint32_t* feat_of_vbase, uint32_t n_feat,
                          const float* snap, const uint32_t* snap_pos, uint32_t row_floats, void* weights, int bf16,
                          float* moments, int sgd, uint32_t* n_both, cudaStream_t st) {
  const uint32_t d4 = (row_floats - 4) / 4;
  if (d4 <= 32)
    pair_v<1>(push, grid, peer_stage, stage, me, mine, counts, theirs, feats, vbase_sorted, feat_of_vbase, n_feat, snap,
              snap_pos, row_floats, weights, bf16, moments, sgd, n_both, st);
  else if (d4 <= 64)
    pair_v<2>(push, grid, peer_stage, stage, me, mine, counts, theirs, feats, vbase_sorted, feat_of_vbase, n_feat, snap,
              snap_pos, row_floats, weights, bf16, moments, sgd, n_both, st);
  else
    pair_v<4>(push, grid, peer_stage, stage, me, mine, counts, theirs, feats, vbase_sorted, feat_of_vbase, n_feat, snap,
              snap_pos, row_floats, weights, bf16, moments, sgd, n_both, st);
}

void launch_pair_push(float* peer_stage, uint32_t me, const uint32_t* mine, const uint32_t* counts,
                      const uint32_t* theirs, uint32_t mine_n, const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat, const float* snap, const uint32_t* snap_pos,
                      uint32_t row_floats, void* weights, int bf16, float* moments, int sgd, uint32_t* n_both,
                      cudaStream_t st) {
  if (!mine_n) return;
  const unsigned grid =
      (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((mine_n + 32 * kPairWarps - 1) / (32 * kPairWarps), 148ull * 8));
  pair_dispatch(true, grid, peer_stage, nullptr, me, mine, counts, theirs, feats, vbase_sorted, feat_of_vbase, n_feat,
                snap, snap_pos, row_floats, weights, bf16, moments, sgd, n_both, st);
}

void launch_pair_recv(const float* stage, uint32_t me, const uint32_t* theirs, const uint32_t* counts,
                      uint32_t theirs_n, const FeatDev* feats, const uint32_t* vbase_sorted,
                      const uint32_t* feat_of_vbase, uint32_t n_feat, uint32_t row_floats, void* weights, int bf16,
                      float* moments, int sgd, cudaStream_t st) {
  if (!theirs_n) return;
  const uint64_t chunks = (theirs_n + 31) / 32;  // one warp per 32-entry chunk, 8 warps per block
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((chunks + 7) / 8, 148ull * 8));
  pair_dispatch(false, grid, nullptr, stage, me, nullptr, counts, theirs, feats, vbase_sorted, feat_of_vbase, n_feat,
                nullptr, nullptr, row_floats, weights, bf16, moments, sgd, nullptr, st);
}

}  // namespace s2d
