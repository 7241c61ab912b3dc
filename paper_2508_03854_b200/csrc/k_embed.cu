// Forward-side kernels of the step:
//   init_rows      device port of init_table (src/embedding.cpp:17-37)
//   bucket_count   K1: ids per (owner, bag) for the input-dist all-to-all
//   bucket_permute K1: bit-exact permute of ids into per-owner send blocks,
//                  canonical (sample, feature, occurrence) order
//                  (build_demand, src/trainer.cpp:283-313)
//   (K2 owner lookup lives in k_stream.cu)
//   combine        requester side: f32(sum_{owner asc} f64(partial))
//                  (pool_and_forward, src/trainer.cpp:372-390)
//   grad_gather    C2 send layout (build_grad_payloads, src/trainer.cpp:440-457)
//
// Layout: LPB lanes serve one bag, each lane owns VPL 16-byte column vectors
// of the row (a row is LPB*16 contiguous bytes per vector).
#include <algorithm>

#include "device.cuh"

namespace s2d {
namespace {

// ---- init_table ----------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:12-19
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint64_t row_key(uint64_t seed, uint64_t table, uint64_t row) {
  uint64_t h = 0x8A5CD789635D2DFFULL;  // make_key, rng.hpp:22-28
  h = mix64(h + 0x9E3779B97F4A7C15ULL + seed);
  h = mix64(h + 0x9E3779B97F4A7C15ULL + table);
  h = mix64(h + 0x9E3779B97F4A7C15ULL + row);
  return h;
}

template <typename WT>
__global__ void k_init_rows(WT* __restrict__ w, uint64_t wbase, uint32_t table_id, uint32_t lo,
                            uint32_t nrows, uint32_t dim, uint64_t seed) {
  const uint32_t d4 = dim / 4;
  const uint64_t total = (uint64_t)nrows * d4;
  const double bound = 1.0 / sqrt((double)dim);
  const double lo_v = -bound, span = __dsub_rn(bound, lo_v);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(i / d4), c4 = (uint32_t)(i % d4);
    const uint64_t key = row_key(seed, table_id, (uint64_t)lo + r);
    double d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t ctr = (uint64_t)c4 * 4 + q + 1;
      const double u = (double)(mix64(key + ctr * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
      d[q] = (double)(float)__dadd_rn(lo_v, __dmul_rn(span, u));
    }
    Vec4<WT>::store(w + wbase + (uint64_t)r * dim + (uint64_t)c4 * 4, d);
  }
}

// ---- combine (requester side) -----------------------------------------------

template <int LPB, int VPL>
__global__ void __launch_bounds__(256) k_combine(const CombineArgs a) {
  pdl_wait();
  constexpr int GPW = 32 / LPB;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPB, gl = lane % LPB;
  const uint64_t BF = (uint64_t)a.B * a.F;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  const uint64_t warp = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  for (uint64_t base = warp * 32; base < BF; base += warps * 32) {
    // lane per bag: which of these 32 bags still need the combine?  (With
    // the engine-owned output the owner of a single-owner table stored the
    // pooled row itself; only its empty bags remain, to be zeroed.)
    bool need = false;
    {
      const uint64_t b = base + lane;
      if (b < BF) {
        need = true;
        const uint32_t f = (uint32_t)(b % a.F);
        if (a.skip_single && __ldg(&a.feats[f].single)) {
          bool any = false;
          for (uint32_t o = 0; o < a.N; ++o) any |= __ldg(a.cnt + (uint64_t)o * BF + b) != 0;
          need = !any;
        }
      }
    }
    uint32_t m = __ballot_sync(0xffffffffu, need);
    while (m) {  // group g takes the g-th remaining bag
      uint32_t mm = m;
      for (uint32_t q = 0; q < grp && mm; ++q) mm &= mm - 1;
      for (int q = 0; q < GPW && m; ++q) m &= m - 1;
      if (!mm) continue;
      const uint64_t b = base + (__ffs(mm) - 1);
      const uint32_t f = (uint32_t)(b % a.F);
      const uint32_t d4 = __ldg(&a.feats[f].dim) >> 2;
      double acc[VPL][4];
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[v][q] = 0.0;
      for (uint32_t o = 0; o < a.N; ++o) {  // ascending owner (trainer.cpp:378-386)
        if (__ldg(a.cnt + (uint64_t)o * BF + b) == 0) continue;
        const float* p = a.recv + __ldg(a.eoff + (uint64_t)o * BF + b);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const uint32_t c4 = gl + v * LPB;
          if (c4 < d4) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(p + c4 * 4));
            acc[v][0] += (double)x.x;
            acc[v][1] += (double)x.y;
            acc[v][2] += (double)x.z;
            acc[v][3] += (double)x.w;
          }
        }
      }
      float* out = a.pooled + (b / a.F) * a.sum_dims + __ldg(&a.feats[f].coff);
      if (__ldg(&a.feats[f].mean)) {  // mean pooling: f32(C * (1/L))
        const uint32_t L = __ldg(a.bag_off + b + 1) - __ldg(a.bag_off + b);
        const double inv = L ? 1.0 / (double)L : 1.0;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[v][q] = acc[v][q] * inv;
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const uint32_t c4 = gl + v * LPB;
        if (c4 < d4) store_f32x4_stream(out + c4 * 4, acc[v]);
      }
    }
  }
}

template <int LPB, int VPL>
__global__ void __launch_bounds__(256) k_grad_gather(const GradGatherArgs a) {
  pdl_wait();
  // kU bags per group iteration: all their row loads are issued before any
  // store, so each group keeps kU rows in flight toward NVLink
  constexpr int GPW = 32 / LPB, kU = 4;
  const uint32_t lane = lane_id();
  const uint32_t grp = lane / LPB, gl = lane % LPB;
  const uint64_t BF = (uint64_t)a.B * a.F;
  const uint64_t slots = (uint64_t)gridDim.x * (blockDim.x / 32) * GPW;
  const uint64_t first = ((uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * GPW + grp;
  for (uint64_t b0 = first * kU; b0 < BF; b0 += slots * kU) {
    float4 x[kU][VPL];
    uint32_t d4[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t b = b0 + u;
      d4[u] = 0;
      if (b < BF) {
        const uint32_t f = (uint32_t)(b % a.F);
        d4[u] = __ldg(&a.feats[f].dim) >> 2;
        const float* up = a.upstream + (b / a.F) * a.sum_dims + __ldg(&a.feats[f].coff);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const uint32_t c4 = gl + v * LPB;
          if (c4 < d4[u]) x[u][v] = __ldg(reinterpret_cast<const float4*>(up + c4 * 4));
        }
        if (__ldg(&a.feats[f].mean)) {  // mean pooling: the wire row is f32(f64(up) * (1/L))
          const uint32_t L = __ldg(a.bag_off + b + 1) - __ldg(a.bag_off + b);
          const double inv = L ? 1.0 / (double)L : 1.0;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            x[u][v].x = (float)((double)x[u][v].x * inv);
            x[u][v].y = (float)((double)x[u][v].y * inv);
            x[u][v].z = (float)((double)x[u][v].z * inv);
            x[u][v].w = (float)((double)x[u][v].w * inv);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t b = b0 + u;
      if (b >= BF) break;
      const uint32_t f = (uint32_t)(b % a.F);
      // (s, f, o ascending) order, trainer.cpp:446-453; single-owner tables
      // have exactly one candidate owner
      uint32_t o = 0, o_end = a.N;
      if (__ldg(&a.feats[f].single)) {
        o = __ldg(&a.ranges[__ldg(&a.feats[f].rbeg)].owner);
        o_end = o + 1;
      }
      for (; o < o_end; ++o) {
        if (__ldg(a.cnt + (uint64_t)o * BF + b) == 0) continue;
        float* dst = reinterpret_cast<float*>(a.peer_dst.p[o]) + a.peer_adj[o] + __ldg(a.eoff + (uint64_t)o * BF + b);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const uint32_t c4 = gl + v * LPB;
          if (c4 < d4[u]) *reinterpret_cast<float4*>(dst + c4 * 4) = x[u][v];
        }
      }
    }
  }
}

// ---- mean pooling, N = 1: scaled gradient rows ------------------------------

// out[s][coff_f + j] = f32(f64(up) * (1/L_(s,f))) for mean-pooled tables,
// up unchanged otherwise; one thread per float4
__global__ void __launch_bounds__(256) k_mean_prescale(const FeatDev* __restrict__ feats, uint32_t F, uint32_t B,
                                                       uint32_t sum_dims, const uint32_t* __restrict__ bag_off,
                                                       const float* __restrict__ up, float* __restrict__ out) {
  pdl_wait();
  const uint32_t q4 = sum_dims / 4;
  const uint64_t n = (uint64_t)B * q4;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / q4), c = (uint32_t)(i % q4) * 4;
    uint32_t f = 0;  // feature of column c (feats sorted by coff)
    for (uint32_t lo = 0, hi = F; hi - lo > 1;) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(&feats[mid].coff) <= c) lo = f = mid;
      else hi = mid;
    }
    float4 x = __ldg(reinterpret_cast<const float4*>(up) + i);
    if (__ldg(&feats[f].mean)) {
      const uint64_t b = (uint64_t)s * F + f;
      const uint32_t L = __ldg(bag_off + b + 1) - __ldg(bag_off + b);
      const double inv = L ? 1.0 / (double)L : 1.0;
      x.x = (float)((double)x.x * inv);
      x.y = (float)((double)x.y * inv);
      x.z = (float)((double)x.z * inv);
      x.w = (float)((double)x.w * inv);
    }
    reinterpret_cast<float4*>(out)[i] = x;
  }
}

// ---- K1 input-dist bucketing -------------------------------------------------

__device__ __forceinline__ uint32_t owner_of(const RangeDev* __restrict__ r, uint32_t beg, uint32_t end,
                                             uint32_t id) {
  // ranges of one table sorted by lo; largest lo <= id
  uint32_t lo = beg, hi = end;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&r[mid].lo) <= id)
      lo = mid;
    else
      hi = mid;
  }
  return __ldg(&r[lo].owner);
}

__global__ void __launch_bounds__(256) k_bucket_count(const BucketArgs a) {
  pdl_wait();
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < a.BF;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = (uint32_t)(b % a.F);
    const uint32_t rows = __ldg(&a.feats[f].rows), rb = __ldg(&a.feats[f].rbeg), re = __ldg(&a.feats[f].rend);
    const uint32_t len = __ldg(a.lengths + b);
    if (re - rb == 1) {  // single-owner table: every id goes to that owner, whose
      // lookup range-checks it (kErrIdRange there); no per-id work here
      const uint32_t ow = __ldg(&a.ranges[rb].owner);
      for (uint32_t o = 0; o < a.N; ++o) {
        const uint32_t c = o == ow ? len : 0u;
        a.cnt[(uint64_t)o * a.BF + b] = c;
        reinterpret_cast<uint32_t*>(a.peer_len.p[o])[(uint64_t)a.me * a.BF + b] = c;
      }
      continue;
    }
    uint32_t cnt[kMaxRanksPerGroup];
    for (uint32_t o = 0; o < a.N; ++o) cnt[o] = 0;
    const uint32_t off = __ldg(a.id_off + b);
    for (uint32_t k = 0; k < len; ++k) {
      const uint32_t id = __ldg(a.ids + off + k);
      if (id >= rows) {
        atomicOr(a.err, kErrIdRange);
        continue;
      }
      cnt[owner_of(a.ranges, rb, re, id)]++;
    }
    for (uint32_t o = 0; o < a.N; ++o) {
      a.cnt[(uint64_t)o * a.BF + b] = cnt[o];
      reinterpret_cast<uint32_t*>(a.peer_len.p[o])[(uint64_t)a.me * a.BF + b] = cnt[o];
    }
  }
}

// Warp per 32 consecutive bags: ids are read 32 at a time in (bag,
// occurrence) order, each lane finds its id's owner, and a per-owner ballot
// prefix gives each id its rank inside the owner's run, so the ids bound for
// one owner leave as contiguous runs (coalesced NVLink stores) in exactly the
// canonical order of build_demand (trainer.cpp:286-307).
__global__ void __launch_bounds__(256) k_bucket_permute(const BucketArgs a) {
  pdl_wait();
  const uint32_t lane = lane_id();
  const uint64_t n_units = (a.BF + 31) / 32;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t u = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < n_units; u += warps) {
    const uint64_t b0 = u * 32;
    const uint32_t nb = (a.BF - b0) < 32 ? (uint32_t)(a.BF - b0) : 32u;
    const uint64_t my_bag = b0 + min(lane, nb - 1);
    const uint32_t my_end = __ldg(a.id_off + my_bag + 1);
    const uint32_t o0 = __ldg(a.id_off + b0);
    const uint32_t o1 = __shfl_sync(0xffffffffu, my_end, nb - 1);
    // running output position per owner (lane o holds owner o's)
    uint32_t run = lane < a.N ? __ldg(a.send_off + (uint64_t)lane * a.BF + b0) : 0u;
    for (uint32_t c = o0; c < o1; c += 32) {
      const uint32_t p = c + lane;
      const bool have = p < o1;
      uint32_t j = 0;  // bag of item p within the unit: # lanes whose end <= p
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, my_end, j + step - 1);
        if (v <= p) j += step;
      }
      const uint32_t f = (uint32_t)((b0 + min(j, nb - 1)) % a.F);
      uint32_t o = 0xffffffffu, id = 0;
      if (have) {
        id = __ldg(a.ids + p);
        const uint32_t rb = __ldg(&a.feats[f].rbeg), re = __ldg(&a.feats[f].rend);
        if (re - rb == 1)  // single owner: every id goes there (its lookup flags bad ids)
          o = __ldg(&a.ranges[rb].owner);
        else if (id < __ldg(&a.feats[f].rows))
          o = owner_of(a.ranges, rb, re, id);
      }
      for (uint32_t q = 0; q < a.N; ++q) {
        const uint32_t sel = __ballot_sync(0xffffffffu, o == q);
        if (!sel) continue;
        const uint32_t base = __shfl_sync(0xffffffffu, run, q);
        if (o == q)
          reinterpret_cast<uint32_t*>(a.peer_ids.p[q])[a.ids_adj[q] + (int64_t)(base + __popc(sel & ((1u << lane) - 1u)))] =
              id;
        if (lane == q) run += __popc(sel);
      }
    }
  }
}

unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap) {
  uint64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

constexpr unsigned kGridCap = 148 * 16;

}  // namespace

void launch_init_rows(void* w, int bf16, const FeatDev* feats_host, uint32_t F, uint64_t seed,
                      cudaStream_t st) {
  for (uint32_t f = 0; f < F; ++f) {
    const FeatDev& fd = feats_host[f];
    if (fd.hi <= fd.lo) continue;
    const uint64_t work = (uint64_t)(fd.hi - fd.lo) * (fd.dim / 4);
    const unsigned grid = grid_for(work, 256, 148 * 32);
    if (bf16)
      k_init_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<__nv_bfloat16*>(w), fd.wbase, f,
                                                       fd.lo, fd.hi - fd.lo, fd.dim, seed);
    else
      k_init_rows<float><<<grid, 256, 0, st>>>(reinterpret_cast<float*>(w), fd.wbase, f, fd.lo,
                                               fd.hi - fd.lo, fd.dim, seed);
    S2D_LAUNCH_CHECK();
  }
}

void launch_combine(const CombineArgs& a, int max_dim, cudaStream_t st) {
  const uint64_t BF = (uint64_t)a.B * a.F;
  if (!BF) return;
  const int d4 = max_dim / 4;
  if (d4 <= 8)
    pdl_launch(k_combine<8, 1>, dim3(grid_for(BF, 256, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 16)
    pdl_launch(k_combine<16, 1>, dim3(grid_for(BF, 256, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 32)
    pdl_launch(k_combine<32, 1>, dim3(grid_for(BF, 256, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 64)
    pdl_launch(k_combine<32, 2>, dim3(grid_for(BF, 256, kGridCap)), dim3(256), 0, st, a);
  else
    pdl_launch(k_combine<32, 4>, dim3(grid_for(BF, 256, kGridCap)), dim3(256), 0, st, a);
}

void launch_grad_gather(const GradGatherArgs& a, int max_dim, cudaStream_t st) {
  const uint64_t BF = (uint64_t)a.B * a.F;
  if (!BF) return;
  const int d4 = max_dim / 4;
  if (d4 <= 8)
    pdl_launch(k_grad_gather<8, 1>, dim3(grid_for(BF, 32 * 4, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 16)
    pdl_launch(k_grad_gather<16, 1>, dim3(grid_for(BF, 16 * 4, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 32)
    pdl_launch(k_grad_gather<32, 1>, dim3(grid_for(BF, 8 * 4, kGridCap)), dim3(256), 0, st, a);
  else if (d4 <= 64)
    pdl_launch(k_grad_gather<32, 2>, dim3(grid_for(BF, 8 * 4, kGridCap)), dim3(256), 0, st, a);
  else
    pdl_launch(k_grad_gather<32, 4>, dim3(grid_for(BF, 8 * 4, kGridCap)), dim3(256), 0, st, a);
}

void launch_bucket_count(const BucketArgs& a, cudaStream_t st) {
  if (!a.BF) return;
  pdl_launch(k_bucket_count, dim3(grid_for(a.BF, 256, kGridCap)), dim3(256), 0, st, a);
}

void launch_bucket_permute(const BucketArgs& a, cudaStream_t st) {
  if (!a.BF) return;
  pdl_launch(k_bucket_permute, dim3(grid_for(a.BF, 256, kGridCap)), dim3(256), 0, st, a);
}

void launch_mean_prescale(const FeatDev* feats, uint32_t F, uint32_t B, uint32_t sum_dims, const uint32_t* bag_off,
                          const float* up, float* out, cudaStream_t st) {
  const uint64_t n = (uint64_t)B * (sum_dims / 4);
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  pdl_launch(k_mean_prescale, dim3(grid), dim3(256), 0, st, feats, F, B, sum_dims, bag_off, up, out);
}

}  // namespace s2d
