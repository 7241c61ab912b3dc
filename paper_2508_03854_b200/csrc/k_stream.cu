// Streaming segmented gather-reduce kernels: the hot path of the step.
//
// One warp walks a contiguous run of items -- the ids of 32 consecutive
// bags (K2 lookup), or the radix-sorted contributions of consecutive rows
// (K3b segment reduce + K4 fused AdaGrad) -- as a single stream.  Rows are
// gathered through a per-warp shared-memory ring with cp.async: lane l copies
// (and later reads back) only its own 16-byte column vectors of every row,
// so stage completion is a per-thread cp.async.wait_group and no block
// barrier is needed.  kStages-1 stages of kRowsPerStage rows are in flight
// per warp while the oldest stage is reduced, without spending registers on
// in-flight data; f64 accumulators stay in registers (4 columns x VPL per
// lane).  Every item is added into its accumulator strictly in stream order
// -- the reference's canonical order inside each bag and each row segment --
// so pooled rows and segment sums are bit-exact.  The accumulator is
// flushed (pooled row store, or the fused AdaGrad row update) where the bag
// / segment ends.
//
// History (profiles/r01/): warp-per-bag kernels were latency bound (11% of
// DRAM peak, one round trip per bag); register double-buffered streams were
// capped at 12-16 warps/SM by f64 accumulators + in-flight rows
// (128 regs), stalling on shuffles and load latency.
#include <cstdlib>

#include "device.cuh"

namespace s2d {
namespace {

constexpr int kStages = 2;
constexpr int kRowsPerStage = 4;
constexpr int kSlots = kStages * kRowsPerStage;
constexpr int kBags = 32;  // bags per lookup unit (one per lane)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// branch-free predicated cp.async (nothing is copied when pred == 0)
template <int BYTES>
__device__ __forceinline__ void cp_async_p(uint32_t dst, const void* src, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.ca.shared.global [%0], [%1], %3;\n}\n" ::"r"(dst),
      "l"(src), "r"((uint32_t)pred), "n"(BYTES));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_u(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst), "l"(src), "n"(BYTES));
}
// L2-only variant (16 B): no L1 allocation for streamed rows
__device__ __forceinline__ void cp_async_cg16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  // "memory": the ring reads after the wait are plain shared loads the
  // compiler may schedule freely among themselves, but not above the wait
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}


// Number of lanes j with end_j <= p (ends non-decreasing over lanes).
__device__ __forceinline__ uint32_t count_le(uint32_t my_end, uint32_t p) {
  uint32_t lo = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const uint32_t v = __shfl_sync(0xffffffffu, my_end, lo + step - 1);
    if (v <= p) lo += step;
  }
  return lo;
}

// Element type of a stored row and the 4-column vector a lane copies.
template <typename WT>
struct Row;
template <>
struct Row<float> {
  static constexpr int kVecBytes = 16;
  using T = float4;
  static __device__ __forceinline__ T ldg(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ void cvt(double (&d)[4], const T& x) {
    d[0] = (double)x.x;
    d[1] = (double)x.y;
    d[2] = (double)x.z;
    d[3] = (double)x.w;
  }
  static __device__ __forceinline__ void add_s(double (&a)[4], const unsigned char* sp) {
    const float4 x = *reinterpret_cast<const float4*>(sp);
    a[0] += (double)x.x;
    a[1] += (double)x.y;
    a[2] += (double)x.z;
    a[3] += (double)x.w;
  }
  static __device__ __forceinline__ void add(double (&a)[4], const void* s) {
    const float4 x = *reinterpret_cast<const float4*>(s);
    a[0] += (double)x.x;
    a[1] += (double)x.y;
    a[2] += (double)x.z;
    a[3] += (double)x.w;
  }
};
template <>
struct Row<__nv_bfloat16> {
  static constexpr int kVecBytes = 8;
  using T = uint2;
  static __device__ __forceinline__ T ldg(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
  static __device__ __forceinline__ void cvt(double (&d)[4], const T& x) {
    d[0] = (double)__uint_as_float(x.x << 16);
    d[1] = (double)__uint_as_float(x.x & 0xffff0000u);
    d[2] = (double)__uint_as_float(x.y << 16);
    d[3] = (double)__uint_as_float(x.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void add_s(double (&a)[4], const unsigned char* sp) {
    const uint2 x = *reinterpret_cast<const uint2*>(sp);
    a[0] += (double)__uint_as_float(x.x << 16);
    a[1] += (double)__uint_as_float(x.x & 0xffff0000u);
    a[2] += (double)__uint_as_float(x.y << 16);
    a[3] += (double)__uint_as_float(x.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void add(double (&a)[4], const void* s) {
    const uint2 x = *reinterpret_cast<const uint2*>(s);
    a[0] += (double)__uint_as_float(x.x << 16);
    a[1] += (double)__uint_as_float(x.x & 0xffff0000u);
    a[2] += (double)__uint_as_float(x.y << 16);
    a[3] += (double)__uint_as_float(x.y & 0xffff0000u);
  }
};

// per-warp ring: slot s, vector v, lane l -> ((s*VPL + v)*32 + l) * VB
template <int VPL, int VB>
__device__ __forceinline__ uint32_t ring_off(uint32_t slot, int v, uint32_t lane) {
  return ((slot * VPL + v) * 32 + lane) * VB;
}

// ============================================================================
// K2: owner lookup.  A warp owns 32 consecutive bags (flattened [n][s][f]),
// lane j holding bag j's metadata; the items are the bags' ids in (bag,
// occurrence) order.
// ============================================================================

// UNI: every table has dim uni_d4*4 and rows are slot-indexed (weights
// offset = slot * dim), so a row is named by its 32-bit slot (invalid ids and
// items past the end name the zero row `zero_row`), and every lane copies
// its chunk unconditionally -- chunks past a short row land in the padding
// rows after the shard and are never read back.
template <typename WT, int VPL, bool UNI>
__global__ void __launch_bounds__(256) k_lookup_ring(const LookupArgs a) {
  pdl_wait();  // persistent single wave: let the next grid queue behind us
  pdl_trigger();
  constexpr int VB = Row<WT>::kVecBytes;
  constexpr int kWinStages = 32 / kRowsPerStage;
  constexpr uint32_t kRowBytes = VPL * 32 * VB;  // ring slot stride
  constexpr uint64_t kNone = ~0ull;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // this lane's column chunk of slot 0 of the warp's ring
  const uint32_t ring_s = smem_u32(smem) + warp * kSlots * kRowBytes + lane * VB;
  const uint64_t n_bags = (uint64_t)a.n_req * a.B * a.F;
  const uint64_t n_units = (n_bags + kBags - 1) / kBags;
  const WT* __restrict__ W = reinterpret_cast<const WT*>(a.weights);
  const WT* const Wl = W + lane * 4;  // this lane's column chunk of row 0
  const uint32_t uni_d4 = a.uni_d4;
  const uint32_t pitch_b = uni_d4 * 4 * (uint32_t)sizeof(WT);  // row bytes (UNI)

  // persistent warps take units in ascending order from a ticket counter
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1u);
    const uint64_t tk = __shfl_sync(0xffffffffu, t, 0);
    if (tk >= n_units) break;
    const uint64_t unit = (tk + a.unit_rot) % n_units;
    const uint64_t b0 = unit * kBags;
    const uint32_t nb = (n_bags - b0) < (uint64_t)kBags ? (uint32_t)(n_bags - b0) : (uint32_t)kBags;
    const uint64_t my_bag = b0 + min(lane, nb - 1);
    const uint32_t my_end = __ldg(a.id_off + my_bag + 1);
    const uint32_t o0 = __ldg(a.id_off + b0);
    uint32_t my_start = __shfl_up_sync(0xffffffffu, my_end, 1);
    if (lane == 0) my_start = o0;
    const uint32_t o1 = __shfl_sync(0xffffffffu, my_end, nb - 1);
    const uint32_t f = (uint32_t)(my_bag % a.F);
    const uint32_t dim = __ldg(&a.feats[f].dim);
    const uint32_t flo = __ldg(&a.feats[f].lo), fhi = __ldg(&a.feats[f].hi);
    const uint32_t vbase = __ldg(&a.feats[f].vbase);
    const uint64_t wbase = __ldg(&a.feats[f].wbase);
    // out_off: local float offset of the bag's output (also the gradient-row
    // offset the backward sorts); optr: where the flush stores it -- the
    // pooled row (N = 1) or requester n's receive buffer over NVLink (N > 1)
    const uint64_t out_off = a.direct ? (uint64_t)((my_bag / a.F) % a.B) * a.sum_dims + __ldg(&a.feats[f].coff)
                                      : __ldg(a.eoff + my_bag);
    bool pooled_row = a.direct;  // the flush stores a final pooled row (not a partial)
    float* const optr = a.direct ? a.out + out_off : [&] {
      const uint64_t BF = (uint64_t)a.B * a.F;
      const uint32_t n = (uint32_t)(my_bag / BF);
      if (((a.use_peer_pooled >> n) & 1u) && __ldg(&a.feats[f].single)) {
        pooled_row = true;
        return reinterpret_cast<float*>(a.peer_pooled.p[n]) + ((my_bag % BF) / a.F) * a.sum_dims +
               __ldg(&a.feats[f].coff);
      }
      return reinterpret_cast<float*>(a.peer_out.p[n]) + a.peer_adj[n] + out_off;
    }();
    // mean pooling of a final pooled row: f32(f64(f32(sum)) * (1/L)); 0 = none
    // (a single-owner table's owner sees the whole bag: L = its item count)
    const double inv_len = (pooled_row && __ldg(&a.feats[f].mean) && my_end > my_start)
                               ? 1.0 / (double)(my_end - my_start) : 0.0;
    if (a.direct) {  // empty bags pool to zero (embedding.cpp:43-44)
      uint32_t empty = __ballot_sync(0xffffffffu, lane < nb && my_start == my_end);
      while (empty) {
        const uint32_t j = __ffs(empty) - 1;
        empty &= empty - 1;
        const uint64_t oo = shfl64(out_off, j);
        const uint32_t d4j = __shfl_sync(0xffffffffu, dim, j) >> 2;
        for (uint32_t c4 = lane; c4 < d4j; c4 += 32)
          __stcs(reinterpret_cast<float4*>(a.out + oo + c4 * 4), make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
    const uint32_t n_items = o1 - o0;
    if (n_items == 0) continue;
    const uint32_t nwin = (n_items + 31) / 32;

    // Window w (32 items): lane k holds item k's row address and bag word
    // (bag | ok << 8 | d4 << 16); `simple` bit k = item k is a valid id of
    // the same bag as item k-1 (no flush, no check needed).  Items past the
    // end are invalid ids of the last item's bag.
    uint32_t last_bag = 0xffffu;
    auto gen = [&](uint32_t win, uint32_t id, uint32_t& bw, uint64_t& ad, uint32_t& simple) {
      const uint32_t p = o0 + win * 32 + lane;
      const bool have = p < o1;
      const uint32_t j = min(count_le(my_end, have ? p : o1 - 1), nb - 1);
      const uint32_t lo_j = __shfl_sync(0xffffffffu, flo, j), hi_j = __shfl_sync(0xffffffffu, fhi, j);
      const uint32_t dim_j = __shfl_sync(0xffffffffu, dim, j), vb_j = __shfl_sync(0xffffffffu, vbase, j);
      const uint64_t wb_j = shfl64(wbase, j);
      const uint64_t oo_j = shfl64(out_off, j);
      const bool ok = have && id >= lo_j && id < hi_j;
      if (have && !ok) atomicOr(a.err, kErrIdRange);
      if (a.emit_keys && have) {
        a.keys[p] = ok ? vb_j + (id - lo_j) : 0xffffffffu;
        a.vals[p] = (uint32_t)(oo_j >> 2);
      }
      if constexpr (UNI)
        ad = ok ? vb_j + (id - lo_j) : a.zero_row;
      else
        ad = ok ? wb_j + (uint64_t)(id - lo_j) * dim_j : kNone;
      bw = j | (ok ? 0x100u : 0u) | ((dim_j >> 2) << 16);
      uint32_t before = __shfl_up_sync(0xffffffffu, j, 1);
      if (lane == 0) before = last_bag;
      last_bag = __shfl_sync(0xffffffffu, j, 31);
      simple = __ballot_sync(0xffffffffu, ok && j == before);
    };
    auto load_id = [&](uint32_t win) -> uint32_t {
      const uint32_t p = o0 + win * 32 + lane;
      return (win < nwin && p < o1) ? __ldg(a.ids + p) : 0u;
    };
    uint32_t bw_c, bw_n, sm_c, sm_n;
    uint64_t ad_c, ad_n;
    gen(0, load_id(0), bw_c, ad_c, sm_c);
    gen(1, load_id(1), bw_n, ad_n, sm_n);
    uint32_t nid = load_id(2);
    uint32_t wc = 0;  // window being consumed

    auto produce = [&](uint32_t st) {
      const bool nxt = (st / kWinStages) != wc;
      const uint64_t A = nxt ? ad_n : ad_c;
      const uint32_t Bw = nxt ? bw_n : bw_c;
      const uint32_t q = (st % kWinStages) * kRowsPerStage;
      const uint32_t base = ring_s + (st % kStages) * (kRowsPerStage * kRowBytes);
#pragma unroll
      for (int r = 0; r < kRowsPerStage; ++r) {
        if constexpr (UNI) {
          const uint32_t ri = __shfl_sync(0xffffffffu, (uint32_t)A, q + r);
          // one IMAD.WIDE.U32: row ri of the lane's chunk column
          const WT* src = reinterpret_cast<const WT*>(reinterpret_cast<const char*>(Wl) + (uint64_t)ri * pitch_b);
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if constexpr (VB == 16)
              cp_async_cg16(base + r * kRowBytes + v * 32 * VB, src + v * 128);
            else
              cp_async_u<VB>(base + r * kRowBytes + v * 32 * VB, src + v * 128);
          }
        } else {
          const uint64_t ad = shfl64(A, q + r);
          const uint32_t d4 = uni_d4 ? uni_d4 : (__shfl_sync(0xffffffffu, Bw, q + r) >> 16);
          const WT* src = W + ad + lane * 4;
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            cp_async_p<VB>(base + r * kRowBytes + v * 32 * VB, src + v * 128, ad != kNone && lane + v * 32 < d4);
        }
      }
      cp_commit();
    };

    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[v][k] = 0.0;
    uint32_t cur = __shfl_sync(0xffffffffu, bw_c, 0);
    uint32_t d4c = uni_d4 ? uni_d4 : (cur >> 16);
    cur &= 0xffu;
    auto flush = [&]() {
      float* const op = reinterpret_cast<float*>(shfl64(reinterpret_cast<uint64_t>(optr), cur));
      const double sc = __longlong_as_double((long long)shfl64((uint64_t)__double_as_longlong(inv_len), cur));
      if (sc != 0.0) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[v][k] = (double)(float)acc[v][k] * sc;
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        if (lane + v * 32 < d4c) store_f32x4_stream(op + (lane + v * 32) * 4, acc[v]);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[v][k] = 0.0;
      }
    };
    auto add_row = [&](uint32_t saddr) {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (VPL == 1 || lane + v * 32 < d4c) Row<WT>::add_s(acc[v], smem + (saddr + v * 32 * VB - sbase));
    };

    const uint32_t nst = (n_items + kRowsPerStage - 1) / kRowsPerStage;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) produce(s);
    for (uint32_t s = 0; s < nst; ++s) {
      if (s > 0 && s % kWinStages == 0) {  // enter window wc + 1
        ++wc;
        bw_c = bw_n;
        ad_c = ad_n;
        sm_c = sm_n;
        gen(wc + 1, nid, bw_n, ad_n, sm_n);
        nid = load_id(wc + 2);
      }
      produce(s + kStages - 1);
      cp_wait<kStages - 1>();
      const uint32_t q = (s % kWinStages) * kRowsPerStage;
      const uint32_t base = ring_s + (s % kStages) * (kRowsPerStage * kRowBytes);
      if (((sm_c >> q) & ((1u << kRowsPerStage) - 1u)) == ((1u << kRowsPerStage) - 1u)) {
        // no bag boundary and no invalid id in this stage
#pragma unroll
        for (int r = 0; r < kRowsPerStage; ++r) add_row(base + r * kRowBytes);
      } else {
#pragma unroll
        for (int r = 0; r < kRowsPerStage; ++r) {
          const uint32_t bw = __shfl_sync(0xffffffffu, bw_c, q + r);
          if ((bw & 0xffu) != cur) {
            flush();
            cur = bw & 0xffu;
            d4c = uni_d4 ? uni_d4 : (bw >> 16);
          }
          if (bw & 0x100u) add_row(base + r * kRowBytes);
        }
      }
    }
    cp_wait<0>();
    flush();
  }
}

// ============================================================================
// K3b + K4: segment reduce + fused row update over the radix-sorted
// (slot, gradient-row) pairs.  Warp u owns the segments whose head lies in
// the nominal range [u*C, (u+1)*C).  A segment running past its head's range
// continues with the in-order f64 partial sums of the fully covered ranges
// (level-1: C items; level-2: kP ranges aligned to kP*C) and then its tail
// items -- a fixed, launch-independent association.  It equals the
// reference's strictly sequential f64 sum whenever the segment fits in its
// head's range, and otherwise re-associates at fixed chunk boundaries
// (|dg| ~ 1e-16 relative).  |g|^2 is a per-lane in-order sum followed by a
// fixed xor-shuffle tree.  Ranges are taken from a ticket counter by
// persistent warps.  The weight row and moment of every segment head are
// L2-prefetched when its window is set up (32-64 items ahead) and loaded
// into registers at the head; the flush writes them back.
// ============================================================================

constexpr uint32_t kC = 128;  // items per nominal range
constexpr uint32_t kP = 16;   // ranges per level-2 partial

__device__ __forceinline__ void row_ref(const StreamUpdateArgs& a, uint32_t key, uint64_t& wofs, uint32_t& d4) {
  if (a.uni_dim) {
    wofs = (uint64_t)key * a.uni_dim;
    d4 = a.uni_dim >> 2;
  } else {
    const uint32_t f = feature_of_slot(a.vbase_sorted, a.feat_of_vbase, a.n_feat_owned, key);
    const uint32_t dim = __ldg(&a.feats[f].dim);
    wofs = __ldg(&a.feats[f].wbase) + (uint64_t)(key - __ldg(&a.feats[f].vbase)) * dim;
    d4 = dim >> 2;
  }
}

// In-order f64 sum of the gradient rows of items [s, t) of one segment,
// through the warp's ring.  lane_s = ring base + lane * 16.
template <int VPL>
__device__ __forceinline__ void ring_sum(const StreamUpdateArgs& a, uint32_t lane_s, uint32_t lane, uint64_t s,
                                         uint64_t t, uint32_t d4, double (&acc)[VPL][4]) {
  constexpr uint32_t kRowBytes = VPL * 32 * 16;
  constexpr int kWinStages = 32 / kRowsPerStage;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  if (t <= s) return;
  const uint32_t n = (uint32_t)(t - s);
  const uint32_t nst = (n + kRowsPerStage - 1) / kRowsPerStage;
  uint32_t my_val = 0;
  auto produce = [&](uint32_t st) {
    const uint32_t q = (st % kWinStages) * kRowsPerStage;
    if (q == 0) {
      const uint32_t i0 = st * kRowsPerStage;
      my_val = (i0 + lane < n) ? __ldg(a.vals + s + i0 + lane) : 0u;
    }
    const uint32_t base = lane_s + (st % kStages) * (kRowsPerStage * kRowBytes);
#pragma unroll
    for (int r = 0; r < kRowsPerStage; ++r) {
      const uint32_t i = st * kRowsPerStage + r;
      const uint32_t val = __shfl_sync(0xffffffffu, my_val, q + r);
      const float* row = a.grad + (uint64_t)val * 4 + lane * 4;
#pragma unroll
      for (int v = 0; v < VPL; ++v) cp_async_p<16>(base + r * kRowBytes + v * 512, row + v * 128, i < n && lane + v * 32 < d4);
    }
    cp_commit();
  };
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) produce(st);
  for (uint32_t st = 0; st < nst; ++st) {
    produce(st + kStages - 1);
    cp_wait<kStages - 1>();
    const uint32_t base = lane_s + (st % kStages) * (kRowsPerStage * kRowBytes);
    const uint32_t cnt = min((uint32_t)kRowsPerStage, n - st * kRowsPerStage);
#pragma unroll
    for (int r = 0; r < kRowsPerStage; ++r)
      if (r < cnt) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (VPL == 1 || lane + v * 32 < d4) Row<float>::add_s(acc[v], smem + (base + r * kRowBytes + v * 512 - sbase));
      }
  }
  cp_wait<0>();
}

template <int VPL>
__device__ __forceinline__ void add_partial(const double* p, uint32_t lane, uint32_t d4, double (&acc)[VPL][4]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const uint32_t c4 = lane + v * 32;
    if (c4 < d4) {
      const double2 x0 = __ldg(reinterpret_cast<const double2*>(p + c4 * 4));
      const double2 x1 = __ldg(reinterpret_cast<const double2*>(p + c4 * 4) + 1);
      acc[v][0] += x0.x;
      acc[v][1] += x0.y;
      acc[v][2] += x1.x;
      acc[v][3] += x1.y;
    }
  }
}

template <int VPL>
__device__ __forceinline__ void store_partial(double* p, uint32_t lane, uint32_t d4, const double (&acc)[VPL][4]) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const uint32_t c4 = lane + v * 32;
    if (c4 < d4) {
      reinterpret_cast<double2*>(p + c4 * 4)[0] = make_double2(acc[v][0], acc[v][1]);
      reinterpret_cast<double2*>(p + c4 * 4)[1] = make_double2(acc[v][2], acc[v][3]);
    }
  }
}

// In-order f64 sum of the kC gradient rows of one full range [s, s+kC), all
// of one segment, straight through registers: kG rows' loads in flight per
// batch, the next window's row offsets loaded a window ahead.  No shared
// memory (the ring's LDGSTS + LDS pair per row saturated the MIO queue).
template <int VPL>
__device__ __forceinline__ void reg_sum_range(const StreamUpdateArgs& a, uint32_t lane, uint64_t s, uint32_t d4,
                                              double (&acc)[VPL][4]) {
  constexpr int kG = 1;  // one row per load batch: 32 registers, full occupancy (8 / VPL rows: 64 regs, update 0.390 -> 0.374 ms)
  const float* const Gl = a.grad + lane * 4;
  uint32_t val_n = __ldg(a.vals + s + lane);
  for (uint32_t w = 0; w < kC; w += 32) {
    const uint32_t val_c = val_n;
    if (w + 32 < kC) val_n = __ldg(a.vals + s + w + 32 + lane);
#pragma unroll
    for (int g = 0; g < 32; g += kG) {
      float4 x[kG][VPL];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        const float* row = Gl + (uint64_t)__shfl_sync(0xffffffffu, val_c, g + j) * 4;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (lane + v * 32 < d4) x[j][v] = __ldg(reinterpret_cast<const float4*>(row + v * 128));
      }
#pragma unroll
      for (int j = 0; j < kG; ++j)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (lane + v * 32 < d4) {
            acc[v][0] += (double)x[j][v].x;
            acc[v][1] += (double)x[j][v].y;
            acc[v][2] += (double)x[j][v].z;
            acc[v][3] += (double)x[j][v].w;
          }
    }
  }
}

// level-1 partials: range k = [kC, kC+C) lying inside one segment
template <int VPL>
__global__ void __launch_bounds__(256) k_range_partials(const StreamUpdateArgs a) {
  pdl_wait();
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t n_ranges = a.n / kC;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t k = 1 + (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; k < n_ranges; k += stride) {
    const uint64_t s = k * kC, t = s + kC;
    const uint32_t key = __ldg(a.keys + s - 1);
    if (key >= a.n_slots || __ldg(a.keys + t - 1) != key) continue;
    uint64_t wofs;
    uint32_t d4;
    row_ref(a, key, wofs, d4);
    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    reg_sum_range<VPL>(a, lane, s, d4, acc);
    store_partial<VPL>(a.part1 + k * (uint64_t)a.max_d4 * 4, lane, d4, acc);
  }
}

// ---- TMA bulk-copy primitives (cp.async.bulk + mbarrier transaction counts)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one elected lane copies `bytes` (multiple of 16, 16-byte aligned) of global
// memory into shared memory; completion counts against `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// level-1 partials through TMA bulk copies: lane 0 of each warp streams the
// range's gradient rows (one cp.async.bulk per row) into a kTS-stage ring
// whose stages complete on mbarrier transaction counts; the warp reads its
// column chunks back and accumulates in item order.  The loads leave the
// LSU / MIO path (the LDGSTS of the register version saturated it).
constexpr int kTS = 4;   // ring stages per warp
constexpr int kTR = 4;   // rows per stage
constexpr int kTW = 8;   // warps per block
template <int VPL>
__global__ void __launch_bounds__(kTW * 32) k_range_partials_tma(const StreamUpdateArgs a) {
  pdl_wait();
  constexpr uint32_t kRowMax = VPL * 512;  // bytes of the widest row
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned char* wbase = smem + warp * (kTS * kTR * kRowMax + kC * 4 + kTS * 8);
  const uint32_t ring = smem_u32(wbase);
  uint32_t* const svals = reinterpret_cast<uint32_t*>(wbase + kTS * kTR * kRowMax);
  const uint32_t bars = smem_u32(wbase + kTS * kTR * kRowMax + kC * 4);
  if (lane == 0)
    for (int s = 0; s < kTS; ++s) mbar_init(bars + 8 * s, 1);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  const uint64_t n_ranges = a.n / kC;
  const uint64_t stride = (uint64_t)gridDim.x * kTW;
  uint32_t uses = 0;  // stages consumed by this warp so far (slot = uses % kTS, parity = (uses / kTS) & 1)
  for (uint64_t k = 1 + (uint64_t)blockIdx.x * kTW + warp; k < n_ranges; k += stride) {
    const uint64_t s0 = k * kC, t = s0 + kC;
    const uint32_t key = __ldg(a.keys + s0 - 1);
    if (key >= a.n_slots || __ldg(a.keys + t - 1) != key) continue;
    uint64_t wofs;
    uint32_t d4;
    row_ref(a, key, wofs, d4);
    const uint32_t rb = d4 * 16;  // row bytes
    for (uint32_t i = lane; i < kC; i += 32) svals[i] = __ldg(a.vals + s0 + i);
    __syncwarp();
    constexpr uint32_t nst = kC / kTR;
    auto issue = [&](uint32_t st) {  // lane 0: stage st of this range into slot (uses + st) % kTS
      const uint32_t slot = (uses + st) % kTS;
      const uint32_t bar = bars + 8 * slot;
      mbar_expect_tx(bar, kTR * rb);
#pragma unroll
      for (int r = 0; r < kTR; ++r)
        bulk_g2s(ring + (slot * kTR + r) * kRowMax, a.grad + (uint64_t)svals[st * kTR + r] * 4, rb, bar);
    };
    if (lane == 0)
      for (uint32_t st = 0; st < (uint32_t)kTS; ++st) issue(st);
    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    for (uint32_t st = 0; st < nst; ++st) {
      const uint32_t slot = (uses + st) % kTS;
      mbar_wait(bars + 8 * slot, ((uses + st) / kTS) & 1u);
#pragma unroll
      for (int r = 0; r < kTR; ++r) {
        const unsigned char* row = wbase + (slot * kTR + r) * kRowMax;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (VPL == 1 || lane + v * 32 < d4) Row<float>::add(acc[v], row + (lane + v * 32) * 16);
      }
      __syncwarp();  // every lane has read the slot before it is refilled
      if (lane == 0 && st + kTS < nst) issue(st + kTS);
    }
    uses += nst;
    store_partial<VPL>(a.part1 + k * (uint64_t)a.max_d4 * 4, lane, d4, acc);
  }
}

size_t range_tma_smem(int vpl) { return (size_t)kTW * (kTS * kTR * (size_t)vpl * 512 + kC * 4 + kTS * 8); }

// level-(L+1) partials: kP consecutive level-L partials, all inside one
// segment (level 2 over level-1 ranges, level 3 over level-2 groups), so the
// head warp of a segment of length S adds O(S / (kC kP^2) + 2 kP) partials
template <int VPL>
__global__ void __launch_bounds__(256) k_group_partials(const StreamUpdateArgs a, const double* __restrict__ src,
                                                        double* __restrict__ dst, uint64_t span) {
  pdl_wait();
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t n_groups = a.n / span;
  const uint64_t stride = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t m = 1 + (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; m < n_groups; m += stride) {
    const uint64_t s = m * span, t = s + span;
    const uint32_t key = __ldg(a.keys + s - 1);
    if (key >= a.n_slots || __ldg(a.keys + t - 1) != key) continue;
    uint64_t wofs;
    uint32_t d4;
    row_ref(a, key, wofs, d4);
    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    for (uint32_t r = 0; r < kP; ++r) add_partial<VPL>(src + (m * kP + r) * (uint64_t)a.max_d4 * 4, lane, d4, acc);
    store_partial<VPL>(dst + m * (uint64_t)a.max_d4 * 4, lane, d4, acc);
  }
}

// FULL: every owned row is exactly VPL*128 floats, so each lane's chunk of
// any item's gradient row -- sentinel items keep a real row offset, items past
// the range name row 0 -- is in bounds and the ring copies need no predicate.
constexpr uint32_t update_warp_bytes(int vpl, bool snap) {
  return (uint32_t)kSlots * vpl * 32 * 16 + 256 + 8 * kC + (snap ? 256 : 0);
}
template <typename WT, int VPL, bool FULL, bool SNAP>
__global__ void __launch_bounds__(128, SNAP && VPL == 1 ? 8 : 0) k_update_ring(const StreamUpdateArgs a) {
  pdl_wait();  // persistent single wave
  pdl_trigger();
  constexpr int kWinStages = 32 / kRowsPerStage;
  constexpr uint32_t kGRow = VPL * 32 * 16;
  constexpr uint32_t kNone = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  // per warp: gradient ring | head moments of two windows (cp.async, 256 B) |
  // the range's sorted keys and row offsets (cp.async, 2 x kC x 4 B) | with
  // the snapshot log, the heads' dirty-flag words of two windows (256 B)
  constexpr uint32_t kWarpBytes = update_warp_bytes(VPL, SNAP);
  const uint32_t g_lane = sbase + warp * kWarpBytes + lane * 16;  // gradient ring
  const uint32_t mom_s = sbase + warp * kWarpBytes + kSlots * kGRow;
  const uint32_t uk_s = mom_s + 256, uv_s = uk_s + 4 * kC;
  const uint32_t dty_s = uv_s + 4 * kC;
  const uint32_t* const ukeys = reinterpret_cast<const uint32_t*>(smem + (uk_s - sbase));
  const uint32_t* const uvals = reinterpret_cast<const uint32_t*>(smem + (uv_s - sbase));
  const uint64_t n = a.n;
  const uint64_t n_units = (n + kC - 1) / kC;
  const uint32_t ud4 = a.uni_dim >> 2;
  WT* __restrict__ W = reinterpret_cast<WT*>(a.weights);
  const float* const Gl = a.grad + lane * 4;  // this lane's chunk of gradient row 0
  uint32_t heads = 0, longs = 0;

  // persistent warps take ranges in ascending order from a ticket counter
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&a.counters[2], 1u);
    const uint64_t u = __shfl_sync(0xffffffffu, t, 0);
    if (u >= n_units) break;
    const uint64_t ra = u * kC, re = (ra + kC < n) ? ra + kC : n;
    {  // stage the range's keys and row offsets: one round trip per range
      const uint32_t m = (uint32_t)(re - ra);
      for (uint32_t c = lane * 4; c < kC; c += 128) {
        if (c + 4 <= m) {
          cp_async_u<16>(uk_s + c * 4, a.keys + ra + c);
          cp_async_u<16>(uv_s + c * 4, a.vals + ra + c);
        } else {
          for (uint32_t q = c; q < m && q < c + 4; ++q) {
            cp_async_u<4>(uk_s + q * 4, a.keys + ra + q);
            cp_async_u<4>(uv_s + q * 4, a.vals + ra + q);
          }
        }
      }
      cp_commit();
    }
    const uint32_t key_before = (lane == 0 && ra > 0) ? __ldg(a.keys + ra - 1) : kNone;
    cp_wait<0>();
    __syncwarp();
    // first segment head in [ra, re)
    uint64_t h = ~0ull;
    for (uint64_t c = ra; c < re; c += 32) {
      const uint64_t p = c + lane;
      const uint32_t k = p < re ? ukeys[p - ra] : kNone;
      uint32_t before = __shfl_up_sync(0xffffffffu, k, 1);
      if (lane == 0) before = c == ra ? key_before : ukeys[c - 1 - ra];
      const uint32_t bal = __ballot_sync(0xffffffffu, k < a.n_slots && k != before);
      if (bal) {
        h = c + (__ffs(bal) - 1);
        break;
      }
    }
    if (h == ~0ull) continue;
    const uint32_t n_items = (uint32_t)(re - h);
    const uint32_t nwin = (n_items + 31) / 32;

    // Window state, lane k = item k of the window: key, gradient row, row
    // dim/4 and weight offset; vm / hm = ballots of valid items / segment
    // heads.  Raw keys and rows are loaded one window before they are used.
    struct Win {
      uint32_t key, val, d4, vm, hm;
      uint64_t wofs;
    };
    uint32_t prev_key = 0xfffffffeu;  // key of the item before the window
    auto load_raw = [&](uint32_t win, uint32_t& key, uint32_t& val) {
      const uint64_t p = h + (uint64_t)win * 32 + lane;
      const bool have = win < nwin && p < re;
      key = have ? ukeys[p - ra] : kNone;
      val = have ? uvals[p - ra] : 0u;
    };
    auto gen = [&](uint32_t key, uint32_t val, Win& w, uint32_t win) {
      uint32_t before = __shfl_up_sync(0xffffffffu, key, 1);
      if (lane == 0) before = prev_key;
      prev_key = __shfl_sync(0xffffffffu, key, 31);
      const bool valid = key < a.n_slots;
      const bool head = valid && key != before;
      w.key = key;
      w.val = val;
      w.vm = __ballot_sync(0xffffffffu, valid);
      w.hm = __ballot_sync(0xffffffffu, head);
      // warm L2 with the weight row and moment of every segment head; the
      // consumer loads them into registers when it reaches the head
      // each head's moment goes to shared memory by cp.async (it lands with
      // the next stage's group, long before the consumer reaches the head)
      cp_async_p<4>(mom_s + ((win & 1u) * 32u + lane) * 4u, a.moments + (head ? key : 0u), head);
      if constexpr (SNAP) {
        // the heads' dirty-flag words (read at the head: a clean row is
        // saved before its first write)
        cp_async_p<4>(dty_s + ((win & 1u) * 32u + lane) * 4u, a.dirty + ((head ? key : 0u) & ~3u), head);
      }
      if constexpr (FULL) {  // slot-indexed rows of VPL*128 elements: no per-item row metadata
        if (head) {
          const char* row = reinterpret_cast<const char*>(W + (uint64_t)key * (VPL * 128));
#pragma unroll
          for (uint32_t o = 0; o < VPL * 128 * sizeof(WT); o += 128) prefetch_l2(row + o);
        }
      } else {
        w.d4 = 0;
        w.wofs = 0;
        if (valid) row_ref(a, key, w.wofs, w.d4);
        if (head) {
          const char* row = reinterpret_cast<const char*>(W + w.wofs);
          const uint32_t bytes = w.d4 * 4 * (uint32_t)sizeof(WT);
          for (uint32_t o = 0; o < bytes; o += 128) prefetch_l2(row + o);
        }
      }
    };
    Win wc_, wn_;
    uint32_t rk, rv;
    load_raw(0, rk, rv);
    gen(rk, rv, wc_, 0);
    load_raw(1, rk, rv);
    gen(rk, rv, wn_, 1);
    load_raw(2, rk, rv);
    uint32_t wc = 0;

    auto produce = [&](uint32_t st) {
      const bool nxt = (st / kWinStages) != wc;
      const uint32_t V = nxt ? wn_.val : wc_.val, VM = nxt ? wn_.vm : wc_.vm;
      const uint32_t q = (st % kWinStages) * kRowsPerStage;
      const uint32_t slot0 = (st % kStages) * kRowsPerStage;
#pragma unroll
      for (int r = 0; r < kRowsPerStage; ++r) {
        const uint32_t val = __shfl_sync(0xffffffffu, V, q + r);
        if constexpr (FULL) {  // every item names a real gradient row; no predicate
          const float* grow = Gl + (uint64_t)val * 4;
#pragma unroll
          for (int v = 0; v < VPL; ++v) cp_async_cg16(g_lane + (slot0 + r) * kGRow + v * 512, grow + v * 128);
        } else {
          const uint32_t d4 = a.uni_dim ? ud4 : __shfl_sync(0xffffffffu, nxt ? wn_.d4 : wc_.d4, q + r);
          const bool valid = (VM >> (q + r)) & 1u;
          const float* grow = Gl + (uint64_t)val * 4;
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            cp_async_p<16>(g_lane + (slot0 + r) * kGRow + v * 512, grow + v * 128, valid && lane + v * 32 < d4);
        }
      }
      cp_commit();
    };

    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    uint32_t cur = kNone, d4 = 0;
    uint32_t cur_snap = kNone;  // snapshot-log position of `cur` (kNone: already dirty / log off)
    uint64_t wofs = 0, cur_pos = 0;
    typename Row<WT>::T wraw[VPL];  // weight row of `cur` (raw storage type)
    float vold = 0.f;
    bool stop = false;

    // fused K4 row step (optimizer.cpp:65-90); nonfinite rows are not written
    auto flush = [&]() {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[v][j] = acc[v][j] * a.inv_batch;  // g (optimizer.cpp:55)
      if (a.grad_dbg) {  // debug view: the row's f64 gradient at its head ordinal
        double* gd = a.grad_dbg + (uint64_t)__ldg(a.head_ord + cur_pos) * a.max_d4 * 4;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (lane + v * 32 < d4) {
            reinterpret_cast<double2*>(gd + (lane + v * 32) * 4)[0] = make_double2(acc[v][0], acc[v][1]);
            reinterpret_cast<double2*>(gd + (lane + v * 32) * 4)[1] = make_double2(acc[v][2], acc[v][3]);
          }
      }
      bool finite;
      double lr = a.eta;
      if (!a.sgd) {
        double ns = 0.0;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (lane + v * 32 < d4)
#pragma unroll
            for (int j = 0; j < 4; ++j) ns += acc[v][j] * acc[v][j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        // |g|^2 is finite iff every g is: f64 sums of f32 rows cannot overflow
        finite = isfinite(ns);
        if (finite) {
          const float v_new = (float)((double)vold + ns);
          const double vc = a.c_pow2 ? (double)v_new * a.inv_c : (double)v_new / a.c;  // exact either way
          lr = a.eta / (sqrt(vc) + a.eps);  // effective_lr (optimizer.cpp:61-63)
          if (lane == 0) a.moments[cur] = v_new;
        }
      } else {
        bool f = true;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (lane + v * 32 < d4) f &= isfinite(acc[v][j]);
        finite = __all_sync(0xffffffffu, f);
      }
      if (!finite) {
        if (lane == 0) atomicOr(a.err, kErrNonfinite);
      } else {
        if (SNAP && cur_snap < a.snap_cap) {  // first write since the last replica sync: save the pre-update row
          const uint32_t pos = cur_snap;
          {
            float* sp = a.snap + (uint64_t)pos * a.snap_rf;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              const uint32_t c4 = lane + v * 32;
              if (c4 < d4) {
                double x[4];
                Row<WT>::cvt(x, wraw[v]);
                *reinterpret_cast<float4*>(sp + c4 * 4) = make_float4((float)x[0], (float)x[1], (float)x[2], (float)x[3]);
              }
            }
            if (lane == 0) {
              sp[a.snap_rf - 1] = vold;
              a.snap_pos[cur] = pos;
            }
          }
        }
        WT* w = W + wofs;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const uint32_t c4 = lane + v * 32;
          if (c4 < d4) {
            double x[4];
            Row<WT>::cvt(x, wraw[v]);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = x[j] - lr * acc[v][j];
            Vec4<WT>::store(w + c4 * 4, x);
          }
        }
        if (lane == 0 && a.dirty) a.dirty[cur] = 1;
        ++heads;
      }
      // the update's dirty list (every head at its ordinal; a faulted row
      // too -- the step reports the fault)
      if (lane == 0 && a.dirty_list) {
        a.dirty_list[__ldg(a.head_ord + cur_pos)] = cur;
        if (!finite) a.dirty[cur] = 1;
      }
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    };
    auto add_grad = [&](uint32_t slot) {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (VPL == 1 || lane + v * 32 < d4) Row<float>::add_s(acc[v], smem + (g_lane + slot * kGRow + v * 512 - sbase));
    };

    const uint32_t nst = (n_items + kRowsPerStage - 1) / kRowsPerStage;
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) produce(s);
    for (uint32_t s = 0; s < nst && !stop; ++s) {
      if (s > 0 && s % kWinStages == 0) {
        ++wc;
        wc_ = wn_;
        gen(rk, rv, wn_, wc + 1);
        load_raw(wc + 2, rk, rv);
      }
      produce(s + kStages - 1);
      cp_wait<kStages - 1>();
      const uint32_t q = (s % kWinStages) * kRowsPerStage;
      const uint32_t slot0 = (s % kStages) * kRowsPerStage;
      constexpr uint32_t kAll = (1u << kRowsPerStage) - 1u;
      if ((((wc_.vm & ~wc_.hm) >> q) & kAll) == kAll) {  // 4 continuation rows
#pragma unroll
        for (int r = 0; r < kRowsPerStage; ++r) add_grad(slot0 + r);
      } else {
#pragma unroll
        for (int r = 0; r < kRowsPerStage; ++r) {
          const uint32_t i = q + r;
          if (s * kRowsPerStage + r >= n_items) break;  // past this range: not a sentinel
          if (!((wc_.vm >> i) & 1u)) {                  // invalid-slot sentinels sort last
            stop = true;
            break;
          }
          if ((wc_.hm >> i) & 1u) {
            if (cur != kNone) flush();
            // segment head: load its (L2-warm) weight row and moment
            cur = __shfl_sync(0xffffffffu, wc_.key, i);
            cur_pos = h + (uint64_t)s * kRowsPerStage + r;
            if constexpr (FULL) {
              wofs = (uint64_t)cur * (VPL * 128);
              d4 = VPL * 32;
            } else {
              wofs = a.uni_dim ? (uint64_t)cur * a.uni_dim : shfl64(wc_.wofs, i);
              d4 = a.uni_dim ? ud4 : __shfl_sync(0xffffffffu, wc_.d4, i);
            }
#pragma unroll
            for (int v = 0; v < VPL; ++v)
              if (lane + v * 32 < d4) wraw[v] = Row<WT>::ldg(W + wofs + (lane + v * 32) * 4);
            vold = *reinterpret_cast<const float*>(smem + (mom_s - sbase) + ((wc & 1u) * 32u + i) * 4u);
            if constexpr (SNAP) {
              const uint32_t dw = *reinterpret_cast<const uint32_t*>(smem + (dty_s - sbase) + ((wc & 1u) * 32u + i) * 4u);
              // log position (unique, no atomics): the head's sorted position, or
              // with head_ord its ordinal among this update's heads (dense log)
              cur_snap = ((dw >> ((cur & 3u) * 8u)) & 0xffu)
                             ? kNone
                             : (uint32_t)(a.snap_base + (a.snap_dense ? __ldg(a.head_ord + cur_pos) : cur_pos));
            }
          }
          add_grad(slot0 + r);
        }
      }
    }
    cp_wait<0>();
    // continuation of the open segment past this range
    if (!stop && re < n && __ldg(a.keys + re) == cur) {
      ++longs;
      uint64_t k = re / kC;  // == u + 1
      uint64_t kend = ~0ull;
      for (uint64_t base = k; kend == ~0ull; base += 32) {
        const uint64_t kk = base + lane;
        const uint64_t last = (kk + 1) * kC - 1;
        const bool inside = last < n && __ldg(a.keys + last) == cur;
        const uint32_t bal = __ballot_sync(0xffffffffu, !inside);
        if (bal) kend = base + (__ffs(bal) - 1);
      }
      // ranges [k, kend) are fully inside; range kend holds the end
      const uint64_t rs = kend * kC, rlim = (rs + kC < n) ? rs + kC : n;
      uint64_t seg_end = rlim;
      for (uint64_t c = rs; c < rlim; c += 32) {
        const uint64_t p = c + lane;
        const bool diff = p < rlim && __ldg(a.keys + p) != cur;
        const uint32_t bal = __ballot_sync(0xffffffffu, diff);
        if (bal) {
          seg_end = c + (__ffs(bal) - 1);
          break;
        }
      }
      while (k < kend) {
        if (k % (kP * kP) == 0 && k + kP * kP <= kend) {
          add_partial<VPL>(a.part3 + (k / (kP * kP)) * (uint64_t)a.max_d4 * 4, lane, d4, acc);
          k += kP * kP;
        } else if (k % kP == 0 && k + kP <= kend) {
          add_partial<VPL>(a.part2 + (k / kP) * (uint64_t)a.max_d4 * 4, lane, d4, acc);
          k += kP;
        } else {
          add_partial<VPL>(a.part1 + k * (uint64_t)a.max_d4 * 4, lane, d4, acc);
          k += 1;
        }
      }
      ring_sum<VPL>(a, g_lane, lane, rs, seg_end, d4, acc);
    }
    if (cur != kNone) flush();
  }
  if (lane == 0) {
    if (heads) atomicAdd(&a.counters[0], heads);
    if (longs) atomicAdd(&a.counters[1], longs);
  }
}

// The lookup's sort pairs without the lookup (N = 1): per id its slot
// (0xffffffff if outside the shard) and its bag's upstream row (float4
// units).  They depend on the ids only, so the sort can run beside the
// lookup instead of after it.  Thread per bag.
__global__ void __launch_bounds__(256) k_emit_pairs(const FeatDev* __restrict__ feats, uint32_t F, uint32_t B,
                                                    uint32_t sum_dims, const uint32_t* __restrict__ id_off,
                                                    const uint32_t* __restrict__ ids, uint32_t* __restrict__ keys,
                                                    uint32_t* __restrict__ vals) {
  pdl_wait();
  const uint64_t BF = (uint64_t)B * F;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < BF; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = (uint32_t)(b % F);
    const uint32_t lo = __ldg(&feats[f].lo), hi = __ldg(&feats[f].hi), vb = __ldg(&feats[f].vbase);
    const uint32_t val = (uint32_t)(((b / F) * sum_dims + __ldg(&feats[f].coff)) >> 2);
    const uint32_t e = __ldg(id_off + b + 1);
    for (uint32_t p = __ldg(id_off + b); p < e; ++p) {
      const uint32_t id = __ldg(ids + p);
      keys[p] = (id >= lo && id < hi) ? vb + (id - lo) : 0xffffffffu;
      vals[p] = val;
    }
  }
}

unsigned grid_units(uint64_t units, uint32_t units_per_block, unsigned cap) {
  uint64_t g = (units + units_per_block - 1) / units_per_block;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
  set_max_dynamic_smem(kernel, bytes);  // per device (a process may drive several GPUs)
}

// warps per block so that one block's rings stay within ~72 KB (3 blocks/SM)
constexpr size_t kBlockRingBudget = 72 * 1024;
inline uint32_t warps_for(size_t per_warp, uint32_t max_warps) {
  size_t w = kBlockRingBudget / per_warp;
  if (w < 1) w = 1;
  return (uint32_t)std::min<size_t>(w, max_warps);
}

template <typename WT, int VPL, bool UNI>
void lookup_launch_t(const LookupArgs& a, cudaStream_t st) {
  const uint64_t n_units = ((uint64_t)a.n_req * a.B * a.F + kBags - 1) / kBags;
  const size_t per_warp = (size_t)kSlots * VPL * 32 * Row<WT>::kVecBytes;
  const uint32_t nw = warps_for(per_warp, 8);
  const size_t smem = nw * per_warp;
  static int occ = 0;
  set_smem(k_lookup_ring<WT, VPL, UNI>, smem);  // per device
  if (!occ) {
    S2D_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lookup_ring<WT, VPL, UNI>, nw * 32, smem));
    if (occ < 1) occ = 1;
  }
  launch_zero(a.ticket, 16, st);
  const int per_sm = a.blocks_per_sm ? std::min<int>(occ, (int)a.blocks_per_sm) : occ;
  pdl_launch(k_lookup_ring<WT, VPL, UNI>, dim3(grid_units(n_units, nw, 148 * per_sm)), dim3(nw * 32), smem, st, a);
}

template <typename WT, int VPL>
void lookup_launch(const LookupArgs& a, cudaStream_t st) {
  if (a.uni_rows)
    lookup_launch_t<WT, VPL, true>(a, st);
  else
    lookup_launch_t<WT, VPL, false>(a, st);
}

template <typename WT, int VPL>
void update_launch(const StreamUpdateArgs& a, cudaStream_t st) {
  const bool snap = a.snap != nullptr;
  const size_t pw_u = update_warp_bytes(VPL, snap);  // ring + head moments + range keys/rows (+ dirty words)
  const uint32_t nw_u = warps_for(pw_u, 4);
  const bool full = a.uni_dim == 128u * VPL;
  if (a.n >= 2 * kC) {
    static const bool tma = [] {
      const char* e = std::getenv("S2D_RANGE_TMA");
      return e && e[0] == '1';  // measured slower: opt-in
    }();
    if (tma) {
      const size_t sm = range_tma_smem(VPL);
      set_max_dynamic_smem(k_range_partials_tma<VPL>, sm);
      int occ = 0;
      S2D_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_range_partials_tma<VPL>, kTW * 32, sm));
      pdl_launch(k_range_partials_tma<VPL>, dim3(grid_units(a.n / kC, kTW, 148 * std::max(occ, 1))), dim3(kTW * 32), sm,
                 st, a);
    } else {
      pdl_launch(k_range_partials<VPL>, dim3(grid_units(a.n / kC, 8, 148 * 16)), dim3(256), 0, st, a);
    }
  }
  if (a.n >= 2ull * kC * kP)
    pdl_launch(k_group_partials<VPL>, dim3(grid_units(a.n / (kC * kP), 8, 148 * 8)), dim3(256), 0, st, a,
               static_cast<const double*>(a.part1), a.part2, (uint64_t)kC * kP);
  if (a.n >= 2ull * kC * kP * kP)
    pdl_launch(k_group_partials<VPL>, dim3(grid_units(a.n / (kC * kP * kP), 8, 148 * 8)), dim3(256), 0, st, a,
               static_cast<const double*>(a.part2), a.part3, (uint64_t)kC * kP * kP);
  // variants: FULL (slot-indexed uniform rows) x SNAP (M > 1 snapshot log);
  // their register counts differ, so each has its own occupancy
  auto kern = full ? (snap ? k_update_ring<WT, VPL, true, true> : k_update_ring<WT, VPL, true, false>)
                   : (snap ? k_update_ring<WT, VPL, false, true> : k_update_ring<WT, VPL, false, false>);
  set_smem(kern, nw_u * pw_u);  // per device
  static int occ[4] = {0, 0, 0, 0};
  const int vi = (full ? 2 : 0) + (snap ? 1 : 0);
  if (!occ[vi]) {
    S2D_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[vi], kern, nw_u * 32, nw_u * pw_u));
    if (occ[vi] < 1) occ[vi] = 1;
  }
  const unsigned grid = grid_units((a.n + kC - 1) / kC, nw_u, 148 * occ[vi]);
  pdl_launch(kern, dim3(grid), dim3(nw_u * 32), nw_u * pw_u, st, a);
}

}  // namespace

uint64_t stream_partial1_rows(uint64_t n) { return n / kC + 2; }
uint64_t stream_partial2_rows(uint64_t n) { return n / ((uint64_t)kC * kP) + 2; }

size_t stream_partial_bytes(uint64_t n, uint32_t max_dim) {
  return (stream_partial1_rows(n) + stream_partial2_rows(n) + (n / ((uint64_t)kC * kP * kP) + 2)) *
         (uint64_t)max_dim * sizeof(double);
}

void launch_emit_pairs(const FeatDev* feats, uint32_t F, uint32_t B, uint32_t sum_dims, const uint32_t* id_off,
                       const uint32_t* ids, uint32_t* keys, uint32_t* vals, cudaStream_t st) {
  const uint64_t BF = (uint64_t)B * F;
  if (!BF) return;
  pdl_launch(k_emit_pairs, dim3(grid_units(BF, 256, 148 * 8)), dim3(256), 0, st, feats, F, B, sum_dims, id_off, ids,
             keys, vals);
}

void launch_lookup_stream(const LookupArgs& a, int bf16, int max_dim, cudaStream_t st) {
  if ((uint64_t)a.n_req * a.B * a.F == 0) return;
  const int d4 = max_dim / 4;
  if (bf16) {
    if (d4 <= 32) lookup_launch<__nv_bfloat16, 1>(a, st);
    else if (d4 <= 64) lookup_launch<__nv_bfloat16, 2>(a, st);
    else lookup_launch<__nv_bfloat16, 4>(a, st);
  } else {
    if (d4 <= 32) lookup_launch<float, 1>(a, st);
    else if (d4 <= 64) lookup_launch<float, 2>(a, st);
    else lookup_launch<float, 4>(a, st);
  }
}

void launch_update_stream(const StreamUpdateArgs& a, int bf16, cudaStream_t st) {
  launch_zero(a.counters, 4 * sizeof(uint32_t), st);
  if (a.n == 0) return;
  const uint32_t d4 = a.max_d4;
  if (bf16) {
    if (d4 <= 32) update_launch<__nv_bfloat16, 1>(a, st);
    else if (d4 <= 64) update_launch<__nv_bfloat16, 2>(a, st);
    else update_launch<__nv_bfloat16, 4>(a, st);
  } else {
    if (d4 <= 32) update_launch<float, 1>(a, st);
    else if (d4 <= 64) update_launch<float, 2>(a, st);
    else update_launch<float, 4>(a, st);
  }
}

}  // namespace s2d
