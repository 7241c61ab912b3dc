// K3a: stable LSD radix sort of (slot, gradient-row) pairs -- the dedup
// half of aggregate_group_gradient's stable_sort by row
// (src/optimizer.cpp:31-35).  Stability keeps each row's contributions in
// canonical arrival order, which the segment reduce relies on for
// bit-exact f64 sums.
//
// One histogram kernel for all digit passes, then one single-sweep kernel
// per digit: tiles claimed in order through an atomic counter, stable
// in-tile ranking with warp match-any, decoupled look-back across tiles for
// the per-digit prefix, shared-memory staging so each digit run leaves the
// CTA as contiguous stores.  HBM traffic per pass: 8 B read + 8 B written
// per pair.  Digits are 8 or 9 bits, whichever needs fewer passes over the
// key width (26-bit slots of config 2: 9+9+8 instead of 8+8+8+2).
#include "device.cuh"

namespace s2d {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIpt = 16;
constexpr int kTile = kThreads * kIpt;  // 4096 pairs
constexpr int kMaxRadix = 512;
constexpr int kMaxPasses = 4;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

int digit_bits(int bits) {
  const int p8 = (bits + 7) / 8, p9 = (bits + 8) / 9;
  return p9 < p8 ? 9 : 8;
}

struct Layout {
  uint64_t ntiles;
  int dbits, radix, npass;
  size_t hist_off, lb_off, ctr_off, total;
};

Layout layout(uint64_t n, int bits) {
  Layout L;
  L.ntiles = (n + kTile - 1) / kTile;
  L.dbits = digit_bits(bits);
  L.radix = 1 << L.dbits;
  L.npass = (bits + L.dbits - 1) / L.dbits;
  if (L.npass < 1) L.npass = 1;
  L.hist_off = 0;
  L.lb_off = (size_t)kMaxPasses * kMaxRadix * 4;
  L.ctr_off = L.lb_off + (size_t)L.npass * L.ntiles * L.radix * sizeof(uint64_t);
  L.total = L.ctr_off + 256;
  return L;
}

__device__ __forceinline__ uint32_t digit_of(uint32_t key, int shift, int pbits) {
  return (key >> shift) & ((1u << pbits) - 1u);
}

template <int RADIX>
__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                         int bits, uint32_t* __restrict__ hist) {
  pdl_wait();
  constexpr int DB = RADIX == 512 ? 9 : 8;
  __shared__ uint32_t h[kMaxPasses][RADIX];
  for (int i = threadIdx.x; i < kMaxPasses * RADIX; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int npass = (bits + DB - 1) / DB;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kThreads) {
    const uint32_t k = __ldg(keys + i);
    for (int p = 0; p < npass; ++p) {
      const int shift = p * DB;
      const int pb = min(DB, bits - shift);
      atomicAdd(&h[p][digit_of(k, shift, pb)], 1u);
    }
  }
  __syncthreads();
  for (int p = 0; p < npass; ++p)
    for (int d = threadIdx.x; d < RADIX; d += kThreads) {
      const uint32_t c = h[p][d];
      if (c) atomicAdd(&hist[p * RADIX + d], c);
    }
}

// exclusive scan of s[0..RADIX) in place (RADIX / kThreads entries per
// thread, Hillis-Steele over the per-thread sums); all threads participate
template <int RADIX>
__device__ __forceinline__ void block_excl_scan(uint32_t* s, uint32_t* tmp) {
  constexpr int DPT = RADIX / kThreads;
  const uint32_t t = threadIdx.x;
  uint32_t v[DPT], sum = 0;
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    v[i] = s[t * DPT + i];
    sum += v[i];
  }
  tmp[t] = sum;
  __syncthreads();
  for (int off = 1; off < kThreads; off <<= 1) {
    const uint32_t add = t >= (uint32_t)off ? tmp[t - off] : 0u;
    __syncthreads();
    tmp[t] += add;
    __syncthreads();
  }
  uint32_t run = tmp[t] - sum;
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    s[t * DPT + i] = run;
    run += v[i];
  }
  __syncthreads();
}

template <int RADIX>
__global__ void __launch_bounds__(kThreads) k_radix_pass(const uint32_t* __restrict__ keys_in,
                                                         const uint32_t* __restrict__ vals_in,
                                                         uint32_t* __restrict__ keys_out,
                                                         uint32_t* __restrict__ vals_out, uint64_t n,
                                                         int shift, int pbits,
                                                         const uint32_t* __restrict__ hist,
                                                         uint64_t* lookback, uint32_t* tile_ctr) {
  pdl_wait();
  constexpr int DPT = RADIX / kThreads;  // digits per thread in the per-digit phases
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint16_t s_whist[kWarps][RADIX];  // per-warp digit counts, then warp offsets (<= kTile)
  __shared__ uint32_t s_dstart[RADIX];
  __shared__ uint32_t s_gbase[RADIX];  // n < 2^32 pairs per rank
  __shared__ uint32_t s_gdig[RADIX];
  __shared__ uint32_t s_tmp[kThreads];
  __shared__ uint32_t s_tile;

  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kWarps * RADIX; i += kThreads) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tbase = tile * kTile;

  uint32_t k[kIpt], v[kIpt], d[kIpt], r[kIpt];
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = tbase + (uint64_t)warp * 32 * kIpt + (uint64_t)i * 32 + lane;
    const bool ok = idx < n;
    k[i] = ok ? __ldg(keys_in + idx) : 0u;
    v[i] = ok ? __ldg(vals_in + idx) : 0u;
    d[i] = ok ? digit_of(k[i], shift, pbits) : (uint32_t)RADIX;
  }
  // stable in-warp ranking, items in (i, lane) order == input order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
    const uint32_t leader = __ffs(peers) - 1;
    const uint32_t below = __popc(peers & ((1u << lane) - 1u));
    uint32_t base = 0;
    if (lane == leader && d[i] < RADIX) {
      base = s_whist[warp][d[i]];
      s_whist[warp][d[i]] = (uint16_t)(base + __popc(peers));
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    r[i] = base + below;
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp offsets, tile count, publish the tile aggregate
  uint32_t count[DPT];
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const uint32_t dg = threadIdx.x * DPT + j;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_whist[w][dg];
      s_whist[w][dg] = (uint16_t)run;
      run += c;
    }
    count[j] = run;
    *((volatile uint64_t*)(lookback + tile * RADIX + dg)) = (tile == 0 ? kFlagInc : kFlagAgg) | run;
    s_dstart[dg] = run;
    s_gdig[dg] = hist[dg];
  }
  __syncthreads();
  block_excl_scan<RADIX>(s_dstart, s_tmp);  // in-tile digit starts
  block_excl_scan<RADIX>(s_gdig, s_tmp);    // global digit bases
  // look-back for this thread's DPT digits, walked in lockstep so their
  // L2 round trips overlap
  {
    uint64_t excl[DPT];
    int64_t t[DPT];
    bool done[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      excl[j] = 0;
      t[j] = (int64_t)tile - 1;
      done[j] = tile == 0;
    }
    bool all = tile == 0;
    while (!all) {
      uint64_t x[DPT];
#pragma unroll
      for (int j = 0; j < DPT; ++j)
        x[j] = done[j] ? 0ull : *((const volatile uint64_t*)(lookback + (uint64_t)t[j] * RADIX + threadIdx.x * DPT + j));
      all = true;
#pragma unroll
      for (int j = 0; j < DPT; ++j) {
        if (!done[j] && (x[j] >> 62) != 0) {
          excl[j] += x[j] & kValMask;
          if ((x[j] >> 62) == 2) done[j] = true;
          else --t[j];
        }
        all = all && done[j];
      }
    }
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const uint32_t dg = threadIdx.x * DPT + j;
      if (tile > 0) *((volatile uint64_t*)(lookback + tile * RADIX + dg)) = kFlagInc | (excl[j] + count[j]);
      s_gbase[dg] = s_gdig[dg] + (uint32_t)excl[j];
    }
  }
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    if (d[i] < RADIX) {
      const uint32_t lp = s_dstart[d[i]] + s_whist[warp][d[i]] + r[i];
      s_keys[lp] = k[i];
      s_vals[lp] = v[i];
    }
  }
  __syncthreads();
  const uint64_t rem = n - tbase;
  const uint32_t tile_n = rem < (uint64_t)kTile ? (uint32_t)rem : (uint32_t)kTile;
  for (uint32_t idx = threadIdx.x; idx < tile_n; idx += kThreads) {
    const uint32_t key = s_keys[idx];
    const uint32_t dd = digit_of(key, shift, pbits);
    const uint32_t pos = s_gbase[dd] + (idx - s_dstart[dd]);
    keys_out[pos] = key;
    vals_out[pos] = s_vals[idx];
  }
}

template <int RADIX>
bool sort_impl(const Layout& L, uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b, uint64_t n,
               int bits, char* base, cudaStream_t st) {
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + L.hist_off);
  uint64_t* lb = reinterpret_cast<uint64_t*>(base + L.lb_off);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(base + L.ctr_off);
  const unsigned hblocks = (unsigned)std::min<uint64_t>(L.ntiles * 2, 148 * 8);
  pdl_launch(k_radix_hist<RADIX>, dim3(hblocks ? hblocks : 1), dim3(kThreads), 0, st,
             static_cast<const uint32_t*>(keys_a), n, bits, hist);
  uint32_t *ki = keys_a, *vi = vals_a, *ko = keys_b, *vo = vals_b;
  for (int p = 0; p < L.npass; ++p) {
    const int shift = p * L.dbits;
    const int pb = std::min(L.dbits, bits - shift);
    pdl_launch(k_radix_pass<RADIX>, dim3((unsigned)L.ntiles), dim3(kThreads), 0, st, static_cast<const uint32_t*>(ki),
               static_cast<const uint32_t*>(vi), ko, vo, n, shift, pb, static_cast<const uint32_t*>(hist + p * RADIX),
               lb + (size_t)p * L.ntiles * RADIX, ctr + p);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  return (L.npass & 1) != 0;
}

}  // namespace

size_t radix_tmp_bytes(uint64_t n, int bits) { return layout(n, bits).total; }

bool radix_sort_pairs(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_b, uint32_t* vals_b,
                      uint64_t n, int bits, void* tmp, size_t tmp_bytes, cudaStream_t st) {
  if (n == 0) return false;
  if (bits < 1) bits = 1;
  if (bits > 32) bits = 32;
  const Layout L = layout(n, bits);
  if (L.total > tmp_bytes) throw Error(S2D_ECUDA, "radix sort workspace too small");
  char* base = reinterpret_cast<char*>(tmp);
  launch_zero(base, L.total, st);
  if (L.radix == 512) return sort_impl<512>(L, keys_a, vals_a, keys_b, vals_b, n, bits, base, st);
  return sort_impl<256>(L, keys_a, vals_a, keys_b, vals_b, n, bits, base, st);
}

}  // namespace s2d
