// K3a: stable LSD radix sort of (slot, gradient-row) pairs -- the dedup
// half of aggregate_group_gradient's stable_sort by row
// (src/optimizer.cpp:31-35).  Stability keeps each row's contributions in
// canonical arrival order, which the segment reduce relies on for
// bit-exact f64 sums.
//
// One histogram kernel for all digit passes, then one single-sweep kernel
// per 8-bit digit: tiles claimed in order through an atomic counter, stable
// in-tile ranking with warp match-any, decoupled look-back across tiles for
// the per-digit prefix, shared-memory staging so each digit run leaves the
// CTA as contiguous stores.  HBM traffic per pass: 8 B read + 8 B written
// per pair.
#include "device.cuh"

namespace s2d {
namespace {

constexpr int kBits = 8;
constexpr int kRadix = 1 << kBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIpt = 16;
constexpr int kTile = kThreads * kIpt;  // 4096 pairs
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

static_assert(kThreads == kRadix, "one thread per digit in the look-back");

struct Layout {
  uint64_t ntiles;
  int npass;
  size_t hist_off, lb_off, ctr_off, total;
};

Layout layout(uint64_t n, int bits) {
  Layout L;
  L.ntiles = (n + kTile - 1) / kTile;
  L.npass = (bits + kBits - 1) / kBits;
  if (L.npass < 1) L.npass = 1;
  L.hist_off = 0;
  L.lb_off = 4096;  // hist: up to 4 passes x 256 u32
  L.ctr_off = L.lb_off + (size_t)L.npass * L.ntiles * kRadix * sizeof(uint64_t);
  L.total = L.ctr_off + 256;
  return L;
}

__device__ __forceinline__ uint32_t digit_of(uint32_t key, int shift, int pbits) {
  return (key >> shift) & ((1u << pbits) - 1u);
}

__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                         int bits, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[4][kRadix];
  for (int i = threadIdx.x; i < 4 * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const int npass = (bits + kBits - 1) / kBits;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * kThreads) {
    const uint32_t k = __ldg(keys + i);
    for (int p = 0; p < npass; ++p) {
      const int shift = p * kBits;
      const int pb = min(kBits, bits - shift);
      atomicAdd(&h[p][digit_of(k, shift, pb)], 1u);
    }
  }
  __syncthreads();
  for (int p = 0; p < npass; ++p) {
    const uint32_t c = h[p][threadIdx.x];
    if (c) atomicAdd(&hist[p * kRadix + threadIdx.x], c);
  }
}

__global__ void __launch_bounds__(kThreads) k_radix_pass(const uint32_t* __restrict__ keys_in,
                                                         const uint32_t* __restrict__ vals_in,
                                                         uint32_t* __restrict__ keys_out,
                                                         uint32_t* __restrict__ vals_out, uint64_t n,
                                                         int shift, int pbits,
                                                         const uint32_t* __restrict__ hist,
                                                         uint64_t* lookback, uint32_t* tile_ctr) {
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint32_t s_whist[kWarps][kRadix];
  __shared__ uint32_t s_dstart[kRadix];
  __shared__ uint64_t s_gbase[kRadix];
  __shared__ uint32_t s_scan[kRadix];
  __shared__ uint32_t s_tile;

  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&s_whist[0][0])[i] = 0;
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
    d[i] = ok ? digit_of(k[i], shift, pbits) : (uint32_t)kRadix;
  }
  // stable in-warp ranking, items in (i, lane) order == input order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
    const uint32_t leader = __ffs(peers) - 1;
    const uint32_t below = __popc(peers & ((1u << lane) - 1u));
    uint32_t base = 0;
    if (lane == leader && d[i] < kRadix) {
      base = s_whist[warp][d[i]];
      s_whist[warp][d[i]] = base + __popc(peers);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    r[i] = base + below;
    __syncwarp();
  }
  __syncthreads();
  // thread t handles digit t: warp offsets, tile count, look-back
  const uint32_t dg = threadIdx.x;
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = s_whist[w][dg];
    s_whist[w][dg] = run;
    run += c;
  }
  const uint32_t count = run;
  uint64_t* lb = lookback + tile * kRadix + dg;
  if (tile == 0) {
    *((volatile uint64_t*)lb) = kFlagInc | count;
  } else {
    *((volatile uint64_t*)lb) = kFlagAgg | count;
  }
  // in-tile digit starts and global digit bases (Hillis-Steele over 256)
  s_scan[dg] = count;
  __syncthreads();
  for (int off = 1; off < kRadix; off <<= 1) {
    const uint32_t add = dg >= (uint32_t)off ? s_scan[dg - off] : 0u;
    __syncthreads();
    s_scan[dg] += add;
    __syncthreads();
  }
  s_dstart[dg] = s_scan[dg] - count;
  __syncthreads();
  s_scan[dg] = hist[dg];
  __syncthreads();
  for (int off = 1; off < kRadix; off <<= 1) {
    const uint32_t add = dg >= (uint32_t)off ? s_scan[dg - off] : 0u;
    __syncthreads();
    s_scan[dg] += add;
    __syncthreads();
  }
  const uint64_t gdig = (uint64_t)s_scan[dg] - hist[dg];
  uint64_t excl = 0;
  if (tile > 0) {
    for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
      const volatile uint64_t* p = lookback + (uint64_t)t * kRadix + dg;
      uint64_t x;
      do {
        x = *p;
      } while ((x >> 62) == 0);
      excl += x & kValMask;
      if ((x >> 62) == 2) break;
    }
    *((volatile uint64_t*)lb) = kFlagInc | (excl + count);
  }
  s_gbase[dg] = gdig + excl;
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    if (d[i] < kRadix) {
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
    const uint64_t pos = s_gbase[dd] + (idx - s_dstart[dd]);
    keys_out[pos] = key;
    vals_out[pos] = s_vals[idx];
  }
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
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + L.hist_off);
  uint64_t* lb = reinterpret_cast<uint64_t*>(base + L.lb_off);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(base + L.ctr_off);
  S2D_CUDA(cudaMemsetAsync(base, 0, L.total, st));
  const unsigned hblocks = (unsigned)std::min<uint64_t>(L.ntiles * 2, 148 * 8);
  k_radix_hist<<<hblocks ? hblocks : 1, kThreads, 0, st>>>(keys_a, n, bits, hist);
  S2D_LAUNCH_CHECK();
  uint32_t *ki = keys_a, *vi = vals_a, *ko = keys_b, *vo = vals_b;
  for (int p = 0; p < L.npass; ++p) {
    const int shift = p * kBits;
    const int pb = std::min(kBits, bits - shift);
    k_radix_pass<<<(unsigned)L.ntiles, kThreads, 0, st>>>(ki, vi, ko, vo, n, shift, pb,
                                                          hist + p * kRadix,
                                                          lb + (size_t)p * L.ntiles * kRadix, ctr + p);
    S2D_LAUNCH_CHECK();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  return (L.npass & 1) != 0;
}

}  // namespace s2d
