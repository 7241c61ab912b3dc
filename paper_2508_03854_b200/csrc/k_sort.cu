// K3a: the dedup half of aggregate_group_gradient's stable_sort by row
// (src/optimizer.cpp:31-35) -- a stable sort of the lookup's (slot,
// gradient-row) pairs by slot.  Stability keeps each row's contributions in
// canonical arrival order, which the segment reduce relies on for bit-exact
// f64 sums.
//
// Slots span the whole shard (26 bits for config 2's 33.6M rows) but a step
// touches few of them (445K), so the keys are first compacted to dense ranks:
//   1. mark    -- one bit per touched slot (bitmap over the shard's slots);
//   2. ranks   -- exclusive popcount scan of the bitmap words; the same pass
//                 emits slot_of_dense[] and decides on the device how many
//                 10-bit digit passes the dense ranks need (config 2: 19 bits
//                 -> 2 passes instead of 3 over slot bits);
//   3. passes  -- LSD over the dense rank, 10-bit digits, reduce-then-scan:
//                 per-tile digit counts (digit-major), one exclusive scan of
//                 the count matrix, then a downsweep that ranks each tile
//                 stably (warp match-any), stages it in shared memory in
//                 digit order and stores each digit run contiguously.  No
//                 inter-CTA look-back chain.  The first pass maps slots to
//                 dense ranks on the fly; the last pass writes slots back
//                 (slot_of_dense) into the final buffers.
// The host launches the passes the key width can need; passes the device
// finds unnecessary exit at once, so the step needs no host round trip.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "device.cuh"

namespace s2d {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kIpt = 16;
constexpr int kTile = kThreads * kIpt;  // 4096 pairs
constexpr int kDBits = 10;
constexpr int kRadix = 1 << kDBits;
constexpr int kMaxPasses = 4;  // 40 bits: any 32-bit dense rank
constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;  // scan tile (count matrix / bitmap words)

// meta words (device): [0] U (distinct valid slots), [1] passes, [2 + p] pass p active
enum { kMetaU = 0, kMetaPasses = 1, kMetaActive = 2, kMetaWords = 8 };

struct Layout {
  uint64_t n, ntiles, n_words, cnt_n, cnt_tiles, word_tiles, sod_n;
  size_t bitmap_off, wpre_off, meta_off, sod_off, cnt_off, cscan_off, tsum_off, wsum_off, total;
};

size_t al(size_t x) { return (x + 255) / 256 * 256; }

Layout layout(uint64_t n, uint32_t n_slots) {
  Layout L;
  L.n = n;
  L.ntiles = (n + kTile - 1) / kTile;
  L.n_words = ((uint64_t)n_slots + 31) / 32 + 1;
  L.cnt_n = (uint64_t)kRadix * L.ntiles;
  L.cnt_tiles = (L.cnt_n + kScanTile - 1) / kScanTile;
  L.word_tiles = (L.n_words + kThreads * 4 - 1) / (kThreads * 4);
  L.sod_n = std::min<uint64_t>(n, n_slots) + 1;
  size_t o = 0;
  L.bitmap_off = o;
  o += al(L.n_words * 4);
  L.wpre_off = o;
  o += al((L.n_words + 1) * 4);
  L.meta_off = o;
  o += al(kMetaWords * 4);
  L.sod_off = o;
  o += al(L.sod_n * 4);
  L.cnt_off = o;
  o += al((L.cnt_n + 1) * 4);
  L.cscan_off = o;  // per-digit totals
  o += al(kRadix * 4);
  L.tsum_off = o;
  o += al((L.cnt_tiles + 1) * 4);
  L.wsum_off = o;
  o += al((L.word_tiles + 1) * 4);
  L.total = o;
  return L;
}

int bit_width64(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// K consecutive keys from `first` (16-byte vector loads when the run is in
// bounds and aligned; keys past n read as 0xffffffff)
template <int K>
__device__ __forceinline__ void load_keys(const uint32_t* __restrict__ keys, uint64_t n, uint64_t first,
                                          uint32_t (&k)[K]) {
  if (first + K <= n && (first & 3u) == 0) {
#pragma unroll
    for (int j = 0; j < K / 4; ++j) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(keys + first) + j);
      k[4 * j] = x.x, k[4 * j + 1] = x.y, k[4 * j + 2] = x.z, k[4 * j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) k[j] = first + j < n ? __ldg(keys + first + j) : 0xffffffffu;
  }
}

// ---- 1. mark touched slots ---------------------------------------------------

constexpr int kMarkThreads = 256;
constexpr int kMarkTile = kMarkThreads * 16;  // keys per CTA
constexpr int kMarkCache = 4096;              // direct-mapped cache of slots this CTA has marked

// Zipf-hot rows hit the same bitmap word from every CTA, and same-line
// requests serialise at an L2 slice: a per-CTA direct-mapped cache of the
// slots already marked keeps the hot rows' repeats on chip, so the bitmap
// sees about one atomicOr per distinct slot per tile.
__global__ void __launch_bounds__(kMarkThreads) k_dd_mark(const uint32_t* __restrict__ keys, uint64_t n,
                                                          uint32_t n_slots, uint32_t* bitmap) {
  pdl_wait();
  __shared__ uint32_t cache[kMarkCache];
  for (int i = threadIdx.x; i < kMarkCache; i += kMarkThreads) cache[i] = 0xffffffffu;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kMarkTile;
  constexpr int kPer = kMarkTile / kMarkThreads;
  uint32_t kk[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const uint64_t idx = base + (uint64_t)i * kMarkThreads + threadIdx.x;
    kk[i] = idx < n ? __ldg(keys + idx) : 0xffffffffu;
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const uint32_t k = kk[i];
    if (k >= n_slots) continue;
    uint32_t* c = cache + (k & (kMarkCache - 1));
    if (*(volatile uint32_t*)c == k) continue;
    *(volatile uint32_t*)c = k;
    atomicOr(bitmap + (k >> 5), 1u << (k & 31u));  // fire and forget (RED): no round trip on the critical path
  }
}

// ---- 2. dense ranks: exclusive popcount scan of the bitmap words ----------

__global__ void __launch_bounds__(kThreads) k_dd_word_reduce(const uint32_t* __restrict__ bitmap, uint64_t n_words,
                                                             uint32_t* __restrict__ wsum) {
  pdl_wait();
  using BR = cub::BlockReduce<uint32_t, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * (kThreads * 4);  // == kWordTile
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t k = base + (uint64_t)i * kThreads + threadIdx.x;
    if (k < n_words) acc += __popc(__ldg(bitmap + k));
  }
  const uint32_t s = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) wsum[blockIdx.x] = s;
}

// single CTA: exclusive scan of tile sums (in place, total at [ntiles]);
// when `meta` is given, derive U and the digit passes of the dense ranks
__global__ void __launch_bounds__(kThreads) k_dd_scan_tiles(uint32_t* __restrict__ tsum, uint64_t ntiles,
                                                            uint32_t* meta, uint32_t* sod, const uint32_t* gate) {
  pdl_wait();
  if (gate && !*gate) return;
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += kThreads) {
    const uint64_t k = base + threadIdx.x;
    const uint32_t x = k < ntiles ? tsum[k] : 0u;
    uint32_t excl, total;
    BS(tmp).ExclusiveSum(x, excl, total);
    const uint32_t c = carry;
    if (k < ntiles) tsum[k] = c + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tsum[ntiles] = carry;
    if (meta) {
      const uint32_t U = carry;
      int bits = 0;  // dense ranks 0..U (U = the invalid-slot sentinel)
      for (uint32_t x = U; x; x >>= 1) ++bits;
      if (bits < 1) bits = 1;
      const uint32_t passes = (uint32_t)((bits + kDBits - 1) / kDBits);
      meta[kMetaU] = U;
      meta[kMetaPasses] = passes;
      for (uint32_t p = 0; p < (uint32_t)kMaxPasses; ++p) meta[kMetaActive + p] = p < passes ? 1u : 0u;
      sod[U] = 0xffffffffu;
    }
  }
}

// per word tile: wpre[w] = dense rank of the first set bit of word w; emits
// slot_of_dense for every set bit (4 words per thread, one 16-byte load)
constexpr int kWordItems = 4;
constexpr int kWordTile = kThreads * kWordItems;

__global__ void __launch_bounds__(kThreads) k_dd_word_scan(const uint32_t* __restrict__ bitmap, uint64_t n_words,
                                                           const uint32_t* __restrict__ wsum,
                                                           uint32_t* __restrict__ wpre, uint32_t* __restrict__ sod) {
  pdl_wait();
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t k0 = (uint64_t)blockIdx.x * kWordTile + (uint64_t)threadIdx.x * kWordItems;
  uint32_t w[kWordItems], ex[kWordItems], c[kWordItems];
  if (k0 + kWordItems <= n_words) {  // the bitmap is 256-byte aligned
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(bitmap + k0));
    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w;
  } else {
#pragma unroll
    for (int i = 0; i < kWordItems; ++i) w[i] = k0 + i < n_words ? __ldg(bitmap + k0 + i) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kWordItems; ++i) c[i] = __popc(w[i]);
  BS(tmp).ExclusiveSum(c, ex);
  const uint32_t off = wsum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kWordItems; ++i) {
    const uint64_t k = k0 + i;
    if (k >= n_words) break;
    uint32_t r = off + ex[i];
    wpre[k] = r;
    for (uint32_t m = w[i]; m; m &= m - 1) sod[r++] = (uint32_t)(k * 32 + (__ffs(m) - 1));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) wpre[n_words] = wsum[gridDim.x];
}

__device__ __forceinline__ uint32_t dense_of(uint32_t slot, uint32_t n_slots, const uint32_t* __restrict__ bitmap,
                                             const uint32_t* __restrict__ wpre, uint32_t U) {
  if (slot >= n_slots) return U;
  const uint32_t w = slot >> 5;
  return __ldg(wpre + w) + __popc(__ldg(bitmap + w) & ((1u << (slot & 31u)) - 1u));
}

// ---- 3. LSD passes over the dense rank ------------------------------------

// per-tile digit counts, digit-major: cnt[d * ntiles + tile]
// per-tile digit counts, digit-major: cnt[d * ntiles + tile].  The first
// pass maps slots to dense ranks and writes them back in place (each key is
// read and rewritten by the same thread).
template <bool FIRST>
__global__ void __launch_bounds__(kThreads) k_dd_upsweep(uint32_t* __restrict__ keys, uint64_t n, int shift,
                                                         uint32_t n_slots, const uint32_t* __restrict__ bitmap,
                                                         const uint32_t* __restrict__ wpre,
                                                         const uint32_t* __restrict__ meta, int pass,
                                                         uint32_t* __restrict__ cnt) {
  pdl_wait();
  if (!__ldg(meta + kMetaActive + pass)) return;
  constexpr int kHW = 4;  // histogram copies (warps w, w + 4 share one)
  __shared__ uint32_t h[kHW][kRadix];
  for (int i = threadIdx.x; i < kHW * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t U = __ldg(meta + kMetaU);
  const uint64_t tbase = (uint64_t)blockIdx.x * kTile;
  uint32_t* const hw = h[(threadIdx.x >> 5) % kHW];
  uint32_t kk[kIpt];
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = tbase + (uint64_t)i * kThreads + threadIdx.x;
    kk[i] = idx < n ? keys[idx] : 0u;
  }
  if (FIRST) {
#pragma unroll
    for (int i = 0; i < kIpt; ++i) kk[i] = dense_of(kk[i], n_slots, bitmap, wpre, U);
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const uint64_t idx = tbase + (uint64_t)i * kThreads + threadIdx.x;
      if (idx < n) keys[idx] = kk[i];
    }
  }
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = tbase + (uint64_t)i * kThreads + threadIdx.x;
    if (idx < n) atomicAdd(&hw[(kk[i] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kThreads)
    cnt[(uint64_t)d * gridDim.x + blockIdx.x] = h[0][d] + h[1][d] + h[2][d] + h[3][d];
}

// per digit d (one CTA): exclusive prefix over the tiles of cnt[d][*] in
// place, and the digit's total; the downsweep scans the kRadix totals itself
constexpr int kRowItems = 8;
__global__ void __launch_bounds__(kThreads) k_dd_row_scan(uint32_t* __restrict__ cnt, uint32_t ntiles,
                                                          uint32_t* __restrict__ totals, const uint32_t* gate) {
  pdl_wait();
  if (!*gate) return;
  using BS = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  uint32_t* row = cnt + (uint64_t)blockIdx.x * ntiles;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < ntiles; base += kThreads * kRowItems) {
    uint32_t v[kRowItems], ex[kRowItems];
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const uint32_t k = base + threadIdx.x * kRowItems + i;
      v[i] = k < ntiles ? row[k] : 0u;
    }
    uint32_t total;
    BS(tmp).ExclusiveSum(v, ex, total);
    const uint32_t c = carry;
#pragma unroll
    for (int i = 0; i < kRowItems; ++i) {
      const uint32_t k = base + threadIdx.x * kRowItems + i;
      if (k < ntiles) row[k] = c + ex[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// exclusive scan of s[0..kRadix) in place (kRadix / kThreads entries per
// thread, warp shuffles + one smem round for the warp totals)
__device__ __forceinline__ void block_excl_scan(uint32_t* s, uint32_t* wtot) {
  constexpr int DPT = kRadix / kThreads;
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  uint32_t v[DPT], sum = 0;
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    v[i] = s[t * DPT + i];
    sum += v[i];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += y;
  }
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  uint32_t wbase = 0;
  for (uint32_t w = 0; w < warp; ++w) wbase += wtot[w];
  uint32_t run = wbase + inc - sum;
#pragma unroll
  for (int i = 0; i < DPT; ++i) {
    s[t * DPT + i] = run;
    run += v[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 3) k_dd_downsweep(const uint32_t* __restrict__ keys_in,
                                                           const uint32_t* __restrict__ vals_in,
                                                           uint32_t* __restrict__ keys_mid, uint32_t* __restrict__ vals_mid,
                                                           uint32_t* __restrict__ keys_fin, uint32_t* __restrict__ vals_fin,
                                                           uint64_t n, int shift, uint32_t n_slots,
                                                           const uint32_t* __restrict__ bitmap,
                                                           const uint32_t* __restrict__ wpre,
                                                           const uint32_t* __restrict__ sod,
                                                           const uint32_t* __restrict__ meta, int pass,
                                                           const uint32_t* __restrict__ coff,
                                                           const uint32_t* __restrict__ totals) {
  pdl_wait();
  if (!__ldg(meta + kMetaActive + pass)) return;
  constexpr int DPT = kRadix / kThreads;
  extern __shared__ __align__(16) unsigned char dsm[];
  uint32_t* const s_keys = reinterpret_cast<uint32_t*>(dsm);                     // [kTile]
  uint32_t* const s_vals = s_keys + kTile;                                      // [kTile]
  uint16_t (*const s_whist)[kRadix] = reinterpret_cast<uint16_t (*)[kRadix]>(s_vals + kTile);  // [kWarps][kRadix]
  uint32_t* const s_dstart = reinterpret_cast<uint32_t*>(&s_whist[kWarps][0]);  // in-tile digit starts
  uint32_t* const s_gbase = s_dstart + kRadix;  // global start of this tile's run of each digit
  uint32_t* const s_wtot = s_gbase + kRadix;    // [kWarps]

  const bool last = __ldg(meta + kMetaPasses) == (uint32_t)pass + 1;
  uint32_t* const keys_out = last ? keys_fin : keys_mid;
  uint32_t* const vals_out = last ? vals_fin : vals_mid;
  const uint32_t U = __ldg(meta + kMetaU);
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = blockIdx.x;
  const uint64_t tbase = tile * kTile;

  uint32_t k[kIpt], v[kIpt], d[kIpt], r[kIpt];
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint64_t idx = tbase + (uint64_t)warp * 32 * kIpt + (uint64_t)i * 32 + lane;
    const bool ok = idx < n;
    k[i] = ok ? __ldg(keys_in + idx) : 0u;
    v[i] = ok ? __ldg(vals_in + idx) : 0u;
    d[i] = ok ? (k[i] >> shift) & (kRadix - 1) : (uint32_t)kRadix;
  }
  // stable in-warp ranking; a warp's items in (i, lane) order == input order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    const uint32_t peers = __match_any_sync(0xffffffffu, d[i]);
    const uint32_t leader = __ffs(peers) - 1;
    const uint32_t below = __popc(peers & ((1u << lane) - 1u));
    uint32_t base = 0;
    if (lane == leader && d[i] < (uint32_t)kRadix) {
      base = s_whist[warp][d[i]];
      s_whist[warp][d[i]] = (uint16_t)(base + __popc(peers));
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    r[i] = base + below;
    __syncwarp();
  }
  __syncthreads();
  // per digit: offsets of the warps inside the digit, tile count, global base
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
    s_dstart[dg] = run;
    s_gbase[dg] = __ldg(totals + dg);  // scanned below into the digit's global base
  }
  __syncthreads();
  block_excl_scan(s_dstart, s_wtot);
  block_excl_scan(s_gbase, s_wtot);
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const uint32_t dg = threadIdx.x * DPT + j;
    s_gbase[dg] += __ldg(coff + (uint64_t)dg * gridDim.x + tile);  // + earlier tiles of the digit
  }
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int i = 0; i < kIpt; ++i) {
    if (d[i] < (uint32_t)kRadix) {
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
    const uint32_t dd = (key >> shift) & (kRadix - 1);
    const uint32_t pos = s_gbase[dd] + (idx - s_dstart[dd]);
    keys_out[pos] = last ? __ldg(sod + key) : key;
    vals_out[pos] = s_vals[idx];
  }
}

constexpr size_t kDownSmem = (size_t)2 * kTile * 4 + (size_t)kWarps * kRadix * 2 + (size_t)2 * kRadix * 4 + kWarps * 4;

}  // namespace

size_t dedup_sort_tmp_bytes(uint64_t n, uint32_t n_slots) { return layout(n, n_slots).total; }

int dedup_sort_max_passes(uint64_t n, uint32_t n_slots) {
  const uint64_t u = std::min<uint64_t>(n, n_slots);  // dense ranks 0..U
  return std::max(1, (bit_width64(u) + kDBits - 1) / kDBits);
}

uint32_t* dedup_sort_bitmap(void* tmp) { return reinterpret_cast<uint32_t*>(tmp); }  // bitmap_off == 0

size_t dedup_sort_bitmap_bytes(uint32_t n_slots) { return (((uint64_t)n_slots + 31) / 32 + 1) * 4; }

void dedup_sort(uint32_t* keys, const uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                uint32_t* keys_tmp2, uint32_t* vals_tmp2, uint32_t* keys_out, uint32_t* vals_out, uint64_t n,
                uint32_t n_slots, void* tmp, size_t tmp_bytes, bool premarked, cudaStream_t st) {
  if (n == 0) return;
  const Layout L = layout(n, n_slots);
  if (L.total > tmp_bytes) throw Error(S2D_ECUDA, "dedup sort workspace too small");
  char* b = reinterpret_cast<char*>(tmp);
  uint32_t* bitmap = reinterpret_cast<uint32_t*>(b + L.bitmap_off);
  uint32_t* wpre = reinterpret_cast<uint32_t*>(b + L.wpre_off);
  uint32_t* meta = reinterpret_cast<uint32_t*>(b + L.meta_off);
  uint32_t* sod = reinterpret_cast<uint32_t*>(b + L.sod_off);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(b + L.cnt_off);
  uint32_t* cscan = reinterpret_cast<uint32_t*>(b + L.cscan_off);
  uint32_t* tsum = reinterpret_cast<uint32_t*>(b + L.tsum_off);
  uint32_t* wsum = reinterpret_cast<uint32_t*>(b + L.wsum_off);
  // 1. mark (unless the producer of the keys marked the bitmap already)
  if (!premarked) {
    launch_zero(bitmap, L.n_words * 4, st);
    pdl_launch(k_dd_mark, dim3((unsigned)((n + kMarkTile - 1) / kMarkTile)), dim3(kMarkThreads), 0, st, keys, n,
               n_slots, bitmap);
  }
  // 2. dense ranks + pass plan
  pdl_launch(k_dd_word_reduce, dim3((unsigned)L.word_tiles), dim3(kThreads), 0, st,
             static_cast<const uint32_t*>(bitmap), L.n_words, wsum);
  pdl_launch(k_dd_scan_tiles, dim3(1), dim3(kThreads), 0, st, wsum, L.word_tiles, meta, sod,
             static_cast<const uint32_t*>(nullptr));
  pdl_launch(k_dd_word_scan, dim3((unsigned)L.word_tiles), dim3(kThreads), 0, st,
             static_cast<const uint32_t*>(bitmap), L.n_words, static_cast<const uint32_t*>(wsum), wpre, sod);
  // 3. passes: a -> tmp -> tmp2 -> ...; the last active pass writes the output
  set_max_dynamic_smem(k_dd_downsweep, kDownSmem);
  const int P = dedup_sort_max_passes(n, n_slots);
  uint32_t* in_k = keys;
  const uint32_t* in_v = vals;
  for (int p = 0; p < P; ++p) {
    uint32_t* mk = (p % 2 == 0) ? keys_tmp : keys_tmp2;
    uint32_t* mv = (p % 2 == 0) ? vals_tmp : vals_tmp2;
    const int shift = p * kDBits;
    const uint32_t* gate = meta + kMetaActive + p;
    if (p == 0)
      pdl_launch(k_dd_upsweep<true>, dim3((unsigned)L.ntiles), dim3(kThreads), 0, st, in_k, n, shift, n_slots,
                 static_cast<const uint32_t*>(bitmap), static_cast<const uint32_t*>(wpre),
                 static_cast<const uint32_t*>(meta), p, cnt);
    else
      pdl_launch(k_dd_upsweep<false>, dim3((unsigned)L.ntiles), dim3(kThreads), 0, st, in_k, n, shift, n_slots,
                 static_cast<const uint32_t*>(bitmap), static_cast<const uint32_t*>(wpre),
                 static_cast<const uint32_t*>(meta), p, cnt);
    pdl_launch(k_dd_row_scan, dim3(kRadix), dim3(kThreads), 0, st, cnt, (uint32_t)L.ntiles, cscan, gate);
    pdl_launch(k_dd_downsweep, dim3((unsigned)L.ntiles), dim3(kThreads), kDownSmem, st, static_cast<const uint32_t*>(in_k),
               in_v, mk, mv, keys_out, vals_out, n, shift, n_slots, static_cast<const uint32_t*>(bitmap),
               static_cast<const uint32_t*>(wpre), static_cast<const uint32_t*>(sod),
               static_cast<const uint32_t*>(meta), p, static_cast<const uint32_t*>(cnt),
               static_cast<const uint32_t*>(cscan));
    in_k = mk;
    in_v = mv;
  }
}

}  // namespace s2d
