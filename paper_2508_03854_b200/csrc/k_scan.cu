// Device-wide exclusive scans used for bag offsets (lengths -> id offsets)
// and entry offsets (non-empty bag -> float offset of its partial/gradient
// row on the wire).  Three phases: per-tile reduce, scan of tile sums (one
// CTA), per-tile scan.  HBM-bound: reads the input twice, writes once.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "device.cuh"

namespace s2d {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

struct OpIdentity {
  __device__ __forceinline__ uint64_t operator()(uint32_t x, uint64_t) const { return x; }
};

struct OpHead {  // 1 at the first index of every run of equal valid keys
  const uint32_t* keys;
  uint32_t n_slots;
  __device__ __forceinline__ uint64_t operator()(uint32_t x, uint64_t k) const {
    return (x < n_slots && (k == 0 || __ldg(keys + k - 1) != x)) ? 1ull : 0ull;
  }
};

struct OpNonzeroDim {
  const FeatDev* feats;
  uint32_t F;
  __device__ __forceinline__ uint64_t operator()(uint32_t x, uint64_t k) const {
    return x ? (uint64_t)__ldg(&feats[k % F].dim) : 0ull;
  }
};

template <typename T, typename Op>
__global__ void __launch_bounds__(kThreads) k_tile_reduce(const uint32_t* __restrict__ in, uint64_t n,
                                                          Op op, T* __restrict__ tile_sum) {
  pdl_wait();
  using BlockReduce = cub::BlockReduce<T, kThreads>;
  __shared__ typename BlockReduce::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  T acc = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kThreads + threadIdx.x;
    if (k < n) acc += (T)op(__ldg(in + k), k);
  }
  const T s = BlockReduce(tmp).Sum(acc);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_scan_tiles(T* __restrict__ tile_sum, uint64_t ntiles) {
  pdl_wait();
  using BlockScan = cub::BlockScan<T, kThreads>;
  __shared__ typename BlockScan::TempStorage tmp;
  __shared__ T carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += kThreads) {
    const uint64_t k = base + threadIdx.x;
    T x = k < ntiles ? tile_sum[k] : 0;
    T excl, total;
    BlockScan(tmp).ExclusiveSum(x, excl, total);
    const T c = carry;
    if (k < ntiles) tile_sum[k] = c + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sum[ntiles] = carry;
}

template <typename T, typename Op>
__global__ void __launch_bounds__(kThreads) k_tile_scan(const uint32_t* __restrict__ in, uint64_t n, Op op,
                                                        const T* __restrict__ tile_sum, uint64_t ntiles,
                                                        T* __restrict__ out) {
  pdl_wait();
  using BlockScan = cub::BlockScan<T, kThreads>;
  __shared__ typename BlockScan::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  // blocked arrangement: thread t owns items [t*kItems, (t+1)*kItems)
  T v[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)threadIdx.x * kItems + i;
    v[i] = k < n ? (T)op(__ldg(in + k), k) : 0;
  }
  T excl[kItems];
  BlockScan(tmp).ExclusiveSum(v, excl);
  const T off = tile_sum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)threadIdx.x * kItems + i;
    if (k < n) out[k] = off + excl[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tile_sum[ntiles];
}

template <typename T, typename Op>
void scan_impl(const uint32_t* in, T* out, uint64_t n, Op op, cudaStream_t st, void* tmp,
               size_t tmp_bytes) {
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  if ((ntiles + 1) * sizeof(T) > tmp_bytes) throw Error(S2D_ECUDA, "scan workspace too small");
  T* tile_sum = reinterpret_cast<T*>(tmp);
  if (ntiles == 0) {
    S2D_CUDA(cudaMemsetAsync(out, 0, sizeof(T), st));
    return;
  }
  pdl_launch(k_tile_reduce<T, Op>, dim3((unsigned)ntiles), dim3(kThreads), 0, st, in, n, op, tile_sum);
  pdl_launch(k_scan_tiles<T>, dim3(1), dim3(kThreads), 0, st, tile_sum, ntiles);
  pdl_launch(k_tile_scan<T, Op>, dim3((unsigned)ntiles), dim3(kThreads), 0, st, in, n, op,
             static_cast<const T*>(tile_sum), ntiles, out);
}

// ---- fused pair: out32 = exclusive scan of x, out64 = exclusive scan of
// (x ? dim(k % F) : 0) over the same input in one read (ids and entry
// floats of the [peer][bag] count matrix) -----------------------------------
struct Pair {
  uint32_t a;
  uint64_t b;
};
struct PairSum {
  __device__ __forceinline__ Pair operator()(const Pair& x, const Pair& y) const { return {x.a + y.a, x.b + y.b}; }
};

__device__ __forceinline__ Pair pair_of(uint32_t x, uint64_t k, const FeatDev* feats, uint32_t F) {
  return {x, x ? (uint64_t)__ldg(&feats[k % F].dim) : 0ull};
}

__global__ void __launch_bounds__(kThreads) k_pair_reduce(const uint32_t* __restrict__ in, uint64_t n,
                                                          const FeatDev* feats, uint32_t F, Pair* __restrict__ tile_sum) {
  pdl_wait();
  using BR = cub::BlockReduce<Pair, kThreads>;
  __shared__ typename BR::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  Pair acc{0u, 0ull};
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kThreads + threadIdx.x;
    if (k < n) {
      const Pair p = pair_of(__ldg(in + k), k, feats, F);
      acc.a += p.a;
      acc.b += p.b;
    }
  }
  const Pair s = BR(tmp).Reduce(acc, PairSum());
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_pair_scan_tiles(Pair* __restrict__ tile_sum, uint64_t ntiles) {
  pdl_wait();
  using BS = cub::BlockScan<Pair, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ Pair carry;
  if (threadIdx.x == 0) carry = {0u, 0ull};
  __syncthreads();
  for (uint64_t base = 0; base < ntiles; base += kThreads) {
    const uint64_t k = base + threadIdx.x;
    const Pair x = k < ntiles ? tile_sum[k] : Pair{0u, 0ull};
    Pair excl, total;
    BS(tmp).ExclusiveScan(x, excl, Pair{0u, 0ull}, PairSum(), total);
    const Pair c = carry;
    if (k < ntiles) tile_sum[k] = {c.a + excl.a, c.b + excl.b};
    __syncthreads();
    if (threadIdx.x == 0) carry = {c.a + total.a, c.b + total.b};
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sum[ntiles] = carry;
}

__global__ void __launch_bounds__(kThreads) k_pair_tile_scan(const uint32_t* __restrict__ in, uint64_t n,
                                                             const FeatDev* feats, uint32_t F,
                                                             const Pair* __restrict__ tile_sum, uint64_t ntiles,
                                                             uint32_t* __restrict__ out32, uint64_t* __restrict__ out64) {
  pdl_wait();
  using BS = cub::BlockScan<Pair, kThreads>;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  Pair v[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)threadIdx.x * kItems + i;
    v[i] = k < n ? pair_of(__ldg(in + k), k, feats, F) : Pair{0u, 0ull};
  }
  Pair excl[kItems];
  BS(tmp).ExclusiveScan(v, excl, Pair{0u, 0ull}, PairSum());
  const Pair off = tile_sum[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = base + (uint64_t)threadIdx.x * kItems + i;
    if (k < n) {
      out32[k] = off.a + excl[i].a;
      out64[k] = off.b + excl[i].b;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out32[n] = tile_sum[ntiles].a;
    out64[n] = tile_sum[ntiles].b;
  }
}

__global__ void k_zero(uint4* p, size_t n16, uint8_t* tail, uint32_t tail_n) {
  pdl_wait();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) p[i] = make_uint4(0, 0, 0, 0);
  if (blockIdx.x == 0 && threadIdx.x < tail_n) tail[threadIdx.x] = 0;
}

}  // namespace

void launch_zero(void* p, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  if (reinterpret_cast<uintptr_t>(p) % 16) throw Error(S2D_ECUDA, "launch_zero needs a 16-byte aligned buffer");
  const size_t n16 = bytes / 16;
  const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((n16 + 255) / 256, 148 * 8));
  pdl_launch(k_zero, dim3(grid), dim3(256), 0, st, reinterpret_cast<uint4*>(p), n16,
             reinterpret_cast<uint8_t*>(p) + n16 * 16, (uint32_t)(bytes % 16));
}

size_t scan_tmp_bytes(uint64_t n) { return ((n + kTile - 1) / kTile + 1) * sizeof(Pair); }

void scan_count_pair(const uint32_t* in, uint32_t* out32, uint64_t* out64, uint64_t n, uint32_t F,
                     const FeatDev* feats, cudaStream_t st, void* tmp, size_t tmp_bytes) {
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  if ((ntiles + 1) * sizeof(Pair) > tmp_bytes) throw Error(S2D_ECUDA, "scan workspace too small");
  if (ntiles == 0) {
    S2D_CUDA(cudaMemsetAsync(out32, 0, sizeof(uint32_t), st));
    S2D_CUDA(cudaMemsetAsync(out64, 0, sizeof(uint64_t), st));
    return;
  }
  Pair* ts = reinterpret_cast<Pair*>(tmp);
  pdl_launch(k_pair_reduce, dim3((unsigned)ntiles), dim3(kThreads), 0, st, in, n, feats, F, ts);
  pdl_launch(k_pair_scan_tiles, dim3(1), dim3(kThreads), 0, st, ts, ntiles);
  pdl_launch(k_pair_tile_scan, dim3((unsigned)ntiles), dim3(kThreads), 0, st, in, n, feats, F,
             static_cast<const Pair*>(ts), ntiles, out32, out64);
}

void scan_u32_to_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t st, void* tmp,
                     size_t tmp_bytes) {
  scan_impl<uint32_t>(in, out, n, OpIdentity{}, st, tmp, tmp_bytes);
}

void scan_heads_u32(const uint32_t* keys, uint32_t* out, uint64_t n, uint32_t n_slots, cudaStream_t st,
                    void* tmp, size_t tmp_bytes) {
  scan_impl<uint32_t>(keys, out, n, OpHead{keys, n_slots}, st, tmp, tmp_bytes);
}

void scan_nonzero_dim_u64(const uint32_t* in, uint64_t* out, uint64_t n, uint32_t F,
                          const FeatDev* feats, cudaStream_t st, void* tmp, size_t tmp_bytes) {
  scan_impl<uint64_t>(in, out, n, OpNonzeroDim{feats, F}, st, tmp, tmp_bytes);
}

}  // namespace s2d
