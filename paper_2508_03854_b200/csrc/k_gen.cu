// Device-side synthetic input: the reference DataGenerator's ids
// (DataGenerator ctor Zipf CDF, src/data.cpp:85-98; gen_batch_into ids,
// data.cpp:115-136), bit-exact.  Bag (s, f) draws L_f ids; draw j is
// u = (mix64(key + (j+1)*gamma) >> 11) * 2^-53 with
// key = make_key({seed, lane = 0, step, rank, s, tag = 1, f}) (rng.hpp), and
// id = min(upper_bound(cdf_f, u), rows_f - 1).  The CDF is the reference's
// sequential f64 prefix of (k+1)^-s divided by the total, built on the host
// with the same libm pow and cached on the device.  One thread per id; ids
// leave in (sample, feature, draw) order, bag lengths are L_f.
#include "device.cuh"

namespace s2d {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

__global__ void k_gen_ids(const GenArgs a) {
  const uint64_t total = (uint64_t)a.B * a.per_sample;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / a.per_sample), r = (uint32_t)(i % a.per_sample);
    uint32_t lo = 0, hi = a.F;  // feature f with cum[f] <= r < cum[f+1]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(a.cum + mid) <= r)
        lo = mid;
      else
        hi = mid;
    }
    const uint32_t f = lo, j = r - __ldg(a.cum + f);
    const uint64_t fields[7] = {a.seed, 0ull, a.step, a.rank, s, 1ull, f};
    uint64_t key = 0x8A5CD789635D2DFFULL;
#pragma unroll
    for (int q = 0; q < 7; ++q) key = mix64(key + 0x9E3779B97F4A7C15ULL + fields[q]);
    const double u = (double)(mix64(key + (uint64_t)(j + 1) * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
    const double* cdf = a.cdf + __ldg(a.cdf_off + f);
    const uint32_t rows = __ldg(a.rows + f);
    uint32_t b = 0, e = rows;  // upper_bound: first k with cdf[k] > u
    while (b < e) {
      const uint32_t m = b + ((e - b) >> 1);
      if (__ldg(cdf + m) > u)
        e = m;
      else
        b = m + 1;
    }
    a.ids[i] = b < rows - 1 ? b : rows - 1;
  }
}

__global__ void k_gen_lengths(const GenArgs a) {
  const uint64_t n = (uint64_t)a.B * a.F;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t f = (uint32_t)(i % a.F);
    a.lengths[i] = __ldg(a.cum + f + 1) - __ldg(a.cum + f);
  }
}

}  // namespace

void launch_gen_batch(const GenArgs& a, cudaStream_t st) {
  const uint64_t n_ids = (uint64_t)a.B * a.per_sample, n_bags = (uint64_t)a.B * a.F;
  if (n_bags) {
    k_gen_lengths<<<(unsigned)std::min<uint64_t>((n_bags + 255) / 256, 148 * 16), 256, 0, st>>>(a);
    S2D_LAUNCH_CHECK();
  }
  if (n_ids) {
    k_gen_ids<<<(unsigned)std::min<uint64_t>((n_ids + 255) / 256, 148 * 32), 256, 0, st>>>(a);
    S2D_LAUNCH_CHECK();
  }
}

}  // namespace s2d
