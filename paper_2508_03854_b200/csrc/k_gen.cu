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
    const uint64_t fields[7] = {a.seed, a.lane, a.step, a.rank, s, 1ull, f};
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

// Synthetic per-sample upstream gradient of the embedding path (SURVEY.md
// 8(d); oracle or_synthetic_upstream): out[s][coff_f + j] =
// f32(1e-3 * z_j), z the Box-Muller normals of CounterRng({seed, step, rank,
// s, f}) in draw order (rng.hpp next_normal: cos first, then the cached sin).
// One thread per (s, f, pair of columns).
__global__ void k_gen_upstream(uint64_t seed, uint64_t step, uint32_t rank, uint32_t B, uint32_t F,
                               const FeatDev* __restrict__ feats, uint32_t sum_dims, uint32_t max_pairs,
                               float* __restrict__ out) {
  const uint64_t total = (uint64_t)B * F * max_pairs;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = (uint32_t)(i % max_pairs);
    const uint64_t sf = i / max_pairs;
    const uint32_t f = (uint32_t)(sf % F), s = (uint32_t)(sf / F);
    const uint32_t D = __ldg(&feats[f].dim);
    if (2 * p >= D) continue;
    const uint64_t fields[5] = {seed, step, rank, s, f};
    uint64_t key = 0x8A5CD789635D2DFFULL;
#pragma unroll
    for (int q = 0; q < 5; ++q) key = mix64(key + 0x9E3779B97F4A7C15ULL + fields[q]);
    const uint64_t c1 = 2ull * p + 1, c2 = 2ull * p + 2;
    const double u1 = (double)((mix64(key + c1 * 0x9E3779B97F4A7C15ULL) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(mix64(key + c2 * 0x9E3779B97F4A7C15ULL) >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double t = 2.0 * 3.141592653589793 * u2;
    float* o = out + (uint64_t)s * sum_dims + __ldg(&feats[f].coff) + 2 * p;
    o[0] = (float)(1e-3 * (r * cos(t)));
    if (2 * p + 1 < D) o[1] = (float)(1e-3 * (r * sin(t)));
  }
}

}  // namespace

void launch_gen_upstream(uint64_t seed, uint64_t step, uint32_t rank, uint32_t B, uint32_t F, const FeatDev* feats,
                         uint32_t sum_dims, uint32_t max_dim, float* out, cudaStream_t st) {
  const uint32_t pairs = (max_dim + 1) / 2;
  const uint64_t n = (uint64_t)B * F * pairs;
  if (!n) return;
  k_gen_upstream<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 32), 256, 0, st>>>(seed, step, rank, B, F, feats,
                                                                                          sum_dims, pairs, out);
  S2D_LAUNCH_CHECK();
}

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
