// Host side of the device-side synthetic input (DataGenerator,
// src/data.cpp:70-136): validates the feature specs like
// FeatureSpec::validate (data.cpp:26-35), builds each table's Zipf CDF
// exactly as the DataGenerator constructor does (sequential f64 sum of
// pow(k+1, -s) with the same libm, divided by the total, last entry 1.0;
// data.cpp:85-98), keeps the CDFs on the device while the exponents are
// unchanged, and launches k_gen_ids / k_gen_lengths (k_gen.cu).
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace s2d {

void Ctx::gen_batch(uint64_t seed, uint64_t step, uint32_t rnk, uint32_t batch, const double* zipf,
                    const uint32_t* ids_per_sample, uint32_t* lengths, uint32_t* ids, int mem, uint64_t lane) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (!zipf || !ids_per_sample) throw Error(S2D_EINVAL, "zipf and ids_per_sample are required");
  if (mem != S2D_HOST && mem != S2D_DEVICE) throw Error(S2D_EINVAL, "mem must be S2D_HOST or S2D_DEVICE");
  for (uint32_t f = 0; f < F; ++f) {
    if (tables[f].rows < 1)
      throw Error(S2D_EINVAL, "feature " + std::to_string(f) + ": num_ids must be >= 1");
    if (!(zipf[f] >= 0.0))
      throw Error(S2D_EINVAL, "feature " + std::to_string(f) + ": zipf_exponent must be >= 0");
  }
  S2D_CUDA(cudaSetDevice(device));
  // CDFs: rebuilt only when an exponent changes
  if (gen_zipf.size() != F || std::memcmp(gen_zipf.data(), zipf, F * sizeof(double)) != 0) {
    gen_cdf_off.assign(F + 1, 0);
    for (uint32_t f = 0; f < F; ++f) gen_cdf_off[f + 1] = gen_cdf_off[f] + tables[f].rows;
    gen_cdf.ensure(gen_cdf_off[F] * sizeof(double));
    std::vector<double> cdf;
    for (uint32_t f = 0; f < F; ++f) {
      const uint32_t n = tables[f].rows;
      cdf.resize(n);
      double total = 0.0;
      for (uint32_t k = 0; k < n; ++k) {
        total += std::pow(static_cast<double>(k + 1), -zipf[f]);
        cdf[k] = total;
      }
      for (auto& v : cdf) v /= total;
      cdf.back() = 1.0;
      S2D_CUDA(cudaMemcpy(gen_cdf.as<double>() + gen_cdf_off[f], cdf.data(), (size_t)n * sizeof(double),
                          cudaMemcpyHostToDevice));
    }
    gen_zipf.assign(zipf, zipf + F);
  }
  // per-table metadata: cum[F+1] | rows[F] | cdf_off[F] (u64, 8-aligned)
  std::vector<uint32_t> cum(F + 1, 0), rows(F);
  for (uint32_t f = 0; f < F; ++f) {
    cum[f + 1] = cum[f] + ids_per_sample[f];
    rows[f] = tables[f].rows;
  }
  const size_t meta_u32 = ((2 * (size_t)F + 1) + 1) & ~(size_t)1;
  gen_meta.ensure(meta_u32 * 4 + (size_t)F * 8);
  std::vector<char> meta(meta_u32 * 4 + (size_t)F * 8, 0);
  std::memcpy(meta.data(), cum.data(), (F + 1) * 4);
  std::memcpy(meta.data() + (F + 1) * 4, rows.data(), F * 4);
  std::memcpy(meta.data() + meta_u32 * 4, gen_cdf_off.data(), F * 8);
  S2D_CUDA(cudaMemcpyAsync(gen_meta.p, meta.data(), meta.size(), cudaMemcpyHostToDevice, stream));
  GenArgs a{};
  a.seed = seed;
  a.step = step;
  a.lane = lane;
  a.rank = rnk;
  a.B = batch;
  a.F = F;
  a.per_sample = cum[F];
  a.cum = gen_meta.as<uint32_t>();
  a.rows = gen_meta.as<uint32_t>() + F + 1;
  a.cdf_off = reinterpret_cast<const uint64_t*>(gen_meta.as<char>() + meta_u32 * 4);
  a.cdf = gen_cdf.as<double>();
  const uint64_t n_bags = (uint64_t)batch * F, n_ids = (uint64_t)batch * cum[F];
  if (mem == S2D_HOST) {
    gen_lengths.ensure(std::max<uint64_t>(n_bags, 1) * 4);
    gen_ids.ensure(std::max<uint64_t>(n_ids, 1) * 4);
    a.lengths = gen_lengths.as<uint32_t>();
    a.ids = gen_ids.as<uint32_t>();
  } else {
    a.lengths = lengths;
    a.ids = ids;
  }
  launch_gen_batch(a, stream);
  if (mem == S2D_HOST) {
    if (n_bags) S2D_CUDA(cudaMemcpyAsync(lengths, a.lengths, n_bags * 4, cudaMemcpyDeviceToHost, stream));
    if (n_ids) S2D_CUDA(cudaMemcpyAsync(ids, a.ids, n_ids * 4, cudaMemcpyDeviceToHost, stream));
  }
  // the host metadata vector dies here: wait for its copy (and host outputs)
  S2D_CUDA(cudaStreamSynchronize(stream));
}

// Synthetic upstream gradient for this rank's batch:
// out[s][coff_f + j] = f32(1e-3 * N(0,1)) from CounterRng({seed, step, rank,
// s, f}); mem says where out lives.
void Ctx::gen_upstream(uint64_t seed, uint64_t step, uint32_t rnk, uint32_t batch, float* out, int mem) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (mem != S2D_HOST && mem != S2D_DEVICE) throw Error(S2D_EINVAL, "mem must be S2D_HOST or S2D_DEVICE");
  S2D_CUDA(cudaSetDevice(device));
  const uint64_t n = (uint64_t)batch * sum_dims;
  float* d = out;
  if (mem == S2D_HOST) {
    upstream_stage.ensure(std::max<uint64_t>(n, 1) * 4);
    d = upstream_stage.as<float>();
  }
  launch_gen_upstream(seed, step, rnk, batch, F, d_feats.as<FeatDev>(), sum_dims, max_dim, d, stream);
  if (mem == S2D_HOST) {
    if (n) S2D_CUDA(cudaMemcpyAsync(out, d, n * 4, cudaMemcpyDeviceToHost, stream));
    S2D_CUDA(cudaStreamSynchronize(stream));
  }
}

}  // namespace s2d
