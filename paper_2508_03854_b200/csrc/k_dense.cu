// Kernels of the dense half of the model (dense.h): the toy DLRM MLPs'
// forward / backward (src/model.cpp:90-133, trainer.cpp:366-438), the dense
// DP gradient fold + SGD step (model.cpp:136-186, trainer.cpp:507-545) and
// the DataGenerator's dense features, ground truth and labels
// (data.cpp:37-68, 137-145).  Thread per output element; every f64
// expression keeps the reference's evaluation order (compiled with
// -fmad=false: no contraction, like -ffp-contract=off).  None of this is on
// the embedding step's hot path: the sizes are the toy model's (hidden
// widths of tens), so the kernels are simple and latency-bound.
#include "dense.h"
#include "device.cuh"

namespace s2d {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint64_t key_of(const uint64_t* fields, int n) {
  uint64_t h = 0x8A5CD789635D2DFFULL;
  for (int q = 0; q < n; ++q) h = mix64(h + kGamma + fields[q]);
  return h;
}

// CounterRng::next_uniform / next_uniform_pos of draw ctr (1-based)
__device__ __forceinline__ double uniform_at(uint64_t key, uint64_t ctr) {
  return (double)(mix64(key + ctr * kGamma) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double uniform_pos_at(uint64_t key, uint64_t ctr) {
  return (double)((mix64(key + ctr * kGamma) >> 11) + 1) * 0x1.0p-53;
}

// normal #i of CounterRng::next_normal's stream (pairs cached: even i the
// cos branch of draws 2p+1, 2p+2, odd i the sin branch)
__device__ __forceinline__ double normal_at(uint64_t key, uint64_t i) {
  const uint64_t p = i >> 1;
  const double u1 = uniform_pos_at(key, 2 * p + 1);
  const double u2 = uniform_at(key, 2 * p + 2);
  const double r = sqrt(-2.0 * log(u1));
  const double t = 2.0 * 3.141592653589793 * u2;
  return (i & 1) ? r * sin(t) : r * cos(t);
}

__device__ __forceinline__ double xin(const MlpInput& x, uint32_t s, uint32_t j) {
  return j < x.n0 ? (double)x.x0[(uint64_t)s * x.n0 + j] : (double)x.x1[(uint64_t)s * x.n1 + (j - x.n0)];
}

// Mlp::forward hidden layer (model.cpp:96-103): z = f64(b1[h]) +
// dot_f64(w1_d[h], f64(x)), dot_f64 = four strided accumulators, tail into
// a0, (a0 + a1) + (a2 + a3) (model.cpp:10-23); hidden = z > 0 ? f32(z) : 0.
__global__ void k_mlp_hidden(const MlpView m, const MlpInput x, uint32_t B, float* __restrict__ hid) {
  const uint64_t n = (uint64_t)B * m.hidden;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / m.hidden), h = (uint32_t)(i % m.hidden);
    const double* w = m.w1d + (uint64_t)h * m.in;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    uint32_t j = 0;
    for (; j + 4 <= m.in; j += 4) {
      a0 += w[j] * xin(x, s, j);
      a1 += w[j + 1] * xin(x, s, j + 1);
      a2 += w[j + 2] * xin(x, s, j + 2);
      a3 += w[j + 3] * xin(x, s, j + 3);
    }
    for (; j < m.in; ++j) a0 += w[j] * xin(x, s, j);
    const double z = (double)m.b1[h] + ((a0 + a1) + (a2 + a3));
    hid[i] = z > 0.0 ? (float)z : 0.0f;
  }
}

// Mlp::forward output layer (model.cpp:104-110): out = f32(f64(b2[o]) +
// dot_f64(w2_d[o], f64(hidden))); prob (the over arch's single logit) =
// sigmoid(f64(logit)) = 1 / (1 + exp(-x)) (model.cpp:25, trainer.cpp:401).
__global__ void k_mlp_out(const MlpView m, const float* __restrict__ hid, uint32_t B, float* __restrict__ out,
                          double* __restrict__ prob) {
  const uint64_t n = (uint64_t)B * m.out;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / m.out), o = (uint32_t)(i % m.out);
    const double* w = m.w2d + (uint64_t)o * m.hidden;
    const float* x = hid + (uint64_t)s * m.hidden;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    uint32_t j = 0;
    for (; j + 4 <= m.hidden; j += 4) {
      a0 += w[j] * (double)x[j];
      a1 += w[j + 1] * (double)x[j + 1];
      a2 += w[j + 2] * (double)x[j + 2];
      a3 += w[j + 3] * (double)x[j + 3];
    }
    for (; j < m.hidden; ++j) a0 += w[j] * (double)x[j];
    const float z = (float)((double)m.b2[o] + ((a0 + a1) + (a2 + a3)));
    out[i] = z;
    if (prob) prob[i] = 1.0 / (1.0 + exp(-(double)z));
  }
}

// backward_rank's head (trainer.cpp:409-423) and over_arch.backward_dx's
// hidden gradient (model.cpp:115-126) for the single-logit over arch:
// loss = y > 0.5 ? -log(p) : -log(1 - p), dlogit = p - y,
// dh[h] = (0.0 + dlogit * w2_d[0][h]), zeroed where hidden <= 0.
__global__ void k_over_backward(const MlpView m, const float* __restrict__ hid, const double* __restrict__ prob,
                                const float* __restrict__ labels, uint32_t B, double* __restrict__ dlogit,
                                double* __restrict__ dh, double* __restrict__ loss) {
  const uint64_t n = (uint64_t)B * m.hidden;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / m.hidden), h = (uint32_t)(i % m.hidden);
    const double p = prob[s], y = (double)labels[s];
    const double d = p - y;
    double g = 0.0;
    g += d * m.w2d[h];
    dh[i] = hid[i] <= 0.0f ? 0.0 : g;
    if (h == 0) {
      dlogit[s] = d;
      loss[s] = y > 0.5 ? -log(p) : -log(1.0 - p);
    }
  }
}

// backward_dx's input gradient (model.cpp:127-135): dx[j] = sum over h
// ascending (d == 0 skipped) of dh[h] * w1_d[h][j]; columns j < n0 leave as
// the f32 wire gradient (trainer.cpp:424-427), the rest as f64 (the dense
// arch's upstream, trainer.cpp:428-431).
__global__ void k_mlp_dx(const MlpView m, const double* __restrict__ dh, uint32_t B, uint32_t n0,
                         float* __restrict__ up, double* __restrict__ dtail) {
  const uint64_t n = (uint64_t)B * m.in;
  const uint32_t n1 = m.in - n0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / m.in), j = (uint32_t)(i % m.in);
    const double* d = dh + (uint64_t)s * m.hidden;
    double acc = 0.0;
    for (uint32_t h = 0; h < m.hidden; ++h) {
      const double dv = d[h];
      if (dv == 0.0) continue;
      acc += dv * m.w1d[(uint64_t)h * m.in + j];
    }
    if (j < n0)
      up[(uint64_t)s * n0 + j] = (float)acc;
    else
      dtail[(uint64_t)s * n1 + (j - n0)] = acc;
  }
}

// backward_dx's hidden gradient for a multi-output layer (the dense arch,
// model.cpp:115-126): dh[h] = sum over o ascending of dout[o] * w2_d[o][h]
// from 0.0, zeroed where hidden <= 0.
__global__ void k_mlp_dhidden(const MlpView m, const float* __restrict__ hid, const double* __restrict__ dout,
                              uint32_t B, double* __restrict__ dh) {
  const uint64_t n = (uint64_t)B * m.hidden;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / m.hidden), h = (uint32_t)(i % m.hidden);
    const double* d = dout + (uint64_t)s * m.out;
    double acc = 0.0;
    for (uint32_t o = 0; o < m.out; ++o) acc += d[o] * m.w2d[(uint64_t)o * m.hidden + h];
    dh[i] = hid[i] <= 0.0f ? 0.0 : acc;
  }
}

// loss_sum (trainer.cpp:410-420): sequential over samples; out[1] = first
// sample with a nonfinite loss (as a double, -1 when none).
__global__ void k_loss_sum(const double* __restrict__ loss, uint32_t B, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double acc = 0.0, bad = -1.0;
  for (uint32_t s = 0; s < B; ++s) {
    const double l = loss[s];
    if (!isfinite(l)) {
      bad = (double)s;
      break;
    }
    acc += l;
  }
  out[0] = acc;
  out[1] = bad;
}

__global__ void k_fold_sgd(const FoldArgs a) {
  const uint64_t nw = (uint64_t)a.P * a.Q, n = nw + a.P;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double g = 0.0;
    if (i < nw) {
      const uint32_t p = (uint32_t)(i / a.Q), q = (uint32_t)(i % a.Q);
      for (uint32_t r = 0; r < a.T; ++r) {
        const double* d = a.d[r];
        const float* x = q < a.n0 ? a.x0[r] + q : a.x1[r] + (q - a.n0);
        const uint32_t xs = q < a.n0 ? a.n0 : a.n1;
        for (uint32_t s = 0; s < a.B; ++s) {
          const double dv = d[(uint64_t)s * a.P + p];
          if (a.skip_zero && dv == 0.0) continue;
          g += dv * (double)x[(uint64_t)s * xs];
        }
      }
      const float w = (float)((double)a.w[i] - a.f * g);
      a.w[i] = w;
      if (a.wd) a.wd[i] = (double)w;
    } else {
      const uint32_t p = (uint32_t)(i - nw);
      for (uint32_t r = 0; r < a.T; ++r) {
        const double* d = a.d[r];
        for (uint32_t s = 0; s < a.B; ++s) {
          const double dv = d[(uint64_t)s * a.P + p];
          if (a.skip_zero && dv == 0.0) continue;
          g += dv;
        }
      }
      a.b[p] = (float)((double)a.b[p] - a.f * g);
    }
  }
}

// out[i] = f32(scale * normal #i) of the stream `key` (GroundTruthModel:
// id contributions with key make_key({seed, 10, f}), dense weights with
// make_key({seed, 11}); data.cpp:43-55)
__global__ void k_gt_normals(uint64_t key, uint64_t n, double scale, float* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (float)(scale * normal_at(key, i));
}

// Sample::dense (data.cpp:137-141): f32 normals of CounterRng({seed, lane 0,
// step, rank, s, kTagDense = 2}).
__global__ void k_gen_dense(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t dd,
                            float* __restrict__ out) {
  const uint64_t n = (uint64_t)B * dd;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / dd), j = (uint32_t)(i % dd);
    const uint64_t f[6] = {seed, lane, step, rank, s, 2ull};
    out[i] = (float)normal_at(key_of(f, 6), j);
  }
}

// Sample::label (data.cpp:142-144): p = sigmoid(GroundTruthModel::logit)
// with logit = bias, + f64(dense_w[j]) * f64(dense[j]) for j ascending, +
// f64(id_contrib[f][id]) for (f, id) in order (data.cpp:57-68); label =
// (first uniform of CounterRng({seed, 0, step, rank, s, kTagLabel = 3})) < p.
__global__ void k_gen_labels(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t F, uint32_t L,
                             const uint32_t* __restrict__ ids, const float* __restrict__ id_contrib, uint32_t rows,
                             const float* __restrict__ dense, const float* __restrict__ dense_w, uint32_t dd,
                             double bias, float* __restrict__ labels) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < B; s += gridDim.x * blockDim.x) {
    double z = bias;
    for (uint32_t j = 0; j < dd; ++j) z += (double)dense_w[j] * (double)dense[(uint64_t)s * dd + j];
    const uint32_t* id = ids + (uint64_t)s * F * L;
    for (uint32_t f = 0; f < F; ++f)
      for (uint32_t j = 0; j < L; ++j) z += (double)id_contrib[(uint64_t)f * rows + id[f * L + j]];
    const double p = 1.0 / (1.0 + exp(-z));
    const uint64_t k[6] = {seed, lane, step, rank, s, 3ull};
    labels[s] = uniform_at(key_of(k, 6), 1) < p ? 1.0f : 0.0f;
  }
}

template <typename WT>
__global__ void k_eval_pool(uint32_t S, uint32_t F, uint32_t L, uint32_t N, const uint32_t* __restrict__ ids,
                            const EvalShard* __restrict__ shards, uint32_t D, float* __restrict__ out) {
  const uint64_t n = (uint64_t)S * F * D;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)(i % D);
    const uint64_t bag = i / D;
    const uint32_t f = (uint32_t)(bag % F);
    const uint32_t* id = ids + bag * L;
    double pool = 0.0;
    for (uint32_t o = 0; o < N; ++o) {
      const EvalShard sh = shards[(uint64_t)f * N + o];
      if (sh.hi <= sh.lo) continue;
      const WT* w = reinterpret_cast<const WT*>(sh.w);
      double partial = 0.0;
      bool hit = false;
      for (uint32_t q = 0; q < L; ++q) {
        const uint32_t r = id[q];
        if (r < sh.lo || r >= sh.hi) continue;
        hit = true;
        partial += (double)(float)w[(uint64_t)(r - sh.lo) * D + j];
      }
      if (hit) pool += (double)(float)partial;
    }
    out[i] = (float)pool;
  }
}

unsigned grid_for(uint64_t n) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

uint64_t rng_make_key(const uint64_t* fields, int n) {
  uint64_t h = 0x8A5CD789635D2DFFULL;
  for (int q = 0; q < n; ++q) h = mix64(h + kGamma + fields[q]);
  return h;
}

void launch_mlp_hidden(const MlpView& m, const MlpInput& x, uint32_t B, float* hid, cudaStream_t st) {
  const uint64_t n = (uint64_t)B * m.hidden;
  if (!n) return;
  k_mlp_hidden<<<grid_for(n), 256, 0, st>>>(m, x, B, hid);
  S2D_LAUNCH_CHECK();
}

void launch_mlp_out(const MlpView& m, const float* hid, uint32_t B, float* out, double* prob, cudaStream_t st) {
  const uint64_t n = (uint64_t)B * m.out;
  if (!n) return;
  k_mlp_out<<<grid_for(n), 256, 0, st>>>(m, hid, B, out, prob);
  S2D_LAUNCH_CHECK();
}

void launch_over_backward(const MlpView& m, const float* hid, const double* prob, const float* labels, uint32_t B,
                          double* dlogit, double* dh, double* loss, cudaStream_t st) {
  const uint64_t n = (uint64_t)B * m.hidden;
  if (!n) return;
  k_over_backward<<<grid_for(n), 256, 0, st>>>(m, hid, prob, labels, B, dlogit, dh, loss);
  S2D_LAUNCH_CHECK();
}

void launch_mlp_dx(const MlpView& m, const double* dh, uint32_t B, uint32_t n0, float* up, double* dtail,
                   cudaStream_t st) {
  const uint64_t n = (uint64_t)B * m.in;
  if (!n) return;
  k_mlp_dx<<<grid_for(n), 256, 0, st>>>(m, dh, B, n0, up, dtail);
  S2D_LAUNCH_CHECK();
}

void launch_mlp_dhidden(const MlpView& m, const float* hid, const double* dout, uint32_t B, double* dh,
                        cudaStream_t st) {
  const uint64_t n = (uint64_t)B * m.hidden;
  if (!n) return;
  k_mlp_dhidden<<<grid_for(n), 256, 0, st>>>(m, hid, dout, B, dh);
  S2D_LAUNCH_CHECK();
}

void launch_loss_sum(const double* loss, uint32_t B, double* out, cudaStream_t st) {
  k_loss_sum<<<1, 32, 0, st>>>(loss, B, out);
  S2D_LAUNCH_CHECK();
}

void launch_fold_sgd(const FoldArgs& a, cudaStream_t st) {
  const uint64_t n = (uint64_t)a.P * a.Q + a.P;
  if (!n) return;
  k_fold_sgd<<<grid_for(n), 256, 0, st>>>(a);
  S2D_LAUNCH_CHECK();
}

void launch_eval_pool(uint32_t S, uint32_t F, uint32_t L, uint32_t N, const uint32_t* ids, const EvalShard* shards,
                      uint32_t D, int bf16, float* out, cudaStream_t st) {
  const uint64_t n = (uint64_t)S * F * D;
  if (!n) return;
  if (bf16)
    k_eval_pool<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(S, F, L, N, ids, shards, D, out);
  else
    k_eval_pool<float><<<grid_for(n), 256, 0, st>>>(S, F, L, N, ids, shards, D, out);
  S2D_LAUNCH_CHECK();
}

void launch_gt_normals(uint64_t key, uint64_t n, double scale, float* out, cudaStream_t st) {
  if (!n) return;
  k_gt_normals<<<grid_for(n), 256, 0, st>>>(key, n, scale, out);
  S2D_LAUNCH_CHECK();
}

void launch_gen_dense(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t dd, float* out,
                      cudaStream_t st) {
  const uint64_t n = (uint64_t)B * dd;
  if (!n) return;
  k_gen_dense<<<grid_for(n), 256, 0, st>>>(seed, lane, step, rank, B, dd, out);
  S2D_LAUNCH_CHECK();
}

void launch_gen_labels(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t F, uint32_t L,
                       const uint32_t* ids, const float* id_contrib, uint32_t rows, const float* dense,
                       const float* dense_w, uint32_t dd, double bias, float* labels, cudaStream_t st) {
  if (!B) return;
  k_gen_labels<<<grid_for(B), 256, 0, st>>>(seed, lane, step, rank, B, F, L, ids, id_contrib, rows, dense, dense_w, dd,
                                             bias, labels);
  S2D_LAUNCH_CHECK();
}

}  // namespace s2d
