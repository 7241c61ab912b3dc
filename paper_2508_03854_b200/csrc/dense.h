// Dense half of the model on the device (src/model.cpp, include/sparse2d/
// model.hpp): the per-rank one-hidden-layer ReLU MLPs of the toy DLRM
// (dense_arch: dense_dim -> dense_hidden -> D, over_arch: F*D + D ->
// over_hidden -> 1), their forward / backward_dx / accumulate_grads /
// apply_sgd, the dense DP step (dense_sync_and_apply, trainer.cpp:507-545),
// and the DataGenerator's dense features and labels (data.cpp:37-68,
// 137-145).  Every f64 expression is evaluated in the reference's order
// (dot_f64's four strided accumulators, model.cpp:10-23; left folds over
// (rank, sample) for the gradients) with -fmad=false, so the MLP state is
// bitwise the reference's wherever CUDA's exp / log / sin / cos round like
// the host libm (sigmoid, the loss, Box-Muller).
#pragma once

#include "comm.h"
#include "common.h"

namespace s2d {

// One Mlp's parameters (model.hpp:33-62): f32 w1 [hidden][in], b1 [hidden],
// w2 [out][hidden], b2 [out] and the f64 mirrors of w1 / w2 (sync_mirror).
struct MlpView {
  uint32_t in, hidden, out;
  float *w1, *b1, *w2, *b2;
  double *w1d, *w2d;
};

// Inputs of an Mlp, column j of sample s: j < n0 ? x0[s*n0 + j] :
// x1[s*n1 + j - n0] (the over arch reads [pooled | dense_arch output]).
struct MlpInput {
  const float* x0;
  uint32_t n0;
  const float* x1;
  uint32_t n1;
};

// Left fold over (rank, sample) of one layer's gradient followed by its SGD
// step in place (accumulate_grads, model.cpp:136-167; apply_sgd 169-186):
// g[p][q] = sum_{r, s} d_r[s][p] * f64(x_r[s][q]), g_b[p] = sum d_r[s][p]
// (terms with d == 0 skipped when skip_zero: the hidden layer), then
// w = f32(f64(w) - f * g) and the f64 mirror.
struct FoldArgs {
  uint32_t T, B, P, Q;
  const double* const* d;  // [T] -> [B][P]
  int skip_zero;
  const float* const* x0;  // [T] -> [B][n0]
  uint32_t n0;
  const float* const* x1;  // [T] -> [B][n1] (may be null when n1 == 0)
  uint32_t n1;
  float* w;
  double* wd;
  float* b;
  double f;  // lr * scale
};

void launch_mlp_hidden(const MlpView& m, const MlpInput& x, uint32_t B, float* hid, cudaStream_t st);
void launch_mlp_out(const MlpView& m, const float* hid, uint32_t B, float* out, double* prob, cudaStream_t st);
void launch_over_backward(const MlpView& m, const float* hid, const double* prob, const float* labels, uint32_t B,
                          double* dlogit, double* dh, double* loss, cudaStream_t st);
void launch_mlp_dx(const MlpView& m, const double* dh, uint32_t B, uint32_t n0, float* up, double* dtail,
                   cudaStream_t st);
void launch_mlp_dhidden(const MlpView& m, const float* hid, const double* dout, uint32_t B, double* dh,
                        cudaStream_t st);
void launch_loss_sum(const double* loss, uint32_t B, double* out, cudaStream_t st);
void launch_fold_sgd(const FoldArgs& a, cudaStream_t st);
// DataGenerator side (data.cpp): ground-truth id contributions and dense
// weights, the per-sample dense features and labels.
void launch_gt_normals(uint64_t key, uint64_t n, double scale, float* out, cudaStream_t st);
void launch_gen_dense(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t dd, float* out,
                      cudaStream_t st);
void launch_gen_labels(uint64_t seed, uint64_t lane, uint64_t step, uint32_t rank, uint32_t B, uint32_t F, uint32_t L,
                       const uint32_t* ids, const float* id_contrib, uint32_t rows, const float* dense,
                       const float* dense_w, uint32_t dd, double bias, float* labels, cudaStream_t st);
// One shard of the consensus replica as pool_ids sees it (ShardRef,
// embedding.hpp): rows [lo, hi) of a table, row r at w + (r - lo) * dim
// (fp32, or bf16 storage widened exactly).
struct EvalShard {
  uint32_t lo, hi;
  const void* w;
};
// pool_ids (embedding.cpp:39-92) of S samples x F fixed-length bags of L ids
// over shards[f * N + o] (o ascending, empty shards skipped): per-shard f64
// partial -> f32, f64 sum over shards -> f32, into out [S][F * D].
void launch_eval_pool(uint32_t S, uint32_t F, uint32_t L, uint32_t N, const uint32_t* ids, const EvalShard* shards,
                      uint32_t D, int bf16, float* out, cudaStream_t st);
// make_key({fields...}) of rng.hpp on the host
uint64_t rng_make_key(const uint64_t* fields, int n);

}  // namespace s2d
