// Standalone fused row step on caller-provided rows: the device code behind
// s2d_adagrad_rows / Python adagrad_row_step (bindings/module.cpp:93-107).
// The same arithmetic as the step's flush in k_stream.cu: moment-scaled
// row-wise AdaGrad (src/optimizer.cpp:65-83) or SGD (85-90), f64 math,
// |g|^2 as a per-lane in-order sum followed by a fixed xor-shuffle tree.
#include "device.cuh"

namespace s2d {
namespace {

// Returns false (and writes nothing) for a nonfinite gradient, like the
// reference's throw before any write (optimizer.cpp:68-73).
template <int VPL>
__device__ __forceinline__ bool row_step(float* w, float* v_ptr, double (&g)[VPL][4], uint32_t d4, double eta,
                                         double eps, double c, int sgd, double* lr_out) {
  const uint32_t lane = lane_id();
  bool finite = true;
#pragma unroll
  for (int v = 0; v < VPL; ++v)
    if (lane + v * 32 < d4)
#pragma unroll
      for (int j = 0; j < 4; ++j) finite &= isfinite(g[v][j]);
  if (!__all_sync(0xffffffffu, finite)) return false;
  double lr = eta;
  if (!sgd) {
    double ns = 0.0;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      if (lane + v * 32 < d4)
#pragma unroll
        for (int j = 0; j < 4; ++j) ns += g[v][j] * g[v][j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
    const float v_new = (float)((double)*v_ptr + ns);
    lr = eta / (sqrt((double)v_new / c) + eps);  // effective_lr (optimizer.cpp:61-63)
    __syncwarp();
    if (lane == 0) *v_ptr = v_new;
  }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const uint32_t c4 = lane + v * 32;
    if (c4 < d4) {
      double x[4];
      Vec4<float>::load_rw(w + c4 * 4, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = x[j] - lr * g[v][j];
      Vec4<float>::store(w + c4 * 4, x);
    }
  }
  if (lr_out && lane == 0) *lr_out = lr;
  return true;
}

template <int VPL>
__global__ void __launch_bounds__(256) k_rows_adagrad(float* w, float* vv, const double* g, double* lr, uint32_t n,
                                                      uint32_t dim, double eta, double eps, double c, int sgd,
                                                      uint32_t* err) {
  const uint32_t lane = lane_id();
  const uint32_t d4 = dim >> 2;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < n; r += warps) {
    double gr[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const uint32_t c4 = lane + v * 32;
#pragma unroll
      for (int j = 0; j < 4; ++j) gr[v][j] = c4 < d4 ? g[(uint64_t)r * dim + c4 * 4 + j] : 0.0;
    }
    const bool ok = row_step<VPL>(w + (uint64_t)r * dim, vv + r, gr, d4, eta, eps, c, sgd, lr ? lr + r : nullptr);
    if (!ok && lane == 0) atomicOr(err, kErrNonfinite);
  }
}

}  // namespace

void launch_rows_adagrad(float* w, float* v, const double* g, double* lr, uint32_t n, uint32_t dim, double eta,
                         double eps, double c, int sgd, uint32_t* err, cudaStream_t st) {
  if (!n) return;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, 148ull * 8));
  if (dim / 4 <= 32)
    k_rows_adagrad<1><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  else if (dim / 4 <= 64)
    k_rows_adagrad<2><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  else
    k_rows_adagrad<4><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  S2D_LAUNCH_CHECK();
}

}  // namespace s2d
