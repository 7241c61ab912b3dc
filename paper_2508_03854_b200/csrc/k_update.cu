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

namespace {

// apply_row_update (src/embedding.cpp:108-129) over a batch of rows: one warp
// per distinct row walks that row's updates in call order (order[] is the
// stable row sort of the call), so a row listed twice gets both updates in
// sequence, each rounded to storage, as two reference calls would.
template <typename W>
__global__ void __launch_bounds__(256) k_apply_rows(W* __restrict__ w, float* __restrict__ v,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ seg,
                                                    const uint32_t* __restrict__ seg_row,
                                                    const double* __restrict__ delta,
                                                    const double* __restrict__ moment, uint32_t nseg,
                                                    uint32_t dim, uint8_t* __restrict__ dirty) {
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); s < nseg; s += warps) {
    const uint32_t b = seg[s], e = seg[s + 1];
    W* row = w + (uint64_t)seg_row[s] * dim;
    for (uint32_t c = lane; c < dim; c += 32) {
      W x = row[c];
      for (uint32_t k = b; k < e; ++k) {
        const double y = (double)(float)x + delta[(uint64_t)order[k] * dim + c];
        if constexpr (sizeof(W) == 4)
          x = (W)(float)y;
        else
          x = __double2bfloat16(y);
      }
      row[c] = x;
    }
    if (lane == 0) {
      v[seg_row[s]] = (float)moment[order[e - 1]];
      if (dirty) dirty[seg_row[s]] = 1;
    }
  }
}

}  // namespace

void launch_apply_rows(void* w, bool bf16, float* v, const uint32_t* order, const uint32_t* seg,
                       const uint32_t* seg_row, const double* delta, const double* moment, uint32_t nseg,
                       uint32_t dim, uint8_t* dirty, cudaStream_t st) {
  if (!nseg) return;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nseg + 7) / 8, 148ull * 8));
  if (bf16)
    k_apply_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(w), v, order, seg, seg_row,
                                                      delta, moment, nseg, dim, dirty);
  else
    k_apply_rows<float><<<grid, 256, 0, st>>>(static_cast<float*>(w), v, order, seg, seg_row, delta, moment,
                                              nseg, dim, dirty);
  S2D_LAUNCH_CHECK();
}

namespace {
template <typename W>
__global__ void __launch_bounds__(256) k_gather_rows(const W* __restrict__ w, const float* __restrict__ v,
                                                     const uint32_t* __restrict__ rows, uint32_t n, uint32_t dim,
                                                     float* __restrict__ w_out, float* __restrict__ v_out) {
  const uint32_t lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += warps) {
    const uint64_t r = rows[i];
    for (uint32_t c = lane; c < dim; c += 32) w_out[(uint64_t)i * dim + c] = (float)w[r * dim + c];
    if (lane == 0) v_out[i] = v[r];
  }
}
}  // namespace

void launch_gather_rows(const void* w, int bf16, const float* v, const uint32_t* rows_local, uint32_t n, uint32_t dim,
                        float* w_out, float* v_out, cudaStream_t st) {
  if (!n) return;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, 148ull * 8));
  if (bf16)
    k_gather_rows<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w), v, rows_local, n, dim,
                                                       w_out, v_out);
  else
    k_gather_rows<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w), v, rows_local, n, dim, w_out, v_out);
  S2D_LAUNCH_CHECK();
}

}  // namespace s2d
