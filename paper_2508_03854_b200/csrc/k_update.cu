// Backward-side kernels after the radix sort:
//   segments        run-length segmentation of the sorted slots: unique rows
//                   (U) and their contribution ranges
//   long_segments   rows with > kChunk contributions are split into fixed
//                   chunks (hot Zipf rows; SURVEY.md 7 "Hard parts")
//   chunk_partials  f64 in-order sum of each chunk
//   update          K3+K4 fused: f64 in-order segment sum x 1/(N*B)
//                   (aggregate_group_gradient, src/optimizer.cpp:25-59), then
//                   moment-scaled row-wise AdaGrad (adagrad_row_step,
//                   src/optimizer.cpp:65-83) or SGD (85-90), reading and
//                   writing each row and its accumulator once.
//
// Numerics: a segment of <= kChunk contributions is summed strictly in
// arrival order (bit-exact vs the reference).  A longer segment is summed
// per chunk in order and the chunk sums are added in order -- deterministic
// and launch-configuration independent, equal to the reference up to f64
// reassociation (<= 1e-15 relative on g).  |g|^2 is a per-lane in-order sum
// followed by a fixed xor-shuffle tree.
#include "device.cuh"

namespace s2d {
namespace {

__global__ void k_seg_write(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ head_off,
                            uint64_t n, uint32_t n_slots, uint32_t* __restrict__ uslot,
                            uint32_t* __restrict__ useg, uint32_t* __restrict__ counters) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    if (k >= n_slots) continue;
    const bool head = (i == 0) || keys[i - 1] != k;
    if (head) {
      const uint32_t u = head_off[i];
      uslot[u] = k;
      useg[u] = (uint32_t)i;
    }
    if (i + 1 == n || keys[i + 1] >= n_slots) {  // last valid key
      const uint32_t U = head_off[n];
      useg[U] = (uint32_t)(i + 1);
      counters[0] = U;
    }
  }
}

__global__ void k_long_segments(const uint32_t* __restrict__ useg, uint32_t* __restrict__ counters,
                                uint32_t* __restrict__ chunk_first, uint32_t* __restrict__ chunk_seg) {
  const uint32_t U = counters[0];
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const uint32_t len = useg[u + 1] - useg[u];
    if (len <= kChunk) continue;
    const uint32_t nch = (len + kChunk - 1) / kChunk;
    const uint32_t base = atomicAdd(&counters[1], nch);
    atomicAdd(&counters[2], 1u);
    chunk_first[u] = base;
    for (uint32_t k = 0; k < nch; ++k) chunk_seg[base + k] = u;
  }
}

// Sum of gradient rows vals[beg..end) in order into acc (lane columns).
template <int VPL>
__device__ __forceinline__ void sum_rows_in_order(const uint32_t* __restrict__ vals, uint32_t beg,
                                                  uint32_t end, const float* __restrict__ grad,
                                                  uint32_t d4, double (&acc)[VPL][4]) {
  constexpr int UNROLL = VPL == 1 ? 8 : (VPL == 2 ? 4 : 2);
  const uint32_t lane = lane_id();
  for (uint32_t c = beg; c < end; c += 32) {
    const uint32_t cnt = min(32u, end - c);
    const uint32_t my = lane < cnt ? __ldg(vals + c + lane) : 0u;
    for (uint32_t t = 0; t < cnt; t += UNROLL) {
      float4 raw[UNROLL][VPL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint32_t val = __shfl_sync(0xffffffffu, my, min(t + u, 31u));
        if (t + u < cnt) {
          const float* row = grad + (uint64_t)val * 4;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const uint32_t c4 = lane + v * 32;
            if (c4 < d4) raw[u][v] = __ldg(reinterpret_cast<const float4*>(row) + c4);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (t + u < cnt) {
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if (lane + v * 32 < d4) {
              acc[v][0] += (double)raw[u][v].x;
              acc[v][1] += (double)raw[u][v].y;
              acc[v][2] += (double)raw[u][v].z;
              acc[v][3] += (double)raw[u][v].w;
            }
          }
        }
      }
    }
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) k_chunk_partials(UpdateArgs a, uint32_t max_d4) {
  const uint32_t lane = lane_id();
  const uint32_t nchunks = a.counters[1];
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); q < nchunks; q += warps) {
    const uint32_t u = __ldg(a.chunk_seg + q);
    const uint32_t k = q - __ldg(a.chunk_base + u);
    const uint32_t s0 = __ldg(a.useg + u), s1 = __ldg(a.useg + u + 1);
    const uint32_t beg = s0 + k * kChunk, end = min(s1, beg + kChunk);
    const uint32_t slot = __ldg(a.uslot + u);
    const uint32_t f = feature_of_slot(a.vbase_sorted, a.feat_of_vbase, a.n_feat_owned, slot);
    const uint32_t d4 = __ldg(&a.feats[f].dim) >> 2;
    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    sum_rows_in_order<VPL>(a.vals, beg, end, a.grad, d4, acc);
    double* out = a.chunk_part + (uint64_t)q * (max_d4 * 4);
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const uint32_t c4 = lane + v * 32;
      if (c4 < d4) {
        double2* o2 = reinterpret_cast<double2*>(out + c4 * 4);
        o2[0] = make_double2(acc[v][0], acc[v][1]);
        o2[1] = make_double2(acc[v][2], acc[v][3]);
      }
    }
  }
}

// Row step on lane-owned columns.  Returns false (and writes nothing) for a
// nonfinite gradient, like the reference's throw before any write
// (optimizer.cpp:68-73).
template <typename WT, int VPL>
__device__ __forceinline__ bool row_step(WT* w, float* v_ptr, double (&g)[VPL][4], uint32_t d4,
                                         double eta, double eps, double c, int sgd, double* lr_out) {
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
    const float v_old = *v_ptr;
    const float v_new = (float)((double)v_old + ns);
    lr = eta / (sqrt((double)v_new / c) + eps);  // effective_lr (optimizer.cpp:61-63)
    __syncwarp();
    if (lane == 0) *v_ptr = v_new;
  }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const uint32_t c4 = lane + v * 32;
    if (c4 < d4) {
      double x[4];
      Vec4<WT>::load_rw(w + c4 * 4, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = x[j] - lr * g[v][j];
      Vec4<WT>::store(w + c4 * 4, x);
    }
  }
  if (lr_out && lane == 0) *lr_out = lr;
  return true;
}

template <typename WT, int VPL>
__global__ void __launch_bounds__(256) k_update(UpdateArgs a, uint32_t max_d4) {
  const uint32_t lane = lane_id();
  const uint32_t U = a.counters[0];
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  WT* W = reinterpret_cast<WT*>(a.weights);
  for (uint32_t u = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); u < U; u += warps) {
    const uint32_t slot = __ldg(a.uslot + u);
    const uint32_t s0 = __ldg(a.useg + u), s1 = __ldg(a.useg + u + 1);
    const uint32_t f = feature_of_slot(a.vbase_sorted, a.feat_of_vbase, a.n_feat_owned, slot);
    const uint32_t dim = __ldg(&a.feats[f].dim), d4 = dim >> 2;
    double acc[VPL][4];
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = 0.0;
    if (s1 - s0 <= kChunk) {
      sum_rows_in_order<VPL>(a.vals, s0, s1, a.grad, d4, acc);
    } else {
      const uint32_t first = __ldg(a.chunk_base + u);
      const uint32_t nch = (s1 - s0 + kChunk - 1) / kChunk;
      for (uint32_t k = 0; k < nch; ++k) {
        const double* p = a.chunk_part + (uint64_t)(first + k) * (max_d4 * 4);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const uint32_t c4 = lane + v * 32;
          if (c4 < d4) {
            const double2 x0 = __ldg(reinterpret_cast<const double2*>(p + c4 * 4));
            const double2 x1 = __ldg(reinterpret_cast<const double2*>(p + c4 * 4) + 1);
            acc[v][0] += x0.x;
            acc[v][1] += x0.y;
            acc[v][2] += x1.x;
            acc[v][3] += x1.y;
          }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[v][j] = acc[v][j] * a.inv_batch;
    const uint32_t local = slot - __ldg(&a.feats[f].vbase);
    WT* w = W + __ldg(&a.feats[f].wbase) + (uint64_t)local * dim;
    const bool ok = row_step<WT, VPL>(w, a.moments + slot, acc, d4, a.eta, a.eps, a.c, a.sgd, nullptr);
    if (lane == 0) {
      if (!ok)
        atomicOr(a.err, kErrNonfinite);
      else if (a.dirty)
        a.dirty[slot] = 1;
    }
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) k_rows_adagrad(float* w, float* vv, const double* g, double* lr,
                                                      uint32_t n, uint32_t dim, double eta, double eps,
                                                      double c, int sgd, uint32_t* err) {
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
    const bool ok = row_step<float, VPL>(w + (uint64_t)r * dim, vv + r, gr, d4, eta, eps, c, sgd,
                                         lr ? lr + r : nullptr);
    if (!ok && lane == 0) atomicOr(err, kErrNonfinite);
  }
}

unsigned persistent_grid(uint64_t rows_upper) {
  const uint64_t want = (rows_upper + 7) / 8;
  const uint64_t cap = 148ull * 8;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, cap));
}

}  // namespace

void run_segments(const SegmentArgs& a, cudaStream_t st) {
  S2D_CUDA(cudaMemsetAsync(a.counters, 0, 4 * sizeof(uint32_t), st));
  if (a.n == 0) return;
  // head_off reuses chunk_base as scratch ([n+1] u32)
  uint32_t* head_off = a.chunk_base;
  scan_heads_u32(a.keys, head_off, a.n, a.n_slots, st, a.tmp, a.tmp_bytes);
  const unsigned g = (unsigned)std::min<uint64_t>((a.n + 255) / 256, 148ull * 16);
  k_seg_write<<<g, 256, 0, st>>>(a.keys, head_off, a.n, a.n_slots, a.uslot, a.useg, a.counters);
  S2D_LAUNCH_CHECK();
  k_long_segments<<<g, 256, 0, st>>>(a.useg, a.counters, a.chunk_base, a.chunk_seg);
  S2D_LAUNCH_CHECK();
}

void launch_update(const UpdateArgs& a, int bf16, int max_dim, uint64_t max_rows, cudaStream_t st) {
  if (max_rows == 0) return;
  const uint32_t max_d4 = (uint32_t)max_dim / 4;
  const unsigned grid = persistent_grid(max_rows);
  const unsigned cgrid = persistent_grid(max_rows / kChunk + 1);
#define S2D_UPD(VPL)                                                                             \
  do {                                                                                           \
    k_chunk_partials<VPL><<<cgrid, 256, 0, st>>>(a, max_d4);                                     \
    S2D_LAUNCH_CHECK();                                                                          \
    if (bf16)                                                                                    \
      k_update<__nv_bfloat16, VPL><<<grid, 256, 0, st>>>(a, max_d4);                             \
    else                                                                                         \
      k_update<float, VPL><<<grid, 256, 0, st>>>(a, max_d4);                                     \
    S2D_LAUNCH_CHECK();                                                                          \
  } while (0)
  if (max_d4 <= 32)
    S2D_UPD(1);
  else if (max_d4 <= 64)
    S2D_UPD(2);
  else
    S2D_UPD(4);
#undef S2D_UPD
}

void launch_rows_adagrad(float* w, float* v, const double* g, double* lr, uint32_t n, uint32_t dim,
                         double eta, double eps, double c, int sgd, uint32_t* err, cudaStream_t st) {
  if (!n) return;
  const unsigned grid = persistent_grid(n);
  if (dim / 4 <= 32)
    k_rows_adagrad<1><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  else if (dim / 4 <= 64)
    k_rows_adagrad<2><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  else
    k_rows_adagrad<4><<<grid, 256, 0, st>>>(w, v, g, lr, n, dim, eta, eps, c, sgd, err);
  S2D_LAUNCH_CHECK();
}

}  // namespace s2d
