// MetricsRow moment statistics on the device (trainer.cpp:745-771):
// eff_lr_p50 / eff_lr_p99 -- percentiles of effective_lr(v) over every row
// of every table of the replica -- and v_mean.  effective_lr is
// non-increasing in v (optimizer.cpp:61-63), so the lr percentile at
// ascending index k is effective_lr of the moment at DESCENDING index k: a
// radix select over the moments' bit patterns (moments are >= 0 and
// finite, so their IEEE bits order like the values) finds it exactly, and
// the host applies the reference's effective_lr to the selected moment.
#include "device.cuh"

namespace s2d {
namespace {

// histogram of the 8-bit digit at `shift` of the moments whose higher bits
// equal `prefix` (under `mask`)
__global__ void __launch_bounds__(256) k_moment_hist(const float* __restrict__ v, uint32_t n, int shift,
                                                     uint32_t mask, uint32_t prefix, uint32_t* __restrict__ hist) {
  pdl_wait();
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t b = __float_as_uint(__ldg(v + i));
    if ((b & mask) == prefix) atomicAdd(&h[(b >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// per-block f64 sums of the moments in index order (grid-size independent
// association only within a block's strided slice; the host adds the block
// sums in block order)
__global__ void __launch_bounds__(256) k_moment_sum(const float* __restrict__ v, uint32_t n,
                                                    double* __restrict__ part) {
  pdl_wait();
  __shared__ double s[256];
  double acc = 0.0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc += (double)__ldg(v + i);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

}  // namespace

constexpr unsigned kMetricBlocks = 148 * 4;

void launch_moment_hist(const float* v, uint32_t n, int shift, uint32_t mask, uint32_t prefix, uint32_t* hist,
                        cudaStream_t st) {
  launch_zero(hist, 256 * 4, st);
  if (!n) return;
  pdl_launch(k_moment_hist, dim3(kMetricBlocks), dim3(256), 0, st, v, n, shift, mask, prefix, hist);
}

void launch_moment_sum(const float* v, uint32_t n, double* part, cudaStream_t st) {
  pdl_launch(k_moment_sum, dim3(kMetricBlocks), dim3(256), 0, st, v, n, part);
}

uint32_t moment_sum_blocks() { return kMetricBlocks; }

}  // namespace s2d
