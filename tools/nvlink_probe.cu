// NVLink peer-write probe (2 GPUs): bandwidth of GPU0 -> GPU1 stores for
//   (a) SM stores, 16 B per lane, 512-byte rows at scattered row offsets
//       (the gradient-gather / remote pooled-row pattern),
//   (b) the same rows staged in shared memory and pushed with one
//       cp.async.bulk (TMA bulk) store of 8 rows per warp,
//   (c) cudaMemcpyPeerAsync of one contiguous buffer (copy engines).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

constexpr int kRowF = 128;  // floats per row (512 B)

__global__ void k_store_rows(const float4* __restrict__ src, float4* dst, const unsigned* __restrict__ perm,
                             unsigned rows) {
  const unsigned lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned nw = (gridDim.x * blockDim.x) >> 5;
  for (unsigned r = warp; r < rows; r += nw) {
    const float4 x = src[(size_t)perm[r] * (kRowF / 4) + lane];
    dst[(size_t)r * (kRowF / 4) + lane] = x;
  }
}

__global__ void k_bulk_rows(const float4* __restrict__ src, char* dst, const unsigned* __restrict__ perm,
                            unsigned rows) {
  constexpr int kG = 8;  // rows per bulk store (4 KB)
  extern __shared__ __align__(128) float4 sm[];
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float4* buf = sm + (size_t)wib * 2 * kG * (kRowF / 4);
  int par = 0;
  for (unsigned g = warp * kG; g < rows; g += nw * kG) {
    float4* b = buf + par * kG * (kRowF / 4);
    // the bulk store that last read this half must be done reading
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
    __syncwarp();
    const unsigned n = min((unsigned)kG, rows - g);
    for (unsigned j = 0; j < n; ++j) b[j * (kRowF / 4) + lane] = src[(size_t)perm[g + j] * (kRowF / 4) + lane];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const unsigned s = (unsigned)__cvta_generic_to_shared(b);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst + (size_t)g * kRowF * 4),
                   "r"(s), "r"(n * kRowF * 4)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    par ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("{\"error\": \"need 2 GPUs\"}\n");
    return 0;
  }
  const unsigned rows = 1u << 18;  // 256K rows = 128 MB
  const size_t bytes = (size_t)rows * kRowF * 4;
  CK(cudaSetDevice(1));
  float* d1;
  CK(cudaMalloc(&d1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  float* s0;
  unsigned* perm;
  CK(cudaMalloc(&s0, bytes));
  CK(cudaMalloc(&perm, rows * 4));
  std::vector<unsigned> h(rows);
  for (unsigned i = 0; i < rows; ++i) h[i] = (unsigned)(((unsigned long long)i * 2654435761ull) % rows);
  CK(cudaMemcpy(perm, h.data(), rows * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(s0, 1, bytes));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time_it = [&](auto&& fn) {
    for (int i = 0; i < 3; ++i) fn();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return bytes * (double)reps / (ms * 1e-3) / 1e9;
  };
  const double sm = time_it([&] {
    k_store_rows<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(s0), reinterpret_cast<float4*>(d1), perm, rows);
  });
  const size_t smem = 8 * 2 * 8 * kRowF * 4;  // 8 warps x 2 halves x 8 rows
  CK(cudaFuncSetAttribute(k_bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double bulk = time_it([&] {
    k_bulk_rows<<<148 * 2, 256, smem>>>(reinterpret_cast<const float4*>(s0), reinterpret_cast<char*>(d1), perm, rows);
  });
  const double ce = time_it([&] { CK(cudaMemcpyPeerAsync(d1, 1, s0, 0, bytes, 0)); });
  // bidirectional: GPU1 stores into GPU0 at the same time (per-direction GB/s)
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  float *s1, *d0;
  unsigned* perm1;
  cudaStream_t st1;
  CK(cudaMalloc(&s1, bytes));
  CK(cudaMalloc(&perm1, rows * 4));
  CK(cudaMemcpy(perm1, h.data(), rows * 4, cudaMemcpyHostToDevice));
  CK(cudaStreamCreateWithFlags(&st1, cudaStreamNonBlocking));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&d0, bytes));
  const double bi = time_it([&] {
    CK(cudaSetDevice(1));
    k_store_rows<<<148 * 8, 256, 0, st1>>>(reinterpret_cast<const float4*>(s1), reinterpret_cast<float4*>(d0), perm1,
                                            rows);
    CK(cudaSetDevice(0));
    k_store_rows<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(s0), reinterpret_cast<float4*>(d1), perm, rows);
    CK(cudaSetDevice(1));
    CK(cudaStreamSynchronize(st1));
    CK(cudaSetDevice(0));
  });
  CK(cudaGetLastError());
  std::printf("{\"sm_store_gbs\": %.1f, \"bulk_store_gbs\": %.1f, \"copy_engine_gbs\": %.1f, "
              "\"sm_store_bidir_gbs_per_direction\": %.1f, \"bytes\": %zu}\n",
              sm, bulk, ce, bi, bytes);
  return 0;
}
