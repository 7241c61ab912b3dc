// Calibration probe (not product code): times CUB's DeviceRadixSort on the
// (slot, gradient-row) pairs of one config-2 step, as a yardstick for the
// hand-written K3a sort (k_sort.cu).  Keys come from tools/sort_probe.py.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/sort_probe.cu -o tools/sort_probe
//   tools/sort_probe keys.bin vals.bin
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static std::vector<uint32_t> load(const char* p) {
  FILE* f = fopen(p, "rb");
  if (!f) { printf("cannot open %s\n", p); exit(1); }
  fseek(f, 0, SEEK_END);
  long n = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<uint32_t> v(n);
  if (fread(v.data(), 4, n, f) != (size_t)n) exit(1);
  fclose(f);
  return v;
}

int main(int argc, char** argv) {
  auto hk = load(argv[1]);
  auto hv = load(argv[2]);
  const int n = (int)hk.size();
  int bits = 0;
  uint32_t mx = 0;
  for (auto k : hk) mx = k > mx ? k : mx;
  while ((1u << bits) <= mx && bits < 32) ++bits;
  uint32_t *k0, *v0, *k1, *v1;
  CK(cudaMalloc(&k0, n * 4)); CK(cudaMalloc(&v0, n * 4)); CK(cudaMalloc(&k1, n * 4)); CK(cudaMalloc(&v1, n * 4));
  CK(cudaMemcpy(k0, hk.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v0, hv.data(), n * 4, cudaMemcpyHostToDevice));
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, bits);
  void* dt;
  CK(cudaMalloc(&dt, tmp));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, n, 0, bits);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cub SortPairs n=%d bits=%d: %.1f us\n", n, bits, ms * 1000 / it);
  }
  // copy yardstick: one pass worth of bytes (read 8 B + write 8 B per pair)
  cudaEventRecord(a);
  for (int w = 0; w < 20; ++w) { CK(cudaMemcpyAsync(k1, k0, n * 4, cudaMemcpyDeviceToDevice)); CK(cudaMemcpyAsync(v1, v0, n * 4, cudaMemcpyDeviceToDevice)); }
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("d2d copy of the pairs (one pass of traffic): %.1f us\n", ms * 1000 / 20);
  return 0;
}
