// Function-level forms of the path's two reductions on the device, for
// callers of the reference's free functions rather than the step:
//   pool_ids / lookup_and_pool (include/sparse2d/embedding.hpp:41-58,
//     src/embedding.cpp:39-106): per bag, per shard in presentation order,
//     the f64 sum of the shard's hits in id order rounded to f32, then the
//     f64 sum of those partials rounded to f32;
//   aggregate_group_gradient (include/sparse2d/optimizer.hpp:36-44,
//     src/optimizer.cpp:25-59): a stable sort of the contributions by row
//     (K3a's radix sort), then per row the f64 sum in arrival order times
//     1/group_batch, rows ascending.
// Host buffers in and out; the work runs on the current device.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "device.cuh"

namespace s2d {
namespace {

// first id (by bag-major position) covered by no shard -> *bad (atomicMin)
__global__ void k_pool_check(const uint32_t* __restrict__ ids, uint64_t n, const uint32_t* __restrict__ lo,
                             const uint32_t* __restrict__ hi, uint32_t n_shards,
                             unsigned long long* __restrict__ bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    bool covered = false;
    for (uint32_t s = 0; s < n_shards && !covered; ++s) covered = id >= lo[s] && id < hi[s];
    if (!covered) atomicMin(bad, (unsigned long long)i);
  }
}

// thread per (bag, column)
__global__ void k_pool_bags(const float* __restrict__ w, uint32_t dim, const uint32_t* __restrict__ lo,
                            const uint32_t* __restrict__ hi, uint32_t n_shards, uint64_t n_bags,
                            const uint64_t* __restrict__ bag_off, const uint32_t* __restrict__ ids,
                            float* __restrict__ out) {
  const uint64_t n = n_bags * dim;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = i / dim;
    const uint32_t j = (uint32_t)(i % dim);
    const uint64_t e0 = bag_off[b], e1 = bag_off[b + 1];
    double pool = 0.0;
    for (uint32_t s = 0; s < n_shards; ++s) {
      double partial = 0.0;
      bool hit = false;
      for (uint64_t e = e0; e < e1; ++e) {
        const uint32_t id = ids[e];
        if (id < lo[s] || id >= hi[s]) continue;
        hit = true;
        partial += (double)w[(uint64_t)id * dim + j];
      }
      if (hit) pool += (double)(float)partial;
    }
    out[i] = (float)pool;
  }
}

// warp per row (segment head h = ord-th head): columns over the lanes, the
// segment's contributions summed in sorted (= arrival) order
__global__ void k_segment_sum(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ order,
                              const uint32_t* __restrict__ heads, uint64_t n, const double* __restrict__ grads,
                              uint32_t dim, double inv_batch, uint32_t* __restrict__ out_rows,
                              double* __restrict__ out_g, uint32_t* __restrict__ out_count) {
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  const uint32_t lane = lane_id();
  for (uint64_t p = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); p < n; p += warps) {
    if (p > 0 && keys[p - 1] == keys[p]) continue;  // not a head
    uint64_t e = p + 1;
    while (e < n && keys[e] == keys[p]) ++e;
    const uint32_t ord = heads[p];
    for (uint32_t j = lane; j < dim; j += 32) {
      double acc = 0.0;
      for (uint64_t q = p; q < e; ++q) acc += grads[(uint64_t)order[q] * dim + j];
      out_g[(uint64_t)ord * dim + j] = acc * inv_batch;
    }
    if (lane == 0) {
      out_rows[ord] = keys[p];
      out_count[ord] = (uint32_t)(e - p);
    }
  }
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

unsigned grid_of(uint64_t n) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16)); }

// device buffers freed on scope exit
struct Scratch {
  std::vector<void*> p;
  template <typename T>
  T* alloc(size_t bytes) {
    void* q = nullptr;
    S2D_CUDA(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
    p.push_back(q);
    return reinterpret_cast<T*>(q);
  }
  ~Scratch() {
    for (void* q : p) dev_free(q);
  }
};

template <typename Fn>
int fguard(Fn&& fn) {
  try {
    fn();
    return S2D_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return S2D_ERUNTIME;
  }
}

}  // namespace
}  // namespace s2d

using s2d::Error;

extern "C" {

int s2d_pool_ids(const float* w, uint32_t rows, uint32_t dim, uint32_t table_id, uint32_t n_shards,
                 const uint32_t* lo, const uint32_t* hi, uint64_t n_bags, const uint64_t* bag_off,
                 const uint32_t* ids, float* out) {
  return s2d::fguard([&] {
    if (n_shards == 0) throw Error(S2D_EINVAL, "empty shard set");
    if (dim > (uint32_t)s2d::kMaxDim) throw Error(S2D_EINVAL, "dim too large for pooling");
    if (!w || !lo || !hi || !bag_off || !out) throw Error(S2D_EINVAL, "null argument");
    for (uint32_t s = 0; s < n_shards; ++s)
      if (lo[s] > hi[s] || hi[s] > rows) throw Error(S2D_EINVAL, "shard range outside the table");
    if (n_bags == 0 || dim == 0) return;
    const uint64_t nnz = bag_off[n_bags];
    if (nnz && !ids) throw Error(S2D_EINVAL, "null ids");
    s2d::Scratch sc;
    float* dw = sc.alloc<float>((size_t)rows * dim * 4);
    uint32_t* dlo = sc.alloc<uint32_t>((size_t)n_shards * 4);
    uint32_t* dhi = sc.alloc<uint32_t>((size_t)n_shards * 4);
    uint64_t* doff = sc.alloc<uint64_t>((n_bags + 1) * 8);
    uint32_t* dids = sc.alloc<uint32_t>(nnz * 4);
    float* dout = sc.alloc<float>((size_t)n_bags * dim * 4);
    unsigned long long* dbad = sc.alloc<unsigned long long>(8);
    S2D_CUDA(cudaMemcpy(dw, w, (size_t)rows * dim * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemcpy(dlo, lo, (size_t)n_shards * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemcpy(dhi, hi, (size_t)n_shards * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemcpy(doff, bag_off, (n_bags + 1) * 8, cudaMemcpyHostToDevice));
    if (nnz) S2D_CUDA(cudaMemcpy(dids, ids, nnz * 4, cudaMemcpyHostToDevice));
    S2D_CUDA(cudaMemset(dbad, 0xff, 8));
    if (nnz) {
      // coverage first, so the error does not depend on shard order (embedding.cpp:46-65)
      s2d::k_pool_check<<<s2d::grid_of(nnz), 256>>>(dids, nnz, dlo, dhi, n_shards, dbad);
      S2D_LAUNCH_CHECK();
      unsigned long long bad = 0;
      S2D_CUDA(cudaMemcpy(&bad, dbad, 8, cudaMemcpyDeviceToHost));
      if (bad != ~0ull) {
        std::string ranges;
        for (uint32_t s = 0; s < n_shards; ++s)
          ranges += " [" + std::to_string(lo[s]) + "," + std::to_string(hi[s]) + ")";
        throw Error(S2D_ERANGE, "lookup id " + std::to_string(ids[bad]) + " outside shard ranges of table " +
                                    std::to_string(table_id) + ":" + ranges);
      }
    }
    s2d::k_pool_bags<<<s2d::grid_of(n_bags * dim), 256>>>(dw, dim, dlo, dhi, n_shards, n_bags, doff, dids, dout);
    S2D_LAUNCH_CHECK();
    S2D_CUDA(cudaMemcpy(out, dout, (size_t)n_bags * dim * 4, cudaMemcpyDeviceToHost));
  });
}

int s2d_aggregate_group_gradient(const uint32_t* rows, const double* grads, uint64_t n, uint32_t group_batch,
                                 uint32_t dim, uint32_t* out_rows, double* out_g, uint32_t* out_count, uint64_t cap,
                                 uint64_t* n_out) {
  return s2d::fguard([&] {
    if (group_batch == 0) throw Error(S2D_EINVAL, "group batch size must be > 0");
    if (!n_out) throw Error(S2D_EINVAL, "null argument");
    *n_out = 0;
    if (n == 0) return;
    if (n >= 0xffffffffull) throw Error(S2D_EINVAL, "too many contributions");
    if (!rows || !grads) throw Error(S2D_EINVAL, "null argument");
    s2d::Scratch sc;
    uint32_t max_row = 0;
    for (uint64_t i = 0; i < n; ++i) max_row = std::max(max_row, rows[i]);
    int bits = 1;
    while (bits < 32 && (max_row >> bits) != 0) ++bits;
    uint32_t* ka = sc.alloc<uint32_t>(n * 4);
    uint32_t* va = sc.alloc<uint32_t>(n * 4);
    uint32_t* kb = sc.alloc<uint32_t>(n * 4);
    uint32_t* vb = sc.alloc<uint32_t>(n * 4);
    double* dg = sc.alloc<double>((size_t)n * dim * 8);
    const size_t tmp_bytes = std::max(s2d::radix_tmp_bytes(n, bits), s2d::scan_tmp_bytes(n + 1));
    void* tmp = sc.alloc<char>(tmp_bytes);
    uint32_t* heads = sc.alloc<uint32_t>((n + 1) * 4);
    S2D_CUDA(cudaMemcpy(ka, rows, n * 4, cudaMemcpyHostToDevice));
    if (dim) S2D_CUDA(cudaMemcpy(dg, grads, (size_t)n * dim * 8, cudaMemcpyHostToDevice));
    s2d::k_iota<<<s2d::grid_of(n), 256>>>(va, n);
    S2D_LAUNCH_CHECK();
    // stable sort by row: arrival order kept within a row (optimizer.cpp:31-35)
    const bool in_b = s2d::radix_sort_pairs(ka, va, kb, vb, n, bits, tmp, tmp_bytes, nullptr);
    const uint32_t* sk = in_b ? kb : ka;
    const uint32_t* sv = in_b ? vb : va;
    // every key is a real row: heads counted with n_slots past the largest
    s2d::scan_heads_u32(sk, heads, n, max_row + 1 > max_row ? max_row + 1 : max_row, nullptr, tmp, tmp_bytes);
    uint32_t U = 0;
    S2D_CUDA(cudaMemcpy(&U, heads + n, 4, cudaMemcpyDeviceToHost));
    *n_out = U;
    if (!out_rows && !out_g && !out_count) return;  // size query
    if (cap < U) throw Error(S2D_EINVAL, "output capacity too small");
    uint32_t* drow = sc.alloc<uint32_t>((size_t)U * 4);
    uint32_t* dcnt = sc.alloc<uint32_t>((size_t)U * 4);
    double* dout = sc.alloc<double>((size_t)U * dim * 8);
    const double inv_batch = 1.0 / static_cast<double>(group_batch);
    s2d::k_segment_sum<<<s2d::grid_of(n * 32), 256>>>(sk, sv, heads, n, dg, dim, inv_batch, drow, dout, dcnt);
    S2D_LAUNCH_CHECK();
    if (out_rows) S2D_CUDA(cudaMemcpy(out_rows, drow, (size_t)U * 4, cudaMemcpyDeviceToHost));
    if (out_count) S2D_CUDA(cudaMemcpy(out_count, dcnt, (size_t)U * 4, cudaMemcpyDeviceToHost));
    if (out_g && dim) S2D_CUDA(cudaMemcpy(out_g, dout, (size_t)U * dim * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
