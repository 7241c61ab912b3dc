// Device helpers shared by the kernels.  Everything is compiled with
// -fmad=false so f64/f32 expressions round exactly as written, matching the
// reference's -ffp-contract=off build (proj/CMakeLists.txt:11-14).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "common.h"

namespace s2d {

__device__ __forceinline__ uint64_t shfl64(uint64_t v, uint32_t src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: a kernel launched with pdl_launch may be
// scheduled while its predecessor on the stream drains; it waits here (first
// statement, before touching any predecessor output) until that grid has
// completed and flushed.  A no-op when launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Let the dependent grid be scheduled now (persistent single-wave kernels
// only: a multi-wave grid would hand its free slots to waiting blocks).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// 16-byte weight vector -> 4 doubles.  fp32: one float4; bf16: 4 x bf16 (8 B).
template <typename WT>
struct Vec4;

template <>
struct Vec4<float> {
  static __device__ __forceinline__ void load(const float* p, double (&d)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    d[0] = (double)x.x;
    d[1] = (double)x.y;
    d[2] = (double)x.z;
    d[3] = (double)x.w;
  }
  static __device__ __forceinline__ void load_rw(const float* p, double (&d)[4]) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    d[0] = (double)x.x;
    d[1] = (double)x.y;
    d[2] = (double)x.z;
    d[3] = (double)x.w;
  }
  static __device__ __forceinline__ void store(float* p, const double (&d)[4]) {
    float4 x;
    x.x = (float)d[0];
    x.y = (float)d[1];
    x.z = (float)d[2];
    x.w = (float)d[3];
    *reinterpret_cast<float4*>(p) = x;
  }
};

template <>
struct Vec4<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, double (&d)[4]) {
    const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    d[0] = (double)__uint_as_float(x.x << 16);
    d[1] = (double)__uint_as_float(x.x & 0xffff0000u);
    d[2] = (double)__uint_as_float(x.y << 16);
    d[3] = (double)__uint_as_float(x.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void load_rw(const __nv_bfloat16* p, double (&d)[4]) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    d[0] = (double)__uint_as_float(x.x << 16);
    d[1] = (double)__uint_as_float(x.x & 0xffff0000u);
    d[2] = (double)__uint_as_float(x.y << 16);
    d[3] = (double)__uint_as_float(x.y & 0xffff0000u);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const double (&d)[4]) {
    // f64 -> bf16 with one round-to-nearest-even (no f32 double rounding)
    uint2 x;
    const uint16_t b0 = __bfloat16_as_ushort(__double2bfloat16(d[0]));
    const uint16_t b1 = __bfloat16_as_ushort(__double2bfloat16(d[1]));
    const uint16_t b2 = __bfloat16_as_ushort(__double2bfloat16(d[2]));
    const uint16_t b3 = __bfloat16_as_ushort(__double2bfloat16(d[3]));
    x.x = (uint32_t)b0 | ((uint32_t)b1 << 16);
    x.y = (uint32_t)b2 | ((uint32_t)b3 << 16);
    *reinterpret_cast<uint2*>(p) = x;
  }
};

__device__ __forceinline__ void load_f32x4_d(const float* p, double (&d)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p));
  d[0] = (double)x.x;
  d[1] = (double)x.y;
  d[2] = (double)x.z;
  d[3] = (double)x.w;
}

__device__ __forceinline__ void store_f32x4_stream(float* p, const double (&d)[4]) {
  float4 x;
  x.x = (float)d[0];
  x.y = (float)d[1];
  x.z = (float)d[2];
  x.w = (float)d[3];
  __stcs(reinterpret_cast<float4*>(p), x);
}

// Feature owning a slot: largest i with vbase_sorted[i] <= slot.
__device__ __forceinline__ uint32_t feature_of_slot(const uint32_t* vbase_sorted,
                                                    const uint32_t* feat_of_vbase, uint32_t n,
                                                    uint32_t slot) {
  uint32_t lo = 0, hi = n;  // invariant: vbase_sorted[lo] <= slot < vbase_sorted[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(vbase_sorted + mid) <= slot)
      lo = mid;
    else
      hi = mid;
  }
  return __ldg(feat_of_vbase + lo);
}

}  // namespace s2d
