// dev_common.cuh -- device helpers shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace cc {
namespace dev {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int W = 4;
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int W = 2;
};

__device__ __forceinline__ float4 ldg_vec(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ double2 ldg_vec(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ void zero_vec(float4 &v) { v = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void zero_vec(double2 &v) { v = make_double2(0.0, 0.0); }
__device__ __forceinline__ void add_vec(double *acc, const float4 &v) {
  acc[0] += (double)v.x;
  acc[1] += (double)v.y;
  acc[2] += (double)v.z;
  acc[3] += (double)v.w;
}
__device__ __forceinline__ void add_vec(double *acc, const double2 &v) {
  acc[0] += v.x;
  acc[1] += v.y;
}

__device__ __forceinline__ void add_same(float4 &a, const float4 &b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}
__device__ __forceinline__ void add_same(double2 &a, const double2 &b) {
  a.x += b.x;
  a.y += b.y;
}
__device__ __forceinline__ float vec_at(const float4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }
__device__ __forceinline__ double vec_at(const double2 &v, int i) { return i == 0 ? v.x : v.y; }

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // SplitMix64 finaliser (reading C-2)
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  return (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
}

// item -> (vertex, neighbour range); true for a heavy-vertex segment
__device__ __forceinline__ bool item_range(const AggWork &w, const int64_t *beg, const int64_t *end, int64_t it,
                                           int32_t &v, int64_t &b, int64_t &e) {
  if (it < w.n_seg) {
    v = w.seg_v[it];
    b = w.seg_b[it];
    e = w.seg_e[it];
    return true;
  }
  v = w.light[it - w.n_seg];
  b = beg[v];
  e = end[v];
  return false;
}

template <typename K>
inline int persistent_grid(K kernel, int threads, size_t smem, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms;
}

}  // namespace dev
}  // namespace cc
