// kernels.cu -- the per-colouring DP kernels for sm_100a (B200).
//
// Every kernel here is memory- or LSU-bound integer-indexed work; there is no
// dense contraction, so no tensor cores (BASELINE.json north_star).  Grids are
// persistent (a multiple of the SM count x resident blocks per SM, from the
// occupancy calculator) and walk their work with a static interleaved stride,
// so every reduction order -- and therefore every result -- is deterministic.
//
//   k_color   colouring, PAPER.md lines 156-158 (reading C-2)
//   k_hist    N(v, {c}) = #{u in N(v): col u = c}: the neighbour sum of the
//             single-vertex table (passive part of size 1)
//   k_agg     N(v, Y) = sum_{u in N(v)} P(u, Y): the inner sum over u of
//             Eq. 1, SpMM-shaped, column-chunked,
//             heavy neighbour lists split into segments (Alg. 4, lines
//             494-523) and reduced deterministically by the last arriver
//   k_lift    T(v, S) = [c_v in S] N(v, S \ {c_v}): a step whose active part
//             is the single root vertex (split sum has one term)
//   k_combine T(v, S) = sum_{S1 u S2 = S} A(v, S1) N(v, S2): the split sum of
//             Eq. 1 over the split table of the step
//   k_root    X = sum_v sum_{S1} A(v, S1) N(v, [k] \ S1): the last step fused
//             with Eq. 3's sum over v, fp64
//   k_pack    halo rows for the 1D partition exchange (Alg. 2 line 15)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace cc {
namespace dev {

namespace {

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
__device__ __forceinline__ void store_vec(float *p, const double *acc) {
  *reinterpret_cast<float4 *>(p) = make_float4((float)acc[0], (float)acc[1], (float)acc[2], (float)acc[3]);
}
__device__ __forceinline__ void store_vec(double *p, const double *acc) {
  *reinterpret_cast<double2 *>(p) = make_double2(acc[0], acc[1]);
}
__device__ __forceinline__ void load_add(const float *p, double *acc) {
  float4 v = *reinterpret_cast<const float4 *>(p);
  add_vec(acc, v);
}
__device__ __forceinline__ void load_add(const double *p, double *acc) {
  double2 v = *reinterpret_cast<const double2 *>(p);
  add_vec(acc, v);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // SplitMix64 finaliser (reading C-2)
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ colour
__global__ void k_color(const int32_t *__restrict__ orig, int64_t n, uint64_t seed, int k,
                        uint8_t *__restrict__ out) {
  const uint64_t s = mix64(seed);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(s ^ (uint64_t)(uint32_t)orig[v]) >> 32;
    out[v] = (uint8_t)((h * (uint64_t)k) >> 32);
  }
}

// ------------------------------------------------------------------ hist
// Work items as in k_agg (light vertices, segments of heavy neighbour lists).
// Segment partial counts are added with atomics into a zeroed row: the values
// are small integers, exact in fp32/fp64, so the result is order-independent.
template <typename T, int G>
__global__ void __launch_bounds__(256) k_hist(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                              const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                              AggWork work, int k, T *__restrict__ out, int64_t ld) {
  constexpr int U = 4;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int64_t n_items = work.n_seg + work.n_light;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; it < n_items; it += ngroups) {
    const bool heavy = it < work.n_seg;
    int64_t b, e;
    int32_t v;
    if (heavy) {
      v = work.seg_v[it];
      b = work.seg_b[it];
      e = work.seg_e[it];
    } else {
      v = work.light[it - work.n_seg];
      b = beg[v];
      e = end[v];
    }
    int cnt[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cnt[j] = 0;
    for (int64_t e0 = b + lane; e0 < e; e0 += G * U) {
      int32_t u[U];
#pragma unroll
      for (int q = 0; q < U; ++q) u[q] = e0 + q * G < e ? __ldg(col + e0 + q * G) : -1;
      int c[U];
#pragma unroll
      for (int q = 0; q < U; ++q) c[q] = u[q] >= 0 ? (int)colors[u[q]] : 16;
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int j = 0; j < 16; ++j) cnt[j] += (c[q] == j);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) cnt[j] += __shfl_xor_sync(gmask, cnt[j], o, G);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j % G == lane && j < k) {
        if (heavy) atomicAdd(out + (int64_t)v * ld + j, (T)cnt[j]);
        else out[(int64_t)v * ld + j] = (T)cnt[j];
      }
  }
}

// ------------------------------------------------------------------ aggregation
template <typename T, int G, int NV, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_agg(AggArgs a, int nchunks, int CW) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int64_t n_items = a.work.n_seg + a.work.n_light;
  const int64_t total = n_items * nchunks;
  const T *__restrict__ src = static_cast<const T *>(a.src);
  T *__restrict__ dst = static_cast<T *>(a.dst);

  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; w < total; w += ngroups) {
    const int chunk = (int)(w / n_items);
    const int64_t it = w - (int64_t)chunk * n_items;
    const bool heavy = it < a.work.n_seg;
    int64_t b, e;
    int32_t v;
    if (heavy) {
      v = a.work.seg_v[it];
      b = a.work.seg_b[it];
      e = a.work.seg_e[it];
    } else {
      v = a.work.light[it - a.work.n_seg];
      b = a.beg[v];
      e = a.end[v];
    }
    const int c0 = chunk * CW + lane * VW;
    bool valid[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) valid[j] = (lane * VW + j * G * VW < CW) && (c0 + j * G * VW < a.W);
    double acc[NV][VW];
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < VW; ++q) acc[j][q] = 0.0;

    for (int64_t e0 = b; e0 < e; e0 += G) {
      const int cnt = (int)min((int64_t)G, e - e0);
      const int32_t my_u = lane < cnt ? __ldg(a.col + e0 + lane) : 0;
      for (int j0 = 0; j0 < cnt; j0 += U) {
        V vals[U][NV];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
          const int32_t u = __shfl_sync(gmask, my_u, (j0 + uu) & (G - 1), G);
          const T *row = src + (int64_t)u * a.ld_src + c0;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            if (j0 + uu < cnt && valid[j]) vals[uu][j] = ldg_vec(row + j * G * VW);
            else zero_vec(vals[uu][j]);
          }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
#pragma unroll
          for (int j = 0; j < NV; ++j) add_vec(acc[j], vals[uu][j]);
      }
    }

    if (!heavy) {
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (valid[j]) {
          T *p = dst + (int64_t)v * a.ld_dst + c0 + j * G * VW;
          if (a.accumulate) load_add(p, acc[j]);
          store_vec(p, acc[j]);
        }
    } else {
      double *sp = a.scratch + it * a.ld_scratch + c0;
#pragma unroll
      for (int j = 0; j < NV; ++j)
        if (valid[j]) {
#pragma unroll
          for (int q = 0; q < VW; q += 2)
            *reinterpret_cast<double2 *>(sp + j * G * VW + q) = make_double2(acc[j][q], acc[j][q + 1]);
        }
      __threadfence();
      __syncwarp(gmask);
      const int32_t hv = a.work.seg_hv[it];
      unsigned prev = 0;
      if (lane == 0) prev = atomicAdd(&a.arrive[(int64_t)hv * nchunks + chunk], 1u);
      prev = __shfl_sync(gmask, prev, 0, G);
      if (prev == (unsigned)(a.work.hv_nseg[hv] - 1)) {  // last arriver reduces in segment order
        __threadfence();
        const int32_t s0 = a.work.hv_first[hv], ns = a.work.hv_nseg[hv];
#pragma unroll
        for (int j = 0; j < NV; ++j)
#pragma unroll
          for (int q = 0; q < VW; ++q) acc[j][q] = 0.0;
        for (int s = 0; s < ns; ++s) {
          const double *p = a.scratch + (int64_t)(s0 + s) * a.ld_scratch + c0;
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if (valid[j]) {
#pragma unroll
              for (int q = 0; q < VW; q += 2) {
                double2 x = __ldcg(reinterpret_cast<const double2 *>(p + j * G * VW + q));
                acc[j][q] += x.x;
                acc[j][q + 1] += x.y;
              }
            }
        }
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (valid[j]) {
            T *p = dst + (int64_t)v * a.ld_dst + c0 + j * G * VW;
            if (a.accumulate) load_add(p, acc[j]);
            store_vec(p, acc[j]);
          }
      }
    }
  }
}

// ------------------------------------------------------------------ lift (a = 1)
template <typename T>
__global__ void __launch_bounds__(256) k_lift(const T *__restrict__ N, int64_t ldN, const uint8_t *__restrict__ colors,
                                              const uint16_t *__restrict__ drop, int64_t n, int Wt,
                                              T *__restrict__ out, int64_t ldO) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; v < n; v += nwarps) {
    const int c = colors[v];
    const T *nr = N + v * ldN;
    T *orow = out + v * ldO;
    for (int r = lane; r < Wt; r += 32) {
      const uint16_t d = __ldg(drop + r * 16 + c);
      orow[r] = d == 0xFFFF ? (T)0 : nr[d];
    }
  }
}

// ------------------------------------------------------------------ combine
template <typename T, int V>
__global__ void __launch_bounds__(256) k_combine(const T *__restrict__ A, int64_t ldA, int WA,
                                                 const T *__restrict__ N, int64_t ldN, int WN,
                                                 const uint32_t *__restrict__ split, int nq, int64_t n,
                                                 T *__restrict__ out, int64_t ldO, int WO) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *As = reinterpret_cast<T *>(smem_raw);
  T *Ns = As + V * WA;
  const int64_t ntiles = (n + V - 1) / V;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * V;
    const int nv = (int)min((int64_t)V, n - v0);
    for (int i = threadIdx.x; i < V * WA; i += blockDim.x) {
      const int r = i / WA, x = i - r * WA;
      As[i] = r < nv ? A[(v0 + r) * ldA + x] : (T)0;
    }
    for (int i = threadIdx.x; i < V * WN; i += blockDim.x) {
      const int r = i / WN, y = i - r * WN;
      Ns[i] = r < nv ? N[(v0 + r) * ldN + y] : (T)0;
    }
    __syncthreads();
    for (int s = threadIdx.x; s < WO; s += blockDim.x) {
      double acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.0;
      for (int q = 0; q < nq; ++q) {
        const uint32_t sp = __ldg(split + (int64_t)q * WO + s);
        const int x = sp & 0xFFFF, y = sp >> 16;
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += (double)As[i * WA + x] * (double)Ns[i * WN + y];
      }
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (i < nv) out[(v0 + i) * ldO + s] = (T)acc[i];
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ root
template <typename T>
__global__ void __launch_bounds__(256) k_root(const T *__restrict__ A, int64_t ldA, int WA, const T *__restrict__ N,
                                              int64_t ldN, const uint16_t *__restrict__ comp,
                                              const uint8_t *__restrict__ colors, int64_t n,
                                              double *__restrict__ partials, double *__restrict__ per_vertex) {
  __shared__ double wsum_s[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  double wsum = 0.0;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; v < n; v += nwarps) {
    double s = 0.0;
    if (A) {
      const T *ar = A + v * ldA;
      const T *nr = N + v * ldN;
      for (int x = lane; x < WA; x += 32) s += (double)ar[x] * (double)nr[__ldg(comp + x)];
    } else if (lane == 0) {
      s = (double)N[v * ldN + __ldg(comp + colors[v])];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (per_vertex) per_vertex[v] = s;
      wsum += s;
    }
  }
  if (lane == 0) wsum_s[warp] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) b += wsum_s[i];
    partials[blockIdx.x] = b;
  }
}

__global__ void k_reduce(const double *__restrict__ partials, int np, double *__restrict__ out) {
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int i = lane; i < np; i += 32) s += partials[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) out[0] = s;
}

// ------------------------------------------------------------------ pack
template <typename T>
__global__ void __launch_bounds__(256) k_pack(const T *__restrict__ src, int64_t ld, const int32_t *__restrict__ idx,
                                              int64_t rows, T *__restrict__ out) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t nvec = ld / VW;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < rows; i += nwarps) {
    const V *s = reinterpret_cast<const V *>(src + (int64_t)idx[i] * ld);
    V *o = reinterpret_cast<V *>(out + i * ld);
    for (int64_t j = lane; j < nvec; j += 32) o[j] = s[j];
  }
}

// ------------------------------------------------------------------ helpers
template <typename K>
int persistent_grid(K kernel, int threads, size_t smem, int num_sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms;
}

template <typename T, int G, int NV, int U = (G * NV >= 32) ? 8 : 4, int MINB = 1>
void agg_go(const AggArgs &a, int nchunks, int CW, int num_sms, cudaStream_t s) {
  auto kern = k_agg<T, G, NV, U, MINB>;
  static int grid = 0;
  if (!grid) grid = persistent_grid(kern, 256, 0, num_sms);
  kern<<<grid, 256, 0, s>>>(a, nchunks, CW);
}

// Tuning variants of the wide-row kernel (G = 32), selected by CC_AGG_VARIANT.
int agg_variant() {
  const char *e = getenv("CC_AGG_VARIANT");
  return e ? atoi(e) : 0;
}

void agg_shape(int VW, int W, int64_t chunk_cols, int *G, int *NV) {
  const int wvec = (W + VW - 1) / VW;  // vectors per row
  if (wvec <= 4) { *G = 4; *NV = 1; }
  else if (wvec <= 8) { *G = 8; *NV = 1; }
  else if (wvec <= 16) { *G = 16; *NV = 1; }
  else if (wvec <= 32) { *G = 32; *NV = 1; }
  else { *G = 32; *NV = 2; }
  if (chunk_cols > 0 && *G == 32) *NV = chunk_cols > 32 * VW ? 2 : 1;  // explicit chunk width
}

// Balanced column chunks: as few passes as the group's capacity allows, with
// equal widths (a multiple of the vector width), so no pass runs nearly empty.
void agg_chunking(int VW, int W, int cap, int *CW, int *nchunks) {
  *nchunks = (W + cap - 1) / cap;
  if (*nchunks < 1) *nchunks = 1;
  const int per = (W + *nchunks - 1) / *nchunks;
  *CW = (per + VW - 1) / VW * VW;
}

template <typename T>
int agg_typed(const AggArgs &a, int64_t chunk_cols, int num_sms, int *nchunks_out, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  int G, NV, CW, nchunks;
  agg_shape(VW, a.W, chunk_cols, &G, &NV);
  agg_chunking(VW, a.W, G * NV * VW, &CW, &nchunks);
  if (nchunks_out) *nchunks_out = nchunks;
  if (a.work.n_seg + a.work.n_light == 0) return 0;
  switch (G * 10 + NV) {
    case 41: agg_go<T, 4, 1>(a, nchunks, CW, num_sms, s); break;
    case 81: agg_go<T, 8, 1>(a, nchunks, CW, num_sms, s); break;
    case 161: agg_go<T, 16, 1>(a, nchunks, CW, num_sms, s); break;
    case 321:
      if (agg_variant() == 3) agg_go<T, 32, 1, 16>(a, nchunks, CW, num_sms, s);
      else agg_go<T, 32, 1>(a, nchunks, CW, num_sms, s);
      break;
    default:
      switch (agg_variant()) {
        case 1: agg_go<T, 32, 2, 4>(a, nchunks, CW, num_sms, s); break;
        case 2: agg_go<T, 32, 2, 4, 2>(a, nchunks, CW, num_sms, s); break;
        case 5: agg_go<T, 32, 2>(a, nchunks, CW, num_sms, s); break;
        default: agg_go<T, 32, 2, 8, 2>(a, nchunks, CW, num_sms, s); break;  // measured best (config 3)
      }
      break;
  }
  return 1;
}

template <typename T, int V>
void combine_go(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint32_t *split,
                int nq, int64_t n, void *out, int64_t ldO, int WO, int num_sms, cudaStream_t s) {
  auto kern = k_combine<T, V>;
  const size_t smem = (size_t)V * (WA + WN) * sizeof(T);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  const int grid = persistent_grid(kern, 256, smem, num_sms);
  kern<<<grid, 256, smem, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, split, nq, n,
                               static_cast<T *>(out), ldO, WO);
}

template <typename T>
void combine_typed(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint32_t *split,
                   int nq, int64_t n, void *out, int64_t ldO, int WO, int num_sms, cudaStream_t s) {
  const size_t row = (size_t)(WA + WN) * sizeof(T);
  const size_t budget = 100 * 1024;
  if (row * 16 <= budget) combine_go<T, 16>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  else if (row * 8 <= budget) combine_go<T, 8>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  else if (row * 4 <= budget) combine_go<T, 4>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  else if (row * 2 <= budget) combine_go<T, 2>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  else combine_go<T, 1>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
}

}  // namespace

int agg_partials_blocks(int num_sms) { return num_sms * 8; }

int agg_nchunks(int elem, int W, int64_t chunk_cols) {
  const int VW = elem == 8 ? 2 : 4;
  int G, NV, CW, nchunks;
  agg_shape(VW, W, chunk_cols, &G, &NV);
  agg_chunking(VW, W, G * NV * VW, &CW, &nchunks);
  return nchunks;
}

int launch_color(const int32_t *orig, int64_t n, uint64_t seed, int k, uint8_t *out, cudaStream_t s) {
  if (n == 0) return 0;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_color<<<grid, 256, 0, s>>>(orig, n, seed, k, out);
  return 1;
}

int launch_hist(int elem, const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                const AggWork &work, int64_t n, int k, void *out, int64_t ld, int num_sms, cudaStream_t s) {
  if (work.n_seg + work.n_light == 0) return 0;
  int launches = 1;
  if (work.n_seg) {  // heavy rows accumulate segment counts atomically
    cudaMemsetAsync(out, 0, (size_t)n * ld * elem, s);
    ++launches;
  }
  if (elem == 8) {
    static int grid = 0;
    if (!grid) grid = persistent_grid(k_hist<double, 8>, 256, 0, num_sms);
    k_hist<double, 8><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, static_cast<double *>(out), ld);
  } else {
    static int grid = 0;
    if (!grid) grid = persistent_grid(k_hist<float, 8>, 256, 0, num_sms);
    k_hist<float, 8><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, static_cast<float *>(out), ld);
  }
  return launches;
}

int launch_agg(int elem, const AggArgs &a, int64_t chunk_cols, int num_sms, int *nchunks_out, cudaStream_t s) {
  return elem == 8 ? agg_typed<double>(a, chunk_cols, num_sms, nchunks_out, s)
                   : agg_typed<float>(a, chunk_cols, num_sms, nchunks_out, s);
}

int launch_lift(int elem, const void *N, int64_t ldN, const uint8_t *colors, const uint16_t *drop, int64_t n, int Wt,
                void *out, int64_t ldO, int num_sms, cudaStream_t s) {
  if (n == 0) return 0;
  if (elem == 8) {
    static int grid = 0;
    if (!grid) grid = persistent_grid(k_lift<double>, 256, 0, num_sms);
    k_lift<double><<<grid, 256, 0, s>>>(static_cast<const double *>(N), ldN, colors, drop, n, Wt,
                                         static_cast<double *>(out), ldO);
  } else {
    static int grid = 0;
    if (!grid) grid = persistent_grid(k_lift<float>, 256, 0, num_sms);
    k_lift<float><<<grid, 256, 0, s>>>(static_cast<const float *>(N), ldN, colors, drop, n, Wt,
                                        static_cast<float *>(out), ldO);
  }
  return 1;
}

int launch_combine(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                   const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, int num_sms,
                   cudaStream_t s) {
  if (n == 0) return 0;
  if (elem == 8) combine_typed<double>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  else combine_typed<float>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, num_sms, s);
  return 1;
}

int launch_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, const uint16_t *comp,
                const uint8_t *colors, int64_t n, double *partials, int n_partials, double *per_vertex,
                double *result, cudaStream_t s) {
  if (elem == 8)
    k_root<double><<<n_partials, 256, 0, s>>>(static_cast<const double *>(A), ldA, WA, static_cast<const double *>(N),
                                               ldN, comp, colors, n, partials, per_vertex);
  else
    k_root<float><<<n_partials, 256, 0, s>>>(static_cast<const float *>(A), ldA, WA, static_cast<const float *>(N),
                                              ldN, comp, colors, n, partials, per_vertex);
  k_reduce<<<1, 32, 0, s>>>(partials, n_partials, result);
  return 2;
}

int launch_pack(int elem, const void *src, int64_t ld, const int32_t *idx, int64_t rows, void *out, cudaStream_t s) {
  if (rows == 0) return 0;
  const int grid = (int)std::min<int64_t>((rows + 7) / 8, 148 * 8);
  if (elem == 8)
    k_pack<double><<<grid, 256, 0, s>>>(static_cast<const double *>(src), ld, idx, rows, static_cast<double *>(out));
  else
    k_pack<float><<<grid, 256, 0, s>>>(static_cast<const float *>(src), ld, idx, rows, static_cast<float *>(out));
  return 1;
}

}  // namespace dev
}  // namespace cc
