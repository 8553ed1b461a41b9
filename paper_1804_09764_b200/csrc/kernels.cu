// kernels.cu -- the per-colouring DP kernels for sm_100a (B200).
//
// Every kernel here is memory- or LSU-bound integer-indexed work; there is no
// dense contraction, so no tensor cores (BASELINE.json north_star).  Grids are
// persistent (a multiple of the SM count x resident blocks per SM, from the
// occupancy calculator) and walk their work with a static interleaved stride,
// so every reduction order -- and therefore every result -- is deterministic.
//
// Tables are colour-compressed (kernels.cuh).  The kernels:
//   k_color   colouring, PAPER.md lines 156-158 (reading C-2)
//   k_csort   per colouring: stable sort of every neighbour range by colour
//             (groups neighbours whose compressed rows share an index space)
//   k_hist    N''(v, {y}): neighbour counts per colour -- the neighbour sum of
//             the single-vertex table (passive part of size 1)
//   k_gather  N''(v, Y'') = sum_{u in N(v)} P(u, Y): the inner sum over u of
//             Eq. 1, SpMM-shaped; per colour group the
//             compressed rows are summed in registers (fp64), then expanded
//             once into the vertex's N'' row in shared memory; heavy
//             neighbour lists are split into segments (Alg. 4)
//             whose partial rows the last arriver sums in segment order
//   k_combine T'(v, S') = sum_{X' u Y'' = S'} A'(v, X') N''(v, Y''): the split
//             sum of Eq. 1, colour-independent in the compressed universe
//   k_root    X = sum_v sum_{X'} A'(v, X') N''(v, [k-1] \ X'): the last step
//             fused with Eq. 3's sum over v, fp64
//   k_pack    halo rows for the 1D partition exchange (Alg. 2 line 15)
// A step whose active part is the single root vertex (a = 1) needs no kernel:
// in the compressed layout its table IS the neighbour sum N''.
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

// item -> (vertex, neighbour range)
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

// ------------------------------------------------------------------ colour
__global__ void k_color(const int32_t *__restrict__ orig, int64_t n, uint64_t seed, int k,
                        uint8_t *__restrict__ out) {
  const uint64_t s = mix64(seed);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(s ^ (uint64_t)(uint32_t)orig[v]) >> 32;
    out[v] = (uint8_t)((h * (uint64_t)k) >> 32);
  }
}

// ------------------------------------------------------------------ colour sort
// One warp per item.  Pass 1 counts colours; pass 2 places each neighbour at
// base[colour] + (rank among equal colours in this 32-wide window), so the
// sort is stable and deterministic.
__global__ void __launch_bounds__(256) k_csort(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                               const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                               AggWork work, int32_t *__restrict__ col_out,
                                               uint16_t *__restrict__ goff) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t n_items = work.n_seg + work.n_light;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; it < n_items; it += nwarps) {
    int32_t v;
    int64_t b, e;
    item_range(work, beg, end, it, v, b, e);
    int cnt[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cnt[j] = 0;
    for (int64_t p = b + lane; p < e; p += 32) {
      const int c = colors[__ldg(col + p)];
#pragma unroll
      for (int j = 0; j < 16; ++j) cnt[j] += (c == j);
    }
    int base[16];
    int run = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt[j] += __shfl_xor_sync(0xffffffffu, cnt[j], o);
      base[j] = run;
      run += cnt[j];
      if (lane == j) goff[it * 16 + j] = (uint16_t)run;
    }
    for (int64_t p0 = b; p0 < e; p0 += 32) {
      const bool ok = p0 + lane < e;
      const int32_t u = ok ? __ldg(col + p0 + lane) : 0;
      const int c = ok ? (int)colors[u] : 16;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const unsigned m = __ballot_sync(0xffffffffu, c == j);
        if (c == j) col_out[b + base[j] + __popc(m & lt)] = u;
        base[j] += __popc(m);
      }
    }
  }
}

// ------------------------------------------------------------------ hist (p = 1)
// Heavy segments add their counts atomically into a zeroed row: the values
// are small integers, exact in fp32/fp64, so the result is order-independent.
template <typename T, int G>
__global__ void __launch_bounds__(256) k_hist(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                              const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                              AggWork work, int k, T *__restrict__ out, int64_t ld) {
  constexpr int U = 4;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = group_mask<G>();
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int64_t n_items = work.n_seg + work.n_light;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; it < n_items; it += ngroups) {
    int32_t v;
    int64_t b, e;
    const bool heavy = item_range(work, beg, end, it, v, b, e);
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
    const int cv = colors[v];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j % G == lane && j < k && j != cv) {
        T *p = out + (int64_t)v * ld + (j < cv ? j : j - 1);  // squeeze: sq_{c_v}(j)
        if (heavy) atomicAdd(p, (T)cnt[j]);
        else *p = (T)cnt[j];
      }
  }
}

// ------------------------------------------------------------------ gather (p >= 2)
template <typename T, int G, int NV, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather(GatherArgs a, int nch) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = G * NV * VW;  // input columns per pass
  extern __shared__ double sacc_all[];
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = group_mask<G>();
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int64_t n_items = a.work.n_seg + a.work.n_light;
  double *sacc = sacc_all + (threadIdx.x / G) * (int64_t)a.W_out;
  const T *__restrict__ src = static_cast<const T *>(a.src);
  T *__restrict__ dst = static_cast<T *>(a.dst);

  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; it < n_items; it += ngroups) {
    int32_t v;
    int64_t b, e;
    const bool heavy = item_range(a.work, a.beg, a.end, it, v, b, e);
    const int cv = a.colors[v];
    for (int j = lane; j < a.W_out; j += G) sacc[j] = 0.0;
    __syncwarp(gmask);
    const uint16_t *go = a.goff + it * 16;
    int gstart = 0;
    for (int cu = 0; cu < a.k; ++cu) {
      const int gend = go[cu];
      if (cu != cv && gend > gstart) {
        const uint16_t *mrow = a.map + (int64_t)(cu * a.k + cv) * a.W_in;
        for (int ch = 0; ch < nch; ++ch) {
          const int c0 = ch * CAP + lane * VW;
          bool valid[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) valid[j] = c0 + j * G * VW < a.W_in;
          double acc[NV][VW];
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) acc[j][q] = 0.0;
          for (int64_t e0 = b + gstart; e0 < b + gend; e0 += G) {
            const int cnt = (int)min((int64_t)G, b + gend - e0);
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
          // expand the colour group's sum into the vertex's N'' row (the map is
          // injective for a fixed colour pair, so lanes never collide)
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) {
              const int y = c0 + j * G * VW + q;
              if (y < a.W_in) {
                const uint16_t m = __ldg(mrow + y);
                if (m != 0xFFFF) sacc[m] += acc[j][q];
              }
            }
        }
        __syncwarp(gmask);
      }
      gstart = gend;
    }

    if (!heavy) {
      T *drow = dst + (int64_t)v * a.ld_dst;
      for (int j = lane; j < a.W_out; j += G) {
        double x = sacc[j];
        if (a.accumulate) x += (double)drow[j];
        drow[j] = (T)x;
      }
    } else {
      double *sp = a.scratch + it * a.ld_scratch;
      for (int j = lane; j < a.W_out; j += G) sp[j] = sacc[j];
      __threadfence();
      __syncwarp(gmask);
      const int32_t hv = a.work.seg_hv[it];
      unsigned prev = 0;
      if (lane == 0) prev = atomicAdd(&a.arrive[hv], 1u);
      prev = __shfl_sync(gmask, prev, 0, G);
      if (prev == (unsigned)(a.work.hv_nseg[hv] - 1)) {  // last arriver reduces in segment order
        __threadfence();
        const int32_t s0 = a.work.hv_first[hv], ns = a.work.hv_nseg[hv];
        T *drow = dst + (int64_t)v * a.ld_dst;
        for (int j = lane; j < a.W_out; j += G) {
          double x = 0.0;
          for (int s = 0; s < ns; ++s) x += __ldcg(a.scratch + (int64_t)(s0 + s) * a.ld_scratch + j);
          if (a.accumulate) x += (double)drow[j];
          drow[j] = (T)x;
        }
      }
    }
    __syncwarp(gmask);
  }
}

// ------------------------------------------------------------------ combine (a >= 2)
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
                                              int64_t ldN, const uint16_t *__restrict__ comp, int64_t n,
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
      s = (double)N[v * ldN];
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

template <typename T, int G, int NV, int U, int MINB = 1>
void gather_go(const GatherArgs &a, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = G * NV * VW;
  auto kern = k_gather<T, G, NV, U, MINB>;
  // shared memory: one fp64 N'' row per group; shrink the block if rows are wide
  const size_t row = (size_t)a.W_out * sizeof(double);
  int groups = 256 / G;
  while (groups > 1 && row * groups > 96 * 1024) groups /= 2;
  const int threads = groups * G;
  const size_t smem = row * groups;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  const int nch = (a.W_in + CAP - 1) / CAP;
  kern<<<grid, threads, smem, s>>>(a, nch);
}

template <typename T>
int gather_typed(const GatherArgs &a, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  if (a.work.n_seg + a.work.n_light == 0) return 0;
  const int wvec = (a.W_in + VW - 1) / VW;
  // one vector per lane per pass (wide rows take several column passes per
  // colour group): few registers, many resident warps, U rows in flight each
  if (wvec <= 4) gather_go<T, 4, 1, 4, 3>(a, num_sms, s);
  else if (wvec <= 8) gather_go<T, 8, 1, 4, 3>(a, num_sms, s);
  else if (wvec <= 16) gather_go<T, 16, 1, 8, 3>(a, num_sms, s);
  else {
    const char *var = getenv("CC_GATHER_VARIANT");  // tuning knob (scripts/agg_sweep.py)
    switch (var ? atoi(var) : 0) {
      case 1: gather_go<T, 32, 1, 8, 3>(a, num_sms, s); break;
      case 2: gather_go<T, 32, 1, 8, 2>(a, num_sms, s); break;
      case 3: gather_go<T, 32, 1, 2, 6>(a, num_sms, s); break;
      case 4: gather_go<T, 32, 1, 4, 5>(a, num_sms, s); break;
      default: gather_go<T, 32, 1, 4, 4>(a, num_sms, s); break;  // measured best (config 3)
    }
  }
  return 1;
}

template <typename T, int V>
void combine_go(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint32_t *split,
                int nq, int64_t n, void *out, int64_t ldO, int WO, int num_sms, cudaStream_t s) {
  auto kern = k_combine<T, V>;
  const size_t smem = (size_t)V * (WA + WN) * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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

int root_partials_blocks(int num_sms) { return num_sms * 8; }

int launch_color(const int32_t *orig, int64_t n, uint64_t seed, int k, uint8_t *out, cudaStream_t s) {
  if (n == 0) return 0;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_color<<<grid, 256, 0, s>>>(orig, n, seed, k, out);
  return 1;
}

int launch_csort(const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                 const AggWork &work, int32_t *col_out, uint16_t *goff, int num_sms, cudaStream_t s) {
  if (work.n_seg + work.n_light == 0) return 0;
  static int grid = 0;
  if (!grid) grid = persistent_grid(k_csort, 256, 0, num_sms);
  k_csort<<<grid, 256, 0, s>>>(beg, end, col, colors, work, col_out, goff);
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

int launch_gather(int elem, const GatherArgs &a, int num_sms, cudaStream_t s) {
  return elem == 8 ? gather_typed<double>(a, num_sms, s) : gather_typed<float>(a, num_sms, s);
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
                int64_t n, double *partials, int n_partials, double *per_vertex, double *result, cudaStream_t s) {
  if (elem == 8)
    k_root<double><<<n_partials, 256, 0, s>>>(static_cast<const double *>(A), ldA, WA, static_cast<const double *>(N),
                                               ldN, comp, n, partials, per_vertex);
  else
    k_root<float><<<n_partials, 256, 0, s>>>(static_cast<const float *>(A), ldA, WA, static_cast<const float *>(N),
                                              ldN, comp, n, partials, per_vertex);
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
