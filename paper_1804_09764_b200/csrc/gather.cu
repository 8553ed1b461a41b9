// gather.cu -- the neighbour-sum kernels of the DP (sm_100a).
//
//   k_csort2       per colouring (one GPU): stable sort of every work item's
//                  neighbour range by neighbour colour (match_any groups),
//                  the 16 colour-group ends, the item descriptor, and the
//                  leaf level N''(v, {y}) in the same pass;
//   k_csort_small  the same for the <= 8-neighbour tail, 4 items per warp;
//   k_csort        the sort alone for the multi-rank local / remote passes
//                  (neighbours whose compressed rows share an index space
//                  become contiguous)
//   k_hist         N''(v, {y}): neighbour counts per colour -- the neighbour
//                  sum of the single-vertex table (passive part of size 1),
//                  multi-rank path
//   k_gather_ring  N''(v, Y'') = sum_{u in N(v)} P(u, Y): the inner sum over
//                  u of Eq. 1, SpMM-shaped.  Rows of the
//                  compressed passive table are fetched with cp.async into a
//                  per-group shared-memory ring; per colour group they are
//                  summed in registers and expanded once into the vertex's
//                  N'' row in shared memory through the colour-pair map.
//                  Heavy neighbour lists are split into segments (Alg. 4,
//                  PAPER.md lines 494-523) whose partial rows the last
//                  arriving segment sums in segment order (deterministic).
//                  Used for rows of <= 16 vectors (4 / 8 lanes per item).
//   k_gather_ldg   the same sum for rows of > 16 vectors: one warp per item,
//                  plain LDG.128 rows, U rows in flight, ~20 instructions per
//                  row (the ring's per-row bookkeeping made it issue-bound);
//                  optionally evaluates the root step in its epilogue.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "dev_common.cuh"

namespace cc {
namespace dev {

namespace {

// ------------------------------------------------------------------ colour sort
// One warp per item.  Pass 1 counts colours; pass 2 places each neighbour at
// base[colour] + (rank among equal colours in this 32-wide window): stable.
__global__ void __launch_bounds__(256) k_csort(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                               const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                               AggWork work, int32_t *__restrict__ col_out,
                                               uint16_t *__restrict__ goff, ItemDesc *__restrict__ desc) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t n_items = work.n_seg + work.n_light;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; it < n_items; it += nwarps) {
    int32_t v;
    int64_t b, e;
    const bool heavy = item_range(work, beg, end, it, v, b, e);
    const int cv = colors[v];
    int cnt[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cnt[j] = 0;
    for (int64_t p = b + lane; p < e; p += 32) {
      const int c = colors[__ldg(col + p)];
#pragma unroll
      for (int j = 0; j < 16; ++j) cnt[j] += (c == j);
    }
    int base[16];
    int run = 0, cv_lo = 0, skip = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt[j] += __shfl_xor_sync(0xffffffffu, cnt[j], o);
      base[j] = run;
      if (j == cv) {
        cv_lo = run;
        skip = cnt[j];
      }
      run += cnt[j];
      if (lane == j) goff[it * 16 + j] = (uint16_t)run;
    }
    if (lane == 0) {
      ItemDesc d;
      d.b = b;
      d.v = v;
      d.n_s = (int32_t)(e - b) - skip;
      d.cv_lo = cv_lo;
      d.skip = skip;
      d.cv = cv;
      d.heavy = heavy ? 1 : 0;
      desc[it] = d;
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

// Colour sort v2 (world 1), fused with the leaf level (hist, p = 1).  One
// warp per item; colour groups via __match_any_sync (one instruction per 32
// neighbours instead of one ballot per colour); the first 4 x 32 neighbours
// stay in registers between the counting and the placing pass; the next
// item's vertex and range are prefetched one and two items ahead.  Writes the
// colour-sorted list, the 16 cumulative group ends, the item descriptor and
// N''(v, {y}) (heavy segments add their counts atomically into zeroed rows:
// small integers, exact in fp32/fp64).
template <typename T>
__global__ void __launch_bounds__(256, 5) k_csort2(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                                const int32_t *__restrict__ col, const uint8_t *__restrict__ colors,
                                                AggWork work, int k, int32_t *__restrict__ col_out,
                                                uint16_t *__restrict__ goff, ItemDesc *__restrict__ desc,
                                                T *__restrict__ hist, int64_t ldh) {
  constexpr int R = 4;  // neighbour chunks of 32 kept in registers
  __shared__ int cnt_all[8][32];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int *cs = cnt_all[threadIdx.x >> 5];
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t n_items = work.n_seg + work.n_light;
  auto vertex_of = [&](int64_t it) -> int32_t {
    return it < work.n_seg ? work.seg_v[it] : (it < n_items ? work.light[it - work.n_seg] : 0);
  };
  // three-stage prefetch across the warp's items: the vertex of item
  // it + 2 nw, the neighbour range and the first 32 neighbour ids of item
  // it + nw are in flight while item it is sorted (78% of configs[3]'s
  // items have <= 32 neighbours: their sort then starts with the colour
  // loads)
  int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  auto range_of = [&](int64_t i, int32_t vv, int64_t &bb, int64_t &ee) {
    if (i >= n_items) {
      bb = ee = 0;
    } else if (i < work.n_seg) {
      bb = work.seg_b[i];
      ee = work.seg_e[i];
    } else {
      bb = beg[vv];
      ee = end[vv];
    }
  };
  int32_t v_next = vertex_of(it);
  int64_t b_next, e_next;
  range_of(it, v_next, b_next, e_next);
  int32_t u_next = lane < e_next - b_next ? __ldg(col + b_next + lane) : 0;
  int32_t v_next2 = vertex_of(it + nwarps);
  for (; it < n_items; it += nwarps) {
    const int32_t v = v_next;
    const bool heavy = it < work.n_seg;
    const int64_t b = b_next, e = e_next;
    const int cv = colors[v];
    const int32_t u0 = u_next;
    v_next = v_next2;
    range_of(it + nwarps, v_next, b_next, e_next);
    v_next2 = vertex_of(it + 2 * nwarps);
    const int d = (int)(e - b);
    cs[lane] = 0;
    __syncwarp();
    int32_t ur[R];
    int cr[R];
#pragma unroll
    for (int ci = 0; ci < R; ++ci) {
      const bool ok = ci * 32 + lane < d;
      ur[ci] = ok ? (ci == 0 ? u0 : __ldg(col + b + ci * 32 + lane)) : 0;
      cr[ci] = ok ? (int)colors[ur[ci]] : 16 + lane % 16;  // invalid lanes: own groups, never counted
    }
    u_next = lane < e_next - b_next ? __ldg(col + b_next + lane) : 0;  // the next item's first ids
#pragma unroll
    for (int ci = 0; ci < R; ++ci) {
      if (ci * 32 < d) {
        const unsigned m = __match_any_sync(0xffffffffu, cr[ci]);
        if (cr[ci] < 16 && (m & lt) == 0) cs[cr[ci]] += __popc(m);
        __syncwarp();
      }
    }
    for (int o0 = R * 32; o0 < d; o0 += R * 32) {  // long lists: R chunks of loads in flight
      int cq[R];
#pragma unroll
      for (int ci = 0; ci < R; ++ci) {
        const int o = o0 + ci * 32;
        const bool ok = o + lane < d;
        const int32_t u = ok ? __ldg(col + b + o + lane) : 0;
        cq[ci] = ok ? (int)colors[u] : 16 + lane % 16;
      }
#pragma unroll
      for (int ci = 0; ci < R; ++ci) {
        if (o0 + ci * 32 < d) {
          const unsigned m = __match_any_sync(0xffffffffu, cq[ci]);
          if (cq[ci] < 16 && (m & lt) == 0) cs[cq[ci]] += __popc(m);
          __syncwarp();
        }
      }
    }
    const int cnt = lane < 16 ? cs[lane] : 0;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int excl = incl - cnt;
    if (lane < 16) goff[it * 16 + lane] = (uint16_t)incl;
    if (hist && lane < k && lane != cv) {
      T *p = hist + (int64_t)v * ldh + (lane < cv ? lane : lane - 1);  // squeeze: sq_{c_v}(lane)
      if (heavy) atomicAdd(p, (T)cnt);
      else *p = (T)cnt;
    }
    const int skip = __shfl_sync(0xffffffffu, cnt, cv), cv_lo = __shfl_sync(0xffffffffu, excl, cv);
    if (lane == 0) {
      ItemDesc dsc;
      dsc.b = b;
      dsc.v = v;
      dsc.n_s = d - skip;
      dsc.cv_lo = cv_lo;
      dsc.skip = skip;
      dsc.cv = cv;
      dsc.heavy = heavy ? 1 : 0;
      desc[it] = dsc;
    }
    // placing pass: cs[c] = running start of colour c
    __syncwarp();
    if (lane < 16) cs[lane] = excl;
    __syncwarp();
    auto place = [&](int32_t u, int c, bool ok) {
      const unsigned m = __match_any_sync(0xffffffffu, c);
      const int base = ok ? cs[c] : 0;
      __syncwarp();
      if (ok) {
        col_out[b + base + __popc(m & lt)] = u;
        if ((m & lt) == 0) cs[c] = base + __popc(m);
      }
      __syncwarp();
    };
#pragma unroll
    for (int ci = 0; ci < R; ++ci)
      if (ci * 32 < d) place(ur[ci], cr[ci], ci * 32 + lane < d);
    for (int o0 = R * 32; o0 < d; o0 += R * 32) {
      int32_t uq[R];
      int cq[R];
#pragma unroll
      for (int ci = 0; ci < R; ++ci) {
        const int o = o0 + ci * 32;
        const bool ok = o + lane < d;
        uq[ci] = ok ? __ldg(col + b + o + lane) : 0;
        cq[ci] = ok ? (int)colors[uq[ci]] : 16 + lane % 16;
      }
#pragma unroll
      for (int ci = 0; ci < R; ++ci)
        if (o0 + ci * 32 < d) place(uq[ci], cq[ci], o0 + ci * 32 + lane < d);
    }
  }
}

// The tail of light items with <= 8 neighbours (most items of an R-MAT
// graph): 4 items per warp, 8 lanes per item, one neighbour per lane.
// Colour groups via __match_any_sync on (group << 5 | colour); per-colour
// counts and starts in shared memory; the same outputs as k_csort2.
template <typename T>
__global__ void __launch_bounds__(256) k_csort_small(const int64_t *__restrict__ beg, const int64_t *__restrict__ end,
                                                     const int32_t *__restrict__ col,
                                                     const uint8_t *__restrict__ colors, AggWork work, int k,
                                                     int64_t small_from, int32_t *__restrict__ col_out,
                                                     uint16_t *__restrict__ goff, ItemDesc *__restrict__ desc,
                                                     T *__restrict__ hist, int64_t ldh) {
  __shared__ int cnt_all[8][4][16], st_all[8][4][16];
  const int lane = threadIdx.x & 31, g = lane >> 3, sl = lane & 7;
  const unsigned lt = (1u << lane) - 1u;
  int *cs = cnt_all[threadIdx.x >> 5][g], *es = st_all[threadIdx.x >> 5][g];
  const int64_t n_items = work.n_seg + work.n_light;
  const int64_t nslots = (int64_t)gridDim.x * blockDim.x / 8;
  for (int64_t base = small_from + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane) / 8;
       base < n_items; base += nslots) {
    const int64_t it = base + g;  // the 4 items of this warp are consecutive
    const bool live = it < n_items;
    const int32_t v = live ? work.light[it - work.n_seg] : 0;
    const int64_t b = live ? beg[v] : 0;
    const int d = live ? (int)(end[v] - b) : 0;
    const int cv = live ? (int)colors[v] : 0;
    const bool ok = sl < d;
    const int32_t u = ok ? __ldg(col + b + sl) : 0;
    const int c = ok ? (int)colors[u] : 16 + sl;
    const unsigned m = __match_any_sync(0xffffffffu, (g << 5) | c);
    const int rank = __popc(m & lt);
    cs[sl] = 0;
    cs[sl + 8] = 0;
    __syncwarp();
    if (ok && rank == 0) cs[c] = __popc(m);
    __syncwarp();
    const int a0 = cs[2 * sl], a1 = cs[2 * sl + 1];
    int incl = a0 + a1;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o, 8);
      if (sl >= o) incl += t;
    }
    const int e0 = incl - a0 - a1;
    es[2 * sl] = e0;
    es[2 * sl + 1] = e0 + a0;
    if (live) {
      uint32_t *gp = reinterpret_cast<uint32_t *>(goff + it * 16);
      gp[sl] = (uint32_t)(e0 + a0) | ((uint32_t)incl << 16);  // group ends of colours 2 sl, 2 sl + 1
      if (hist) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * sl + h;
          if (j < k && j != cv) hist[(int64_t)v * ldh + (j < cv ? j : j - 1)] = (T)(h ? a1 : a0);
        }
      }
    }
    __syncwarp();
    if (ok) col_out[b + es[c] + rank] = u;
    if (live && sl == 0) {
      ItemDesc dsc;
      dsc.b = b;
      dsc.v = v;
      dsc.skip = cs[cv];
      dsc.n_s = d - dsc.skip;
      dsc.cv_lo = es[cv];
      dsc.cv = cv;
      dsc.heavy = 0;
      desc[it] = dsc;
    }
    __syncwarp();
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

// shared-memory loads / stores of an N'' row entry by its 32-bit shared address
template <typename AccT>
__device__ __forceinline__ AccT lds_acc(uint32_t addr);
template <>
__device__ __forceinline__ float lds_acc<float>(uint32_t addr) {
  float x;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(addr) : "memory");
  return x;
}
template <>
__device__ __forceinline__ double lds_acc<double>(uint32_t addr) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr) : "memory");
  return x;
}
__device__ __forceinline__ void sts_acc_f(uint32_t addr, float x) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(x) : "memory");
}
__device__ __forceinline__ void sts_acc_d(uint32_t addr, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(x) : "memory");
}
template <typename AccT>
__device__ __forceinline__ void sts_acc(uint32_t addr, AccT x) {
  if constexpr (std::is_same<AccT, float>::value) sts_acc_f(addr, x);
  else sts_acc_d(addr, x);
}

// ------------------------------------------------------------------ shared epilogue
// Write the item's N'' row (light vertex) or its partial (heavy segment; the
// last arriving segment of the vertex sums all partials in segment order).
// fp32 shared-memory N'' rows hold value x 2^-64 (an exact power-of-two
// scale): integer counts up to 6e57 stay in range (configs[4]'s root row
// reaches ~1e38 unscaled) and 1 stays a normal number.
template <typename AccT>
struct AccScale {
  static constexpr double in = 1.0, out = 1.0;
};
template <>
struct AccScale<float> {
  static constexpr double in = 0x1p-64, out = 0x1p64;
};

// A block sum into the row's scale.  fp32 block, fp32 row: one FMUL by the
// power of two -- exact, bit-identical to the route through fp64 (two F2F on
// the 16-lane conversion pipe and a DMUL per entry, which made the per-group
// flush of the short-tail launches conversion-bound).
template <typename AccT, typename T>
__device__ __forceinline__ AccT scale_in(T x) {
  if constexpr (std::is_same<AccT, float>::value && std::is_same<T, float>::value) return x * 0x1p-64f;
  else return (AccT)((double)x * AccScale<AccT>::in);
}

template <typename T, int G, typename AccT = double>
__device__ __forceinline__ void gather_epilogue(const GatherArgs &a, const AccT *sacc, int64_t it, int32_t v,
                                                bool heavy, int lane, unsigned gmask) {
  T *drow = static_cast<T *>(a.dst) + (int64_t)v * a.ld_dst;
  // a sibling pair's part 2 goes to its own N'' table (entries o2.. of the virtual row)
  T *drow2 = a.src2 ? static_cast<T *>(a.dst2) + (int64_t)v * a.ld_dst2 - a.o2 : drow;
  if (!heavy) {
    if constexpr (std::is_same<AccT, float>::value && std::is_same<T, float>::value) {
      if (!a.accumulate && !a.src2) {  // fp32 row to fp32 table: the same value without the fp64 round trip
        for (int j = lane; j < a.W_out; j += G) drow[j] = sacc[j] * 0x1p64f;
        return;
      }
    }
    for (int j = lane; j < a.W_out; j += G) {
      T *d = j < a.o2 ? drow + j : drow2 + j;
      double x = (double)sacc[j] * AccScale<AccT>::out;
      if (a.accumulate) x += (double)*d;
      *d = (T)x;
    }
    return;
  }
  double *sp = a.scratch + it * a.ld_scratch;
  for (int j = lane; j < a.W_out; j += G) sp[j] = (double)sacc[j] * AccScale<AccT>::out;
  __threadfence();
  __syncwarp(gmask);
  const int32_t hv = a.work.seg_hv[it];
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(&a.arrive[hv], 1u);
  prev = __shfl_sync(gmask, prev, 0, G);
  if (prev == (unsigned)(a.work.hv_nseg[hv] - 1)) {
    __threadfence();
    const int32_t s0 = a.work.hv_first[hv], ns = a.work.hv_nseg[hv];
    for (int j = lane; j < a.W_out; j += G) {
      T *d = j < a.o2 ? drow + j : drow2 + j;
      double x = 0.0;
      for (int s = 0; s < ns; ++s) x += __ldcg(a.scratch + (int64_t)(s0 + s) * a.ld_scratch + j);
      if (a.accumulate) x += (double)*d;
      *d = (T)x;
    }
  }
}

// Sibling pair: row base / stride of virtual 16-byte vector q and whether it
// holds columns of its part (ring kernel: no sector skip).
template <typename T, int VW>
__device__ __forceinline__ bool pair_base(const GatherArgs &a, int q, const char *&base, uint32_t &ld_bytes) {
  const bool second = q >= a.nvec1;
  const int qq = second ? q - a.nvec1 : q;
  base = static_cast<const char *>(second ? a.src2 : a.src) + (size_t)qq * 16;
  ld_bytes = (uint32_t)((second ? a.ld_src2 : a.ld_src) * sizeof(T));
  return qq * VW < (second ? a.W_in2 : a.nvec1 * VW);
}
// Sibling pair: the colour-pair map entries of virtual vector q as virtual N'' indices.
template <int VW>
__device__ __forceinline__ void pair_map(const GatherArgs &a, int q, int cu, int cv, uint16_t (&m)[VW]) {
  const bool second = q >= a.nvec1;
  const int qq = second ? q - a.nvec1 : q;
#pragma unroll
  for (int i = 0; i < VW; ++i) m[i] = 0xFFFF;
  if (qq * VW >= (second ? a.W_in2 : a.nvec1 * VW)) return;
  const uint16_t *mrow = second ? a.map2 + (int64_t)(cu * a.k + cv) * a.map_ld2 : a.map + (int64_t)(cu * a.k + cv) * a.map_ld;
  if constexpr (VW == 4) {
    const uint2 w = __ldg(reinterpret_cast<const uint2 *>(mrow + qq * VW));
    m[0] = w.x & 0xFFFF;
    m[1 % VW] = w.x >> 16;
    m[2 % VW] = w.y & 0xFFFF;
    m[3 % VW] = w.y >> 16;
  } else {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(mrow + qq * VW));
    m[0] = w & 0xFFFF;
    m[1 % VW] = w >> 16;
  }
  const int off = second ? a.o2 : 0;
#pragma unroll
  for (int i = 0; i < VW; ++i)
    if (m[i] != 0xFFFF) m[i] = (uint16_t)(m[i] + off);
}

// Sibling pair: the part of virtual 16-byte vector q (a lane's vector of the
// pass), its row base and stride, whether the destination colour can use it
// (sector skip) and its colour-pair map entries as virtual N'' indices.
template <typename T, int VW>
__device__ __forceinline__ void pair_vector(const GatherArgs &a, int q, int cu, int cv, const char *&base,
                                            uint32_t &ld_bytes, bool &use, uint16_t (&m)[VW]) {
  use = pair_base<T, VW>(a, q, base, ld_bytes);
  const bool second = q >= a.nvec1;
  const uint32_t *sk = second ? a.skip2 : a.skip;
  if (sk && use) {
    const int qq = second ? q - a.nvec1 : q;
    const int cvu = cv < cu ? cv : cv - 1;  // sq_{c_u}(c_v)
    use = !((__ldg(sk + (int64_t)cvu * (second ? a.skip_words2 : a.skip_words) + (qq >> 5)) >> (qq & 31)) & 1u);
  }
  pair_map<VW>(a, q, cu, cv, m);
}

// Fused root epilogue (root_mode 1 / 2): X_v = sum_{X'} A'(v, X') N''(v, comp X')
// in fp64, written to per_vertex[v]; a heavy vertex's segments are first
// summed (in segment order) by the last arriving segment.
template <typename T, typename AccT = double>
__device__ __forceinline__ void root_epilogue(const GatherArgs &a, AccT *sacc, int64_t it, int32_t v, bool heavy,
                                              int lane) {
  if (heavy) {
    double *sp = a.scratch + it * a.ld_scratch;
    for (int j = lane; j < a.W_out; j += 32) sp[j] = (double)sacc[j] * AccScale<AccT>::out;
    __threadfence();
    __syncwarp();
    const int32_t hv = a.work.seg_hv[it];
    unsigned prev = 0;
    if (lane == 0) prev = atomicAdd(&a.arrive[hv], 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != (unsigned)(a.work.hv_nseg[hv] - 1)) return;
    __threadfence();
    const int32_t s0 = a.work.hv_first[hv], ns = a.work.hv_nseg[hv];
    for (int j = lane; j < a.W_out; j += 32) {
      double x = 0.0;
      for (int s = 0; s < ns; ++s) x += __ldcg(a.scratch + (int64_t)(s0 + s) * a.ld_scratch + j);
      sacc[j] = (AccT)(x * AccScale<AccT>::in);
    }
    __syncwarp();
  }
  double d = 0.0;
  if (a.root_mode == 2) {
    for (int x = lane; x < a.WA; x += 32)
      d += ((double)sacc[x] * AccScale<AccT>::out) * ((double)sacc[__ldg(a.comp + x)] * AccScale<AccT>::out);
  } else {
    const T *ar = static_cast<const T *>(a.rA) + (int64_t)v * a.ldA;
    for (int x = lane; x < a.WA; x += 32) d += (double)ar[x] * ((double)sacc[__ldg(a.comp + x)] * AccScale<AccT>::out);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if (lane == 0) a.per_vertex[v] = d;
}

// expand with the group's colour-pair map already in registers (packed
// 16-bit entries, loaded when the group opened, so that its latency hides
// behind the group's rows); rings of G <= 8 lanes send 0xFFFF entries to the
// discard slot sacc[W_out] (all loads before the stores), G = 32 branches
template <int NV, int VW, int G, typename AccT = double>
__device__ __forceinline__ void expand_map(const GatherArgs &a, const uint32_t (&mp)[NV][2], AccT (&acc)[NV][VW],
                                           AccT *sacc, uint32_t sacc_sh) {
  if constexpr (G <= 8) {
    const uint32_t discard = (uint32_t)a.W_out;
    uint32_t d[NV][VW];  // shared addresses from the row's (opaque) base: no per-entry rematerialisation
    AccT old[NV][VW];
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        d[j][q] = sacc_sh + (uint32_t)sizeof(AccT) * min((mp[j][q >> 1] >> (16 * (q & 1))) & 0xFFFFu, discard);
        old[j][q] = lds_acc<AccT>(d[j][q]);
      }
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        sts_acc<AccT>(d[j][q], old[j][q] + acc[j][q]);
        acc[j][q] = (AccT)0;
      }
  } else {
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int q = 0; q < VW; ++q) {
        const uint32_t m = (mp[j][q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
        if (m != 0xFFFFu) sacc[m] += acc[j][q];
        acc[j][q] = (AccT)0;
      }
  }
}
// the group's map entries for the lane's vectors (0xFFFF past the row end)
template <int NV, int VW, int G>
__device__ __forceinline__ void load_map(const GatherArgs &a, int cu, int cv, int c0, uint32_t (&mp)[NV][2]) {
  const uint16_t *mrow = a.map + (int64_t)(cu * a.k + cv) * a.map_ld + a.col_base;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int y0 = c0 + j * G * VW;
    mp[j][0] = mp[j][1] = 0xFFFFFFFFu;
    if (y0 < a.W_in) {
      if constexpr (VW == 4) {
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(mrow + y0));
        mp[j][0] = w.x;
        mp[j][1] = w.y;
      } else {
        mp[j][0] = __ldg(reinterpret_cast<const uint32_t *>(mrow + y0));
      }
    }
  }
}

// the same for a sibling pair (virtual vectors lane + j G)
template <int NV, int VW, int G>
__device__ __forceinline__ void expand_pair(const GatherArgs &a, int cu, int cv, int lane, double (&acc)[NV][VW],
                                            double *sacc) {
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    uint16_t m[VW];
    pair_map<VW>(a, lane + j * G, cu, cv, m);
#pragma unroll
    for (int q = 0; q < VW; ++q) {
      if (m[q] != 0xFFFF) sacc[m[q]] += acc[j][q];
      acc[j][q] = 0.0;
    }
  }
}

// ------------------------------------------------------------------ gather, cp.async ring
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes, uint64_t policy) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes), "l"(policy)
               : "memory");
}
// L2 policies: hub rows (the most re-gathered; internal ids are degree-ordered,
// so they are the lowest row ids) are kept, all other rows stream through.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// fp32 rows are summed in blocks of up to 8 consecutive rows in fp32 and the
// blocks in fp64 (relative error <= 7 u32 + O(n u64) per entry; DESIGN.md
// reading C-6); fp64 rows are summed in fp64.
// AccT = float (fp32 tables, launches whose items have <= 1024 neighbours):
// the blocks are added in fp32, scaled by 2^-64, and the N'' row is kept in
// fp32 as in the lean gather -- at most ceil(1024 / 8) + k - 1 fp32 additions
// per entry (C-6), no fp64 conversions or additions in the loop.
template <typename T, int G, int NV, int D, int MINB, bool PAIR = false, typename AccT = double>
__global__ void __launch_bounds__(256, MINB) k_gather_ring(GatherArgs a, int nch) {
  static_assert(std::is_same<AccT, double>::value || (!PAIR && sizeof(T) == 4), "fp32 rows: unpaired fp32 tables");
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = G * NV * VW;  // input columns per pass
  constexpr int BLK = 8;            // fp32 block length
  extern __shared__ __align__(16) unsigned char smem_ring[];
  const int lane = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  const unsigned gmask = group_mask<G>();
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int64_t n_items = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
  const int groups_per_block = blockDim.x / G;
  V *ring = reinterpret_cast<V *>(smem_ring) + (int64_t)grp * D * NV * G;  // [D][NV][G]
  AccT *sacc = reinterpret_cast<AccT *>(reinterpret_cast<V *>(smem_ring) + (int64_t)groups_per_block * D * NV * G) +
               (int64_t)grp * (a.W_out + 1);  // + the discard slot
  const T *__restrict__ src = static_cast<const T *>(a.src);
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  uint32_t sacc_sh = (uint32_t)__cvta_generic_to_shared(sacc);
  asm volatile("mov.u32 %0, %0;" : "+r"(sacc_sh));

  for (int64_t it = a.item_from + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; it < n_items;
       it += ngroups) {
    // the item's descriptor (one 32-byte load): first neighbour position,
    // vertex, stream length (the neighbours minus v's own colour group),
    // that group's start and size, v's colour, heavy segment or not
    const int4 dx = __ldg(reinterpret_cast<const int4 *>(a.desc + it));
    const int4 dy = __ldg(reinterpret_cast<const int4 *>(a.desc + it) + 1);
    const int64_t b = (int64_t)(((uint64_t)(uint32_t)dx.y << 32) | (uint32_t)dx.x);
    const int32_t v = dx.z;
    const int n_s = dx.w, cv_lo = dy.x, skip = dy.y, cv = dy.z;
    const bool heavy = dy.w != 0;
    for (int j = lane; j < a.W_out; j += G) sacc[j] = (AccT)0;
    __syncwarp(gmask);
    const uint16_t *go = a.goff + it * 16;
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * CAP + lane * VW;
      int nbytes[NV];
      const char *jb[NV];  // sibling pair: per-vector row base and stride
      uint32_t jld[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        if constexpr (PAIR) nbytes[j] = pair_base<T, VW>(a, lane + j * G, jb[j], jld[j]) ? 16 : 0;
        else nbytes[j] = c0 + j * G * VW < a.W_in ? 16 : 0;
      }
      // neighbour ids: a window of G stream positions per lane, one window ahead
      auto load_idx = [&](int r) -> int32_t {
        return r < n_s ? __ldg(a.col + b + (r < cv_lo ? r : r + skip)) : 0;
      };
      int win = 0;
      int32_t idx_cur = load_idx(lane), idx_nxt = load_idx(G + lane);
      auto issue = [&](int r) {
        if (r >= win + G) {
          win += G;
          idx_cur = idx_nxt;
          idx_nxt = load_idx(win + G + lane);
        }
        const int32_t u = __shfl_sync(gmask, idx_cur, r - win, G);
        if (r < n_s) {
          V *slot = ring + (r % D) * NV * G + lane;
          const uint64_t pol = u < a.hub_rows ? pol_keep : pol_stream;
          if constexpr (PAIR) {
#pragma unroll
            for (int j = 0; j < NV; ++j)
              cp_async16(slot + j * G, nbytes[j] ? jb[j] + (uint64_t)u * jld[j] : jb[0] + (uint64_t)u * jld[0],
                         nbytes[j], pol);
          } else {
            const T *row = src + (int64_t)u * a.ld_src + c0;
#pragma unroll
            for (int j = 0; j < NV; ++j)
              cp_async16(slot + j * G, nbytes[j] ? row + j * G * VW : row, nbytes[j], pol);
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int r = 0; r < D - 1; ++r) issue(r);
      // current colour group (stream coordinates): the non-empty groups
      // other than v's own as a bit mask from the item's 16 group ends (two
      // 16-byte loads), so that the walk skips empty colours without loads
      int gc = 0, gend_s = -1;
      unsigned gleft = 0;
      {
        const uint4 ga = __ldg(reinterpret_cast<const uint4 *>(go)), gb = __ldg(reinterpret_cast<const uint4 *>(go) + 1);
        const uint32_t gw[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        int prev = 0;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int hi = (int)((gw[c >> 1] >> (16 * (c & 1))) & 0xFFFFu);
          if (c < a.k && c != cv && hi > prev) gleft |= 1u << c;
          prev = hi;
        }
      }
      uint32_t mp[NV][2];  // the open group's colour-pair map (non-pair rings)
      auto next_group = [&]() {
        if (!gleft) {
          gc = a.k;
          gend_s = -1;
          return;
        }
        gc = __ffs(gleft) - 1;
        gleft &= gleft - 1;
        gend_s = (int)go[gc] - (gc > cv ? skip : 0);
        if constexpr (!PAIR) load_map<NV, VW, G>(a, gc, cv, c0, mp);
      };
      next_group();
      AccT acc[NV][VW];
#pragma unroll
      for (int j = 0; j < NV; ++j)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[j][q] = (AccT)0;
      float4 blk[NV];
      int nb = 0;
#pragma unroll
      for (int j = 0; j < NV; ++j) blk[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = 0; i < n_s; ++i) {
        issue(i + D - 1);
        cp_async_wait<D - 1>();
        const V *slot = ring + (i % D) * NV * G + lane;
        if constexpr (VW == 4) {  // fp32 storage: fp32 blocks of BLK rows
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const float4 x = reinterpret_cast<const float4 *>(slot)[j * G];
            blk[j].x += x.x;
            blk[j].y += x.y;
            blk[j].z += x.z;
            blk[j].w += x.w;
          }
          const bool gend = i + 1 == gend_s;
          if (++nb == BLK || gend) {
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              if constexpr (std::is_same<AccT, float>::value) {
                acc[j][0] = fmaf(blk[j].x, 0x1p-64f, acc[j][0]);
                acc[j][1] = fmaf(blk[j].y, 0x1p-64f, acc[j][1]);
                acc[j][2] = fmaf(blk[j].z, 0x1p-64f, acc[j][2]);
                acc[j][3] = fmaf(blk[j].w, 0x1p-64f, acc[j][3]);
              } else {
                add_vec(acc[j], blk[j]);
              }
              blk[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            nb = 0;
          }
        } else {
#pragma unroll
          for (int j = 0; j < NV; ++j)
            if constexpr (std::is_same<AccT, double>::value) add_vec(acc[j], slot[j * G]);
        }
        if (i + 1 == gend_s) {  // end of a colour group: expand into N''
          if constexpr (PAIR) expand_pair<NV, VW, G>(a, gc, cv, lane, acc, sacc);
          else expand_map<NV, VW, G, AccT>(a, mp, acc, sacc, sacc_sh);
          __syncwarp(gmask);
          next_group();
        }
      }
      cp_async_wait<0>();
      __syncwarp(gmask);
    }
    gather_epilogue<T, G, AccT>(a, sacc, it, v, heavy, lane, gmask);
    __syncwarp(gmask);
  }
}

// ------------------------------------------------------------------ gather, lean register rows
// One warp per item; lane l owns the 16-byte column vectors l, l+32, ... of
// the pass.  The item's colour groups are contiguous in the colour-sorted
// neighbour list (goff), so a group's rows are read from positions
// [b + lo_g, b + hi_g) directly: 32 neighbour ids per coalesced load, then U
// rows in flight per lane (U x NV independent LDG.128), summed in the storage
// type over chunks of <= 32 rows and expanded into the fp64 N'' row in shared
// memory through the colour-pair map (held in registers for the group).  The
// next item's descriptor and group ends are loaded while the current item
// runs.  Per row: one SHFL, one address, NV loads and 4 NV (fp32) adds.
__device__ __forceinline__ void load_desc(const GatherArgs &a, int64_t it, int lane, int4 &x, int4 &y, int &go) {
  const int4 *d = reinterpret_cast<const int4 *>(a.desc + it);
  x = __ldg(d);
  y = __ldg(d + 1);
  go = lane < 16 ? (int)__ldg(a.goff + it * 16 + lane) : 0;
}

template <typename T, int NV, int U, typename AccT = double, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_gather_ldg(GatherArgs a, int nch) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = 32 * NV * VW;  // columns per pass
  extern __shared__ __align__(16) unsigned char sacc_raw[];
  const int lane = threadIdx.x & 31;
  // the warp's N'' row, plus a discard slot (index W_out) that takes the
  // map's 0xFFFF entries, so that the block flush needs no branches
  AccT *sacc = reinterpret_cast<AccT *>(sacc_raw) + (threadIdx.x >> 5) * (int64_t)(a.W_out + 1);
  const uint32_t discard = (uint32_t)a.W_out;
  // the row's shared-memory address, opaque to the compiler: under the 80-register
  // cap of the short-tail launches it was rematerialised (S2R, shift, IMAD) for
  // every entry of every flush
  uint32_t sacc_sh = (uint32_t)__cvta_generic_to_shared(sacc);
  asm volatile("mov.u32 %0, %0;" : "+r"(sacc_sh));
  const bool noskip = !a.skip;
  const int64_t n_items = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const char *__restrict__ srcb = static_cast<const char *>(a.src);
  const uint32_t ld_bytes = (uint32_t)(a.ld_src * sizeof(T));
  // (L2 evict-last hints for hub rows measured neutral here: plain loads)

  int64_t it = a.item_from + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int4 dx = make_int4(0, 0, 0, 0), dy = make_int4(0, 0, 0, 0);
  int go_n = 0;
  if (it < n_items) load_desc(a, it, lane, dx, dy, go_n);
  for (; it < n_items; it += nw) {
    const int64_t b = (int64_t)(((uint64_t)(uint32_t)dx.y << 32) | (uint32_t)dx.x);
    const int32_t v = dx.z;
    const int cv = dy.z;
    const bool heavy = dy.w != 0;
    const int hi_l = go_n;
    const int lo_l = __shfl_up_sync(0xffffffffu, hi_l, 1);
    // non-empty colour groups other than v's own
    unsigned gm = __ballot_sync(0xffffffffu, lane < a.k && lane != cv && hi_l > (lane == 0 ? 0 : lo_l));
    if (it + nw < n_items) load_desc(a, it + nw, lane, dx, dy, go_n);  // prefetch the next item
    for (int j = lane; j < a.W_out; j += 32) sacc[j] = 0.0;
    __syncwarp();
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * CAP + lane * VW;
      // lanes past the row end of slot j skip that load (map entries 0xFFFF)
      bool valid[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) valid[j] = c0 + j * 32 * VW < a.W_in;
      // (opaque: otherwise rematerialised from the thread id for every row under the register cap)
      uint64_t lbase_u = reinterpret_cast<uint64_t>(srcb + (size_t)c0 * sizeof(T));
      asm volatile("mov.u64 %0, %0;" : "+l"(lbase_u));
      const char *lbase = reinterpret_cast<const char *>(lbase_u);
      for (unsigned g = gm; g; g &= g - 1) {
        const int cu = __ffs(g) - 1;
        const int lo = cu == 0 ? 0 : __shfl_sync(0xffffffffu, hi_l, cu - 1);
        const int hi = __shfl_sync(0xffffffffu, hi_l, cu);
        int32_t u_next = lane < hi - lo ? __ldg(a.col + b + lo + lane) : 0;
        // colour-pair map of this group for the lane's columns (16-bit
        // entries, packed in pairs).  A vector whose entries are all 0xFFFF
        // holds only colour sets that contain v's colour (in u's universe):
        // never used by v, not read (sector skipping at 16-byte granularity;
        // knob sector_skip = 0 reads every vector)
        uint32_t mp[NV][VW / 2];
        bool use[NV];
        const uint16_t *mrow = a.map + (int64_t)(cu * a.k + cv) * a.map_ld + a.col_base;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (valid[j]) {
            if constexpr (VW == 4) {
              const uint2 w = __ldg(reinterpret_cast<const uint2 *>(mrow + c0 + j * 32 * VW));
              mp[j][0] = w.x;
              mp[j][1 % (VW / 2)] = w.y;
            } else {
              mp[j][0] = __ldg(reinterpret_cast<const uint32_t *>(mrow + c0 + j * 32 * VW));
            }
          } else {
#pragma unroll
            for (int q = 0; q < VW / 2; ++q) mp[j][q] = 0xFFFFFFFFu;
          }
          bool live = false;
#pragma unroll
          for (int q = 0; q < VW / 2; ++q) live |= mp[j][q] != 0xFFFFFFFFu;
          use[j] = valid[j] && (live || noskip);
        }
        for (int p = lo; p < hi; p += 32) {
          const int cnt = min(32, hi - p);
          const int32_t my_u = u_next;
          if (p + 32 < hi) u_next = p + 32 + lane < hi ? __ldg(a.col + b + p + 32 + lane) : 0;  // next chunk's ids
          V blk[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) zero_vec(blk[j]);
          int r = 0;
          V x[U][NV];
#pragma unroll
          for (int uu = 0; uu < U; ++uu)
#pragma unroll
            for (int j = 0; j < NV; ++j) zero_vec(x[uu][j]);
          for (; r + U <= cnt; r += U) {  // full blocks of U rows: no row predicates
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
              const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, my_u, r + uu);
              const V *row = reinterpret_cast<const V *>(lbase + (uint64_t)u * ld_bytes);
#pragma unroll
              for (int j = 0; j < NV; ++j)
                if (use[j]) x[uu][j] = __ldg(row + 32 * j);
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
#pragma unroll
              for (int j = 0; j < NV; ++j) add_same(blk[j], x[uu][j]);
          }
          if constexpr (U == 2) {
            if (r < cnt) {  // tail: exactly one row
              const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, my_u, r);
              const V *row = reinterpret_cast<const V *>(lbase + (uint64_t)u * ld_bytes);
#pragma unroll
              for (int j = 0; j < NV; ++j)
                if (use[j]) x[0][j] = __ldg(row + 32 * j);
#pragma unroll
              for (int j = 0; j < NV; ++j) add_same(blk[j], x[0][j]);
            }
          } else if (r < cnt) {  // tail
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
              const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, my_u, (r + uu) & 31);
              const V *row = reinterpret_cast<const V *>(lbase + (uint64_t)u * ld_bytes);
#pragma unroll
              for (int j = 0; j < NV; ++j) {
                if (r + uu < cnt && use[j]) x[uu][j] = __ldg(row + 32 * j);
                else zero_vec(x[uu][j]);
              }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
#pragma unroll
              for (int j = 0; j < NV; ++j) add_same(blk[j], x[uu][j]);
          }
          // fp32: a block of <= 32 rows summed in fp32, then added into the
          // N'' row (C-6); 0xFFFF entries land in the discard slot.
          // All loads first, then all stores: the map is injective per colour
          // pair, so only discarded entries can alias
          // (the map words are pinned here so that the 4 NV entry addresses are
          // computed after the row loops instead of living across them)
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW / 2; ++q) asm volatile("" : "+r"(mp[j][q]));
          uint32_t d[NV][VW];
          AccT old[NV][VW];
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) {
              d[j][q] = sacc_sh + (uint32_t)sizeof(AccT) * min((mp[j][q >> 1] >> (16 * (q & 1))) & 0xFFFFu, discard);
              old[j][q] = lds_acc<AccT>(d[j][q]);
            }
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) sts_acc<AccT>(d[j][q], old[j][q] + scale_in<AccT>(vec_at(blk[j], q)));
        }
        __syncwarp();  // groups of different colours may map to the same N'' entries
      }
    }
    if (a.root_mode) root_epilogue<T, AccT>(a, sacc, it, v, heavy, lane);
    else gather_epilogue<T, 32, AccT>(a, sacc, it, v, heavy, lane, 0xffffffffu);
    __syncwarp();
  }
}

// ------------------------------------------------------------------ gather, narrow rows
// Rows of <= 16 vectors: one warp per item as in k_gather_ldg (no divergence
// between items), but a row is covered by G lanes, so one warp-wide load
// instruction reads RG = 32 / G rows of the same colour group (lane = row
// slot rs x column vector vl); U such loads per lane in flight.  At the end
// of a chunk of <= 32 rows the RG slot sums are combined by XOR shuffles
// (fp32 block of <= 32 rows, then fp64: DESIGN.md C-6) and expanded into the
// fp64 N'' row through the colour-pair map, vector j by slot j mod RG.
template <typename T, int G, int NV, int U, int MINB = 2, typename AccT = double, bool PAIR = false>
__global__ void __launch_bounds__(256, MINB) k_gather_rows(GatherArgs a, int nch) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr int RG = 32 / G;
  constexpr int CAP = G * NV * VW;  // columns per pass
  extern __shared__ __align__(16) unsigned char sacc_raw[];
  const int lane = threadIdx.x & 31, vl = lane % G, rs = lane / G;
  AccT *sacc = reinterpret_cast<AccT *>(sacc_raw) + (threadIdx.x >> 5) * (int64_t)(a.W_out + 1);  // + discard slot
  const uint32_t discard = (uint32_t)a.W_out;
  // (opaque registers for the row's shared address and the lane's row base, as in k_gather_ldg)
  uint32_t sacc_sh = (uint32_t)__cvta_generic_to_shared(sacc);
  asm volatile("mov.u32 %0, %0;" : "+r"(sacc_sh));
  const bool noskip = !a.skip;
  const int64_t n_items = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const char *__restrict__ srcb = static_cast<const char *>(a.src);
  const uint32_t ld_bytes = (uint32_t)(a.ld_src * sizeof(T));

  int64_t it = a.item_from + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int4 dx = make_int4(0, 0, 0, 0), dy = make_int4(0, 0, 0, 0);
  int go_n = 0;
  if (it < n_items) load_desc(a, it, lane, dx, dy, go_n);
  for (; it < n_items; it += nw) {
    const int64_t b = (int64_t)(((uint64_t)(uint32_t)dx.y << 32) | (uint32_t)dx.x);
    const int32_t v = dx.z;
    const int cv = dy.z;
    const bool heavy = dy.w != 0;
    const int hi_l = go_n;
    const int lo_l = __shfl_up_sync(0xffffffffu, hi_l, 1);
    const unsigned gm = __ballot_sync(0xffffffffu, lane < a.k && lane != cv && hi_l > (lane == 0 ? 0 : lo_l));
    if (it + nw < n_items) load_desc(a, it + nw, lane, dx, dy, go_n);  // prefetch the next item
    for (int j = lane; j < a.W_out; j += 32) sacc[j] = 0.0;
    __syncwarp();
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * CAP + vl * VW;
      bool valid[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) valid[j] = c0 + j * G * VW < a.W_in;
      uint64_t lbase_u = reinterpret_cast<uint64_t>(srcb + (size_t)c0 * sizeof(T));
      asm volatile("mov.u64 %0, %0;" : "+l"(lbase_u));
      const char *lbase = reinterpret_cast<const char *>(lbase_u);
      for (unsigned g = gm; g; g &= g - 1) {
        const int cu = __ffs(g) - 1;
        const int lo = cu == 0 ? 0 : __shfl_sync(0xffffffffu, hi_l, cu - 1);
        const int hi = __shfl_sync(0xffffffffu, hi_l, cu);
        bool use[NV];
        uint16_t m[NV][VW];
        uint32_t mw[NV][2];  // unpaired: the packed map words (entries taken at the flush)
        // sibling pair: per-vector row base and stride (part 1 or part 2)
        const char *jb[NV];
        uint32_t jld[NV];
        if constexpr (PAIR) {
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            uint16_t mm[VW];
            pair_vector<T, VW>(a, vl + j * G, cu, cv, jb[j], jld[j], use[j], mm);
#pragma unroll
            for (int q = 0; q < VW; ++q) m[j][q] = rs == j % RG ? mm[q] : (uint16_t)0xFFFF;
          }
        } else {
          // every lane loads its vectors' map entries (lanes of one vector
          // share the address); a vector whose entries are all 0xFFFF holds
          // only colour sets containing v's colour: not read (16-byte sector
          // skipping; knob sector_skip = 0 reads it).  Only the row slot
          // rs == j mod RG adds vector j into N'' (the others: discard slot)
          const uint16_t *mrow = a.map + (int64_t)(cu * a.k + cv) * a.map_ld + a.col_base;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            jb[j] = lbase + (size_t)j * G * 16;
            jld[j] = ld_bytes;
            uint32_t w0 = 0xFFFFFFFFu, w1 = 0xFFFFFFFFu;
            if (valid[j]) {
              if constexpr (VW == 4) {
                const uint2 w = __ldg(reinterpret_cast<const uint2 *>(mrow + c0 + j * G * VW));
                w0 = w.x;
                w1 = w.y;
              } else {
                w0 = __ldg(reinterpret_cast<const uint32_t *>(mrow + c0 + j * G * VW));
              }
            }
            use[j] = valid[j] && (noskip || w0 != 0xFFFFFFFFu || w1 != 0xFFFFFFFFu);
            mw[j][0] = w0;
            mw[j][1] = w1;
          }
        }
        int32_t u_next = lane < hi - lo ? __ldg(a.col + b + lo + lane) : 0;
        for (int p = lo; p < hi; p += 32) {
          const int cnt = min(32, hi - p);
          const int32_t my_u = u_next;
          if (p + 32 < hi) u_next = p + 32 + lane < hi ? __ldg(a.col + b + p + 32 + lane) : 0;
          V blk[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) zero_vec(blk[j]);
          for (int r = 0; r < cnt; r += RG * U) {
            V x[U][NV];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
              const int rr = r + uu * RG + rs;
              const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, my_u, rr & 31);
              if constexpr (PAIR) {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                  if (rr < cnt && use[j]) x[uu][j] = __ldg(reinterpret_cast<const V *>(jb[j] + (uint64_t)u * jld[j]));
                  else zero_vec(x[uu][j]);
                }
              } else {
                const V *row = reinterpret_cast<const V *>(lbase + (uint64_t)u * ld_bytes);
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                  if (rr < cnt && use[j]) x[uu][j] = __ldg(row + G * j);
                  else zero_vec(x[uu][j]);
                }
              }
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu)
#pragma unroll
              for (int j = 0; j < NV; ++j) add_same(blk[j], x[uu][j]);
          }
          // the RG row slots' sums
#pragma unroll
          for (int off = G; off < 32; off <<= 1)
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              V o;
              if constexpr (VW == 4) {
                o.x = __shfl_xor_sync(0xffffffffu, blk[j].x, off);
                o.y = __shfl_xor_sync(0xffffffffu, blk[j].y, off);
                o.z = __shfl_xor_sync(0xffffffffu, blk[j].z, off);
                o.w = __shfl_xor_sync(0xffffffffu, blk[j].w, off);
              } else {
                o.x = __shfl_xor_sync(0xffffffffu, blk[j].x, off);
                o.y = __shfl_xor_sync(0xffffffffu, blk[j].y, off);
              }
              add_same(blk[j], o);
            }
          // into N'' (0xFFFF: the discard slot; all loads before the stores)
          uint32_t d[NV][VW];
          AccT old[NV][VW];
          if constexpr (!PAIR) {  // (pinned: the entry addresses are computed here, not held across the loads)
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              asm volatile("" : "+r"(mw[j][0]));
              asm volatile("" : "+r"(mw[j][1]));
            }
          }
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) {
              uint32_t idx;
              if constexpr (PAIR) idx = min((uint32_t)m[j][q], discard);
              else idx = rs == j % RG ? min((mw[j][q >> 1] >> (16 * (q & 1))) & 0xFFFFu, discard) : discard;
              d[j][q] = sacc_sh + (uint32_t)sizeof(AccT) * idx;
              old[j][q] = lds_acc<AccT>(d[j][q]);
            }
#pragma unroll
          for (int j = 0; j < NV; ++j)
#pragma unroll
            for (int q = 0; q < VW; ++q) sts_acc<AccT>(d[j][q], old[j][q] + scale_in<AccT>(vec_at(blk[j], q)));
        }
        __syncwarp();  // groups of different colours may map to the same N'' entries
      }
    }
    gather_epilogue<T, 32, AccT>(a, sacc, it, v, heavy, lane, 0xffffffffu);
    __syncwarp();
  }
}

// ------------------------------------------------------------------ gather, wide rows, short lists
// The items with <= 32 neighbours (most items of an R-MAT graph; measured:
// 78% of configs[3]'s items, 14.7 of the p = 5 gather's 69 ms for 7% of its
// DRAM bytes): the lean kernel waits for every colour group in turn (its ids,
// then its rows), several dependent round trips per item.  Here a warp
// loads the whole stream's ids at once (one coalesced load; <= 32 rows), then
// issues the rows B at a time ACROSS colour-group boundaries and walks them
// in order, expanding a group's sum into N'' when the colour changes.  Same
// sums in the same order as the lean kernel (fp32 blocks of one colour group,
// then the N'' row); no sector skipping (whole rows).
template <typename T, int NV, int B, typename AccT>
__global__ void __launch_bounds__(128) k_gather_short(GatherArgs a, int nch) {
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = 32 * NV * VW;  // columns per pass
  extern __shared__ __align__(16) unsigned char sacc_raw[];
  const int lane = threadIdx.x & 31;
  AccT *sacc = reinterpret_cast<AccT *>(sacc_raw) + (threadIdx.x >> 5) * (int64_t)a.W_out;
  const int64_t n_items = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const char *__restrict__ srcb = static_cast<const char *>(a.src);
  const uint32_t ld_bytes = (uint32_t)(a.ld_src * sizeof(T));

  int64_t it = a.item_from + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int4 dx = make_int4(0, 0, 0, 0), dy = make_int4(0, 0, 0, 0);
  int go_n = 0;
  if (it < n_items) load_desc(a, it, lane, dx, dy, go_n);
  for (; it < n_items; it += nw) {
    const int64_t b = (int64_t)(((uint64_t)(uint32_t)dx.y << 32) | (uint32_t)dx.x);
    const int32_t v = dx.z;
    const int n_s = dx.w, cv_lo = dy.x, skip = dy.y, cv = dy.z;
    const int go = go_n;  // lane j < 16: end of colour group j (item positions)
    if (it + nw < n_items) load_desc(a, it + nw, lane, dx, dy, go_n);  // prefetch the next item
    // the stream (the item's neighbours minus v's own colour group): ids and colours, one lane each
    const int ip = lane < cv_lo ? lane : lane + skip;  // item position of stream position lane
    const int32_t my_u = lane < n_s ? __ldg(a.col + b + ip) : 0;
    int my_cu = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) my_cu += (j < a.k) && (__shfl_sync(0xffffffffu, go, j) <= ip);
    for (int j = lane; j < a.W_out; j += 32) sacc[j] = (AccT)0;
    __syncwarp();
    for (int ch = 0; ch < nch; ++ch) {
      const int c0 = ch * CAP + lane * VW;
      bool valid[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) valid[j] = c0 + j * 32 * VW < a.W_in;
      const char *lbase = srcb + (size_t)c0 * sizeof(T);
      int cur = -1;
      uint16_t m[NV][VW];
      V blk[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) zero_vec(blk[j]);
      auto flush = [&]() {  // the colour group's block sum into N'' (fp32 block, then the N'' row)
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const double e[4] = {(double)vec_at(blk[j], 0), (double)vec_at(blk[j], 1), (double)vec_at(blk[j], 2 % VW),
                               (double)vec_at(blk[j], 3 % VW)};
#pragma unroll
          for (int q = 0; q < VW; ++q)
            if (m[j][q] != 0xFFFF) sacc[m[j][q]] += (AccT)(e[q] * AccScale<AccT>::in);
          zero_vec(blk[j]);
        }
      };
      for (int r0 = 0; r0 < n_s; r0 += B) {
        V x[B][NV];
#pragma unroll
        for (int bb = 0; bb < B; ++bb) {  // B rows in flight, whatever their colour groups
          const int r = r0 + bb;
          const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, my_u, r & 31);
          const V *row = reinterpret_cast<const V *>(lbase + (uint64_t)u * ld_bytes);
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            if (r < n_s && valid[j]) x[bb][j] = __ldg(row + 32 * j);
            else zero_vec(x[bb][j]);
          }
        }
#pragma unroll
        for (int bb = 0; bb < B; ++bb) {
          const int r = r0 + bb;
          const int cu = __shfl_sync(0xffffffffu, my_cu, r & 31);
          if (r < n_s && cu != cur) {  // warp-uniform: a new colour group
            if (cur >= 0) flush();
            __syncwarp();  // groups of different colours may map to the same N'' entries
            cur = cu;
            const uint16_t *mrow = a.map + (int64_t)(cu * a.k + cv) * a.map_ld + a.col_base;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
              if (valid[j]) {
                if constexpr (VW == 4) {
                  const uint2 w = __ldg(reinterpret_cast<const uint2 *>(mrow + c0 + j * 32 * VW));
                  m[j][0] = w.x & 0xFFFF;
                  m[j][1 % VW] = w.x >> 16;
                  m[j][2 % VW] = w.y & 0xFFFF;
                  m[j][3 % VW] = w.y >> 16;
                } else {
                  const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(mrow + c0 + j * 32 * VW));
                  m[j][0] = w & 0xFFFF;
                  m[j][1 % VW] = w >> 16;
                }
              } else {
#pragma unroll
                for (int q = 0; q < VW; ++q) m[j][q] = 0xFFFF;
              }
            }
          }
#pragma unroll
          for (int j = 0; j < NV; ++j) add_same(blk[j], x[bb][j]);
        }
      }
      if (cur >= 0) flush();
      __syncwarp();
    }
    if (a.root_mode) root_epilogue<T, AccT>(a, sacc, it, v, false, lane);
    else gather_epilogue<T, 32, AccT>(a, sacc, it, v, false, lane, 0xffffffffu);
    __syncwarp();
  }
}

template <typename T, int NV, int B>
void short_go(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = 32 * NV * VW;
  const bool acc32 = sizeof(T) == 4 && (a.W_out > 1600 || (kn.acc32 && !a.root_mode));
  auto kern = acc32 ? k_gather_short<T, NV, B, float> : k_gather_short<T, NV, B, double>;
  const size_t row = (size_t)a.W_out * (acc32 ? sizeof(float) : sizeof(double));
  int warps = 4;
  while (warps > 1 && row * warps > 200 * 1024) warps /= 2;
  const int threads = warps * 32;
  const size_t smem = row * warps;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  const int nch = (a.W_in + CAP - 1) / CAP;
  kern<<<grid, threads, smem, s>>>(a, nch);
}

template <typename T, int G, int NV, int U, int MINB = 3, bool PAIR = false>
void rows_go(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = G * NV * VW;
  // 3 CTAs of 8 warps per SM (<= 85 registers, no spills): configs[2] -4%,
  // configs[3] -1 to -2% against 2 CTAs (profiles/r1/SUMMARY.md)
  // fp32 tables: fp32 shared-memory rows as in the lean gather (C-6)
  const bool acc32 = sizeof(T) == 4 && kn.acc32;
  auto kern = acc32 ? k_gather_rows<T, G, NV, U, MINB, float, PAIR> : k_gather_rows<T, G, NV, U, MINB, double, PAIR>;
  const size_t row = (size_t)(a.W_out + 1) * (acc32 ? sizeof(float) : sizeof(double));  // + the discard slot
  int warps = 8;
  while (warps > 1 && row * warps > 200 * 1024) warps /= 2;
  const int threads = warps * 32;
  const size_t smem = row * warps;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  const int nch = (a.W_in + CAP - 1) / CAP;
  kern<<<grid, threads, smem, s>>>(a, nch);
}

template <typename T, int NV, int U, int MINB = 2>
void ldg_go(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = 32 * NV * VW;
  // fp32 tables with N'' rows wider than 1600 entries (configs[4]'s root:
  // 3432) keep the shared-memory row in fp32 so that 16 warps fit per SM
  // (each entry adds at most k-1 colour-group block sums; C-6)
  // fp32 tables keep the shared-memory N'' row in fp32 (scaled by 2^-64):
  // half the shared memory leaves more L1 for the rows (configs[3]: gathers
  // -1.5 to -2%), and rows wider than 1600 entries (configs[4]'s fused root)
  // need it to fit 16 warps per SM.  Each entry adds at most ceil(s/32) +
  // k - 1 fp32 block sums (C-6); CC_ACC32=0 keeps fp64 rows where
  // they fit.
  const bool acc32 = sizeof(T) == 4 && (a.W_out > 1600 || (kn.acc32 && !a.root_mode));
  auto kern = acc32 ? k_gather_ldg<T, NV, U, float, MINB> : k_gather_ldg<T, NV, U, double, MINB>;
  const size_t row = (size_t)(a.W_out + 1) * (acc32 ? sizeof(float) : sizeof(double));  // + the discard slot
  int warps = 8;
  while (warps > 1 && row * warps > 200 * 1024) warps /= 2;
  // knob wide_warps: fewer warps per CTA for N'' rows of > 8 KB (more L1 left for the rows in flight)
  if (kn.wide_warps > 0 && row > 8 * 1024) warps = std::min(warps, kn.wide_warps);
  // knob tail_warps: smaller CTAs for the short-tail launches (MINB = 3 variants)
  if (MINB == 3 && kn.tail_warps > 0) warps = std::min(warps, kn.tail_warps);
  const int threads = warps * 32;
  const size_t smem = row * warps;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  const int nch = (a.W_in + CAP - 1) / CAP;
  kern<<<grid, threads, smem, s>>>(a, nch);
}

// ------------------------------------------------------------------ launchers
template <typename T, int G, int NV, int D, int MINB = 1, bool PAIR = false, bool SHORT = false>
void ring_go(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  constexpr int CAP = G * NV * VW;
  // SHORT (the short tail of narrow_impl = 4: items of <= 1024 neighbours): fp32 rows for fp32 tables
  constexpr bool F32 = SHORT && !PAIR && sizeof(T) == 4;
  if constexpr (F32) {
    if (!kn.acc32) return ring_go<T, G, NV, D, MINB, PAIR, false>(a, kn, num_sms, s);
  }
  using AccT = typename std::conditional<F32, float, double>::type;
  auto kern = k_gather_ring<T, G, NV, D, MINB, PAIR, AccT>;
  const size_t per_group = (size_t)D * NV * G * 16 + (size_t)(a.W_out + 1) * sizeof(AccT);  // + discard slot
  int groups = 256 / G;
  // (sibling pairs: as many groups as MINB CTAs per SM allow)
  while (groups > 1 && (PAIR ? per_group * groups * MINB > 224 * 1024 : per_group * groups > 100 * 1024)) groups /= 2;
  const int threads = groups * G;
  const size_t smem = per_group * groups;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  const int nch = (a.W_in + CAP - 1) / CAP;
  kern<<<grid, threads, smem, s>>>(a, nch);
}

// A sibling pair of narrow passives (GatherArgs::src2): one traversal, the
// long lists row-parallel and the short tail on rings as for one narrow
// table, over the virtual row of both parts (<= 24 vectors).
template <typename T>
int pair_typed(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  constexpr int VW = Vec<T>::W;
  const int wvec = (a.W_in + VW - 1) / VW;
  const int64_t from = a.item_from, to = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
  const int64_t split = std::min(std::max(a.item_split, from), to);
  GatherArgs h = a, t = a;
  h.item_to = split;
  t.item_from = split;
  int launches = 0;
  if (h.item_from < h.item_to) {
    if (wvec <= 8) rows_go<T, 8, 1, 4, 3, true>(h, kn, num_sms, s);
    else if (wvec <= 16) rows_go<T, 8, 2, 4, 3, true>(h, kn, num_sms, s);
    else if (kn.rows_variant == 2) rows_go<T, 8, 3, 4, 2, true>(h, kn, num_sms, s);  // more rows in flight
    else rows_go<T, 8, 3, 3, 3, true>(h, kn, num_sms, s);
    ++launches;
  }
  if (t.item_from < t.item_to) {
    if (wvec <= 8) ring_go<T, 8, 1, 4, 2, true>(t, kn, num_sms, s);
    else if (wvec <= 16) ring_go<T, 8, 2, 4, 3, true>(t, kn, num_sms, s);
    else ring_go<T, 8, 3, 4, 2, true>(t, kn, num_sms, s);
    ++launches;
  }
  return launches;
}

template <typename T>
int gather_typed(const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {  // returns the launches
  constexpr int VW = Vec<T>::W;
  const int wvec = (a.W_in + VW - 1) / VW;
  if (a.src2) return pair_typed<T>(a, kn, num_sms, s);
  // default: rows of <= 16 vectors go to the narrow kernels, wider rows to
  // the lean kernel (measured, profiles/r1/SUMMARY.md).  The fused root
  // exists in the lean kernel only.
  const bool lean = kn.gather_impl ? kn.gather_impl == 2 : wvec > 16;
  if (lean || a.root_mode) {
    const int64_t to = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
    if (a.lean_split > a.item_from && a.lean_split < to) {  // two launches: long lists, short tail
      GatherArgs h = a, t = a;
      h.item_to = a.lean_split;
      h.lean_split = -1;
      t.item_from = a.lean_split;
      t.lean_split = -1;
      return gather_typed<T>(h, kn, num_sms, s) + gather_typed<T>(t, kn, num_sms, s);
    }
    // the items with <= 32 neighbours on the short-list kernel (knob short_lists)
    if (kn.short_lists && a.short_from < to) {
      const int64_t sf = std::max(a.short_from, a.item_from);
      int launches = 0;
      if (a.item_from < sf) {
        GatherArgs h = a;
        h.item_to = sf;
        h.short_from = to;  // (no further split)
        launches += gather_typed<T>(h, kn, num_sms, s);
      }
      GatherArgs t = a;
      t.item_from = sf;
      t.item_to = to;
      if (kn.short_lists == 1) {
        if (wvec <= 32) short_go<T, 1, 8>(t, kn, num_sms, s);
        else if (wvec <= 64) short_go<T, 2, 8>(t, kn, num_sms, s);
        else if (wvec <= 96) short_go<T, 3, 6>(t, kn, num_sms, s);
        else short_go<T, 4, 4>(t, kn, num_sms, s);
      } else if (kn.short_lists == 2) {  // the lean kernel, fewer rows in flight, more warps
        // (configs[3]: 155.8 -> 149.0 ms per colouring with the tail at <= 128 neighbours;
        // rows of > 96 vectors keep the long-list kernel: 3 CTAs would spill)
        if (wvec <= 32) ldg_go<T, 1, 2, 3>(t, kn, num_sms, s);
        else if (wvec <= 64) ldg_go<T, 2, 2, 3>(t, kn, num_sms, s);
        else if (wvec <= 96) ldg_go<T, 3, 2, 3>(t, kn, num_sms, s);
        else ldg_go<T, 4, 2>(t, kn, num_sms, s);
      } else if (kn.short_lists == 4) {  // U = 3 at 3 CTAs/SM
        if (wvec <= 32) ldg_go<T, 1, 3, 3>(t, kn, num_sms, s);
        else if (wvec <= 64) ldg_go<T, 2, 3, 3>(t, kn, num_sms, s);
        else if (wvec <= 96) ldg_go<T, 3, 3, 3>(t, kn, num_sms, s);
        else ldg_go<T, 4, 2, 3>(t, kn, num_sms, s);
      } else {
        if (wvec <= 32) ldg_go<T, 1, 1, 4>(t, kn, num_sms, s);
        else if (wvec <= 64) ldg_go<T, 2, 1, 4>(t, kn, num_sms, s);
        else if (wvec <= 96) ldg_go<T, 3, 1, 4>(t, kn, num_sms, s);
        else ldg_go<T, 4, 1, 4>(t, kn, num_sms, s);
      }
      return launches + 1;
    }
    if (wvec <= 32) ldg_go<T, 1, 8>(a, kn, num_sms, s);
    else if (wvec <= 64) ldg_go<T, 2, 8>(a, kn, num_sms, s);
    else if (wvec <= 96) ldg_go<T, 3, 4>(a, kn, num_sms, s);
    else if (kn.wide_nv == 6 && wvec > 128) ldg_go<T, 6, 2>(a, kn, num_sms, s);  // (knob wide_nv: fewer passes)
    else ldg_go<T, 4, 2>(a, kn, num_sms, s);
    return 1;
  }
  // narrow rows: long lists (items before a.item_split) on warp-per-item
  // row-parallel loads, the short tail on sub-warp rings
  if (kn.narrow_impl == 4 && wvec <= 16) {
    const int64_t from = a.item_from, to = a.item_to >= 0 ? a.item_to : a.work.n_seg + a.work.n_light;
    const int64_t split = std::min(std::max(a.item_split, from), to);
    GatherArgs h = a, t = a;
    h.item_from = from;
    h.item_to = split;
    t.item_from = split;
    t.item_to = to;
    int launches = 0;
    if (h.item_from < h.item_to) {
      if (kn.rows_variant == 1) {  // fewer rows in flight, more warps
        if (wvec <= 4) rows_go<T, 4, 1, 2, 4>(h, kn, num_sms, s);
        else if (wvec <= 8) rows_go<T, 8, 1, 2, 4>(h, kn, num_sms, s);
        else rows_go<T, 8, 2, 2, 4>(h, kn, num_sms, s);
      } else if (kn.rows_variant == 2) {  // more rows in flight
        if (wvec <= 4) rows_go<T, 4, 1, 8, 2>(h, kn, num_sms, s);
        else if (wvec <= 8) rows_go<T, 8, 1, 8, 2>(h, kn, num_sms, s);
        else rows_go<T, 8, 2, 8, 2>(h, kn, num_sms, s);
      } else {
        if (wvec <= 4) rows_go<T, 4, 1, 4>(h, kn, num_sms, s);
        else if (wvec <= 8) rows_go<T, 8, 1, 4>(h, kn, num_sms, s);
        else rows_go<T, 8, 2, 4>(h, kn, num_sms, s);
      }
      ++launches;
    }
    if (t.item_from < t.item_to) {
      if (wvec <= 4) ring_go<T, 4, 1, 4, 3, false, true>(t, kn, num_sms, s);
      else if (wvec <= 8) ring_go<T, 8, 1, 4, 2, false, true>(t, kn, num_sms, s);
      else ring_go<T, 8, 2, 4, 3, false, true>(t, kn, num_sms, s);
      ++launches;
    }
    return launches;
  }
  if (kn.narrow_impl >= 1 && kn.narrow_impl <= 3 && wvec <= 16) {
    if (wvec <= 4) rows_go<T, 4, 1, 4>(a, kn, num_sms, s);
    else if (wvec <= 8) rows_go<T, 8, 1, 4>(a, kn, num_sms, s);
    else rows_go<T, 8, 2, 4>(a, kn, num_sms, s);
    return 1;
  }
  // narrow rows: small rings (more resident groups) measured faster
  // (p = 2: D 16 -> 4: 12.3 -> 9.0 ms; p = 3: G 16 x 1 -> 8 x 2 vectors,
  // D 4: 31.5 -> 19.8 ms, the lean kernel 27.8 ms)
  if (wvec <= 4) ring_go<T, 4, 1, 4, 3>(a, kn, num_sms, s);  // 3 CTAs/SM: configs[2] -1.5%
  else if (wvec <= 8) ring_go<T, 8, 1, 4, 2>(a, kn, num_sms, s);
  else if (wvec <= 16) ring_go<T, 8, 2, 4, 3>(a, kn, num_sms, s);
  else if (wvec <= 32) ring_go<T, 32, 1, 16, 2>(a, kn, num_sms, s);
  else if (wvec <= 64) ring_go<T, 32, 2, 8, 2>(a, kn, num_sms, s);
  else ring_go<T, 32, 4, 4, 2>(a, kn, num_sms, s);
  return 1;
}

}  // namespace

int launch_csort(const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                 const AggWork &work, int32_t *col_out, uint16_t *goff, ItemDesc *desc, int num_sms,
                 cudaStream_t s) {
  if (work.n_seg + work.n_light == 0) return 0;
  const int grid = persistent_grid(k_csort, 256, 0, num_sms);
  k_csort<<<grid, 256, 0, s>>>(beg, end, col, colors, work, col_out, goff, desc);
  return 1;
}

int launch_csort_hist(int elem, const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                      const AggWork &work, int k, int32_t *col_out, uint16_t *goff, ItemDesc *desc, void *hist,
                      int64_t ldh, int64_t hist_rows, int64_t small_from, const Knobs &kn, int num_sms,
                      cudaStream_t s) {
  const int64_t n_items = work.n_seg + work.n_light;
  if (n_items == 0) return 0;
  int launches = 1;
  // the items before small_from: one warp each (k_csort2 walks n_items on its
  // own work view, so it gets a view truncated to small_from)
  AggWork head = work;
  const bool split = kn.csort_small != 0;
  if (split && small_from < n_items) head.n_light = small_from - work.n_seg;
  if (hist && work.n_seg) {  // heavy rows accumulate segment counts atomically
    cudaMemsetAsync(hist, 0, (size_t)hist_rows * ldh * elem, s);
    ++launches;
  }
  if (elem == 8) {
    const int grid = persistent_grid(k_csort2<double>, 256, 0, num_sms);
    k_csort2<double><<<grid, 256, 0, s>>>(beg, end, col, colors, head, k, col_out, goff, desc,
                                          static_cast<double *>(hist), ldh);
  } else {
    const int grid = persistent_grid(k_csort2<float>, 256, 0, num_sms);
    k_csort2<float><<<grid, 256, 0, s>>>(beg, end, col, colors, head, k, col_out, goff, desc,
                                         static_cast<float *>(hist), ldh);
  }
  if (split && small_from < n_items) {
    ++launches;
    if (elem == 8) {
      const int grid = persistent_grid(k_csort_small<double>, 256, 0, num_sms);
      k_csort_small<double><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, small_from, col_out, goff, desc,
                                                 static_cast<double *>(hist), ldh);
    } else {
      const int grid = persistent_grid(k_csort_small<float>, 256, 0, num_sms);
      k_csort_small<float><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, small_from, col_out, goff, desc,
                                                static_cast<float *>(hist), ldh);
    }
  }
  return launches;
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
    const int grid = persistent_grid(k_hist<double, 8>, 256, 0, num_sms);
    k_hist<double, 8><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, static_cast<double *>(out), ld);
  } else {
    const int grid = persistent_grid(k_hist<float, 8>, 256, 0, num_sms);
    k_hist<float, 8><<<grid, 256, 0, s>>>(beg, end, col, colors, work, k, static_cast<float *>(out), ld);
  }
  return launches;
}

int launch_gather(int elem, const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s) {
  if (a.work.n_seg + a.work.n_light == 0) return 0;
  return elem == 8 ? gather_typed<double>(a, kn, num_sms, s) : gather_typed<float>(a, kn, num_sms, s);
}

}  // namespace dev
}  // namespace cc
