// kernels.cu -- colouring, combine, root and halo-pack kernels (sm_100a).
// The neighbour-sum kernels (colour sort, hist, gather) live in gather.cu.
//
// Every kernel here is memory- or LSU-bound integer-indexed work; there is no
// dense contraction, so no tensor cores (BASELINE.json north_star).  Grids are
// persistent (a multiple of the SM count x resident blocks per SM, from the
// occupancy calculator) and walk their work with a static interleaved stride,
// so every reduction order -- and therefore every result -- is deterministic.
//
//   k_color   colouring, PAPER.md lines 156-158 (reading C-2)
//   k_permute_colors  a caller's colouring to the internal row order
//   k_combine T'(v, S') = sum_{X' u Y'' = S'} A'(v, X') N''(v, Y''): the split
//             sum of Eq. 1, colour-independent in the
//             compressed (k-1)-colour universe -- V-tile kernel (thread per
//             output set) for low-intensity steps
//   k_combine_lane  lane-per-vertex split walk for the other shapes
//   k_combine_z     register-blocked split walk over a Z-block cover
//   k_rowsum  root of a template with fewer vertices than colours
//   k_root    X = sum_v sum_{X'} A'(v, X') N''(v, [k-1] \ X'): the last step
//             fused with Eq. 3's sum over v, fp64
//   k_pack    halo rows for the 1D partition exchange (Alg. 2 line 15)
// A step whose active part is the single root vertex (a = 1) needs no kernel:
// in the compressed layout its table IS the neighbour sum N''.
#include <algorithm>

#include "dev_common.cuh"

namespace cc {
namespace dev {

namespace {

// ------------------------------------------------------------------ colour
__global__ void k_color(const int32_t *__restrict__ orig, int64_t n, uint64_t seed, int k,
                        uint8_t *__restrict__ out) {
  const uint64_t s = mix64(seed);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = mix64(s ^ (uint64_t)(uint32_t)orig[v]) >> 32;
    out[v] = (uint8_t)((h * (uint64_t)k) >> 32);
  }
}

// A caller-supplied colouring (original ids) -> the internal row order, with
// the range check [0, k) on the device (bad[0] |= 1 on a violation).
__global__ void k_permute_colors(const uint8_t *__restrict__ by_orig, const int32_t *__restrict__ orig, int64_t n,
                                 int k, uint8_t *__restrict__ out, unsigned *__restrict__ bad) {
  bool ok = true;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t c = by_orig[orig[i]];
    ok &= c < k;
    out[i] = c;
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// ------------------------------------------------------------------ combine (a >= 2)
// V vertices per CTA: their A' and N'' rows are staged in shared memory
// TRANSPOSED (column-major over the tile's vertices), so one 16-byte load
// feeds VW vertices of the same split.  One thread per output colour set
// walks the split table (coalesced, L1/L2 resident).  Accumulation is in the
// storage type: fp64 tables -> DFMA; fp32 tables -> FFMA over at most
// C(t-1, a-1) terms (relative error <= C(t-1,a-1) * 2^-24, C-6).
template <typename T, int V>
__global__ void __launch_bounds__(256) k_combine(const T *__restrict__ A, int64_t ldA, int WA,
                                                 const T *__restrict__ N, int64_t ldN, int WN,
                                                 const uint32_t *__restrict__ split, int nq, int64_t n,
                                                 T *__restrict__ out, int64_t ldO, int WO, int o_lo, int o_hi) {
  using VT = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  static_assert(V % VW == 0, "tile must be a multiple of the vector width");
  constexpr int SV = V == VW ? V : V + VW;  // padded row stride spreads rows over the banks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *As = reinterpret_cast<T *>(smem_raw);  // [WA][SV]
  T *Ns = As + SV * WA;                     // [WN][SV]
  const int64_t ntiles = (n + V - 1) / V;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * V;
    const int nv = (int)min((int64_t)V, n - v0);
    for (int i = threadIdx.x; i < V * WA; i += blockDim.x) {
      const int r = i / WA, x = i - r * WA;
      As[x * SV + r] = r < nv ? A[(v0 + r) * ldA + x] : (T)0;
    }
    for (int i = threadIdx.x; i < V * WN; i += blockDim.x) {
      const int r = i / WN, y = i - r * WN;
      Ns[y * SV + r] = r < nv ? N[(v0 + r) * ldN + y] : (T)0;
    }
    __syncthreads();
    for (int s = o_lo + threadIdx.x; s < o_hi; s += blockDim.x) {
      T acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = (T)0;
      for (int q = 0; q < nq; ++q) {
        const uint32_t sp = __ldg(split + (int64_t)q * ((WO + 7) & ~7) + s);
        const VT *ax = reinterpret_cast<const VT *>(As + (sp & 0xFFFF) * SV);
        const VT *ny = reinterpret_cast<const VT *>(Ns + (sp >> 16) * SV);
#pragma unroll
        for (int i = 0; i < V / VW; ++i) {
          const VT av = ax[i], nv4 = ny[i];
          if constexpr (VW == 4) {
            acc[4 * i + 0] = fmaf(av.x, nv4.x, acc[4 * i + 0]);
            acc[4 * i + 1] = fmaf(av.y, nv4.y, acc[4 * i + 1]);
            acc[4 * i + 2] = fmaf(av.z, nv4.z, acc[4 * i + 2]);
            acc[4 * i + 3] = fmaf(av.w, nv4.w, acc[4 * i + 3]);
          } else {
            acc[2 * i + 0] = fma(av.x, nv4.x, acc[2 * i + 0]);
            acc[2 * i + 1] = fma(av.y, nv4.y, acc[2 * i + 1]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (i < nv) out[(v0 + i) * ldO + s] = acc[i];
    }
    __syncthreads();
  }
}

// Warp-per-vertex combine for low-intensity steps (few split terms per output,
// e.g. the p = 1 steps (t; t-1, 1): t - 1 terms): the split-table slice of the
// outputs [o_lo, o_hi) sits in shared memory once per CTA; each warp stages
// its vertex's A' and N'' rows in shared memory (one coalesced load each, the
// next vertex's already in registers), then a lane per output walks its split
// pairs and the outputs go out coalesced.  Latency of the row loads is hidden
// by the next vertex's prefetch and by 16 warps per SM.
// The same walk with the split pairs in registers (nq = NQ splits per
// output, <= 256 outputs): a lane owns outputs lane + 32 i for the whole
// launch, so its split entries are loaded once; per vertex an output costs
// NQ x (two shared-memory reads + FMA).  Same sums in the same order as
// k_combine_warp.
template <typename T, int PF, int NQ, int NO>
__global__ void __launch_bounds__(256) k_combine_wreg(const T *__restrict__ A, int64_t ldA, int WA,
                                                     const T *__restrict__ N, int64_t ldN, int WN,
                                                     const uint32_t *__restrict__ split, int64_t n,
                                                     T *__restrict__ out, int64_t ldO, int WO, int o_lo, int o_hi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int WOp = (WO + 7) & ~7, nout = o_hi - o_lo;
  uint32_t sp[NO][NQ];
#pragma unroll
  for (int i = 0; i < NO; ++i)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int o = lane + 32 * i;
      sp[i][q] = o < nout ? __ldg(split + (int64_t)q * WOp + o_lo + o) : 0u;
    }
  T *rows = reinterpret_cast<T *>(smem_raw) + (size_t)warp * (WA + WN);
  const int64_t nw = (int64_t)gridDim.x * nwarp;
  int64_t v = (int64_t)blockIdx.x * nwarp + warp;
  T pa[PF], pn[PF];
  auto fetch = [&](int64_t u) {
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int x = lane + 32 * i;
      pa[i] = (u < n && x < WA) ? __ldg(A + u * ldA + x) : (T)0;
      pn[i] = (u < n && x < WN) ? __ldg(N + u * ldN + x) : (T)0;
    }
  };
  fetch(v);
  for (; v < n; v += nw) {
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int x = lane + 32 * i;
      if (x < WA) rows[x] = pa[i];
      if (x < WN) rows[WA + x] = pn[i];
    }
    __syncwarp();
    fetch(v + nw);  // the next vertex's rows are in flight during this one's walk
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      if (32 * i < nout) {  // warp-uniform
        const int o = lane + 32 * i;
        T acc = (T)0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc = fma(rows[sp[i][q] & 0xFFFF], rows[WA + (sp[i][q] >> 16)], acc);
        if (o < nout) out[v * ldO + o_lo + o] = acc;
      }
    }
    __syncwarp();
  }
}

template <typename T, int PF>
__global__ void __launch_bounds__(256) k_combine_warp(const T *__restrict__ A, int64_t ldA, int WA,
                                                      const T *__restrict__ N, int64_t ldN, int WN,
                                                      const uint32_t *__restrict__ split, int nq, int64_t n,
                                                      T *__restrict__ out, int64_t ldO, int WO, int o_lo, int o_hi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int WOp = (WO + 7) & ~7, nout = o_hi - o_lo;
  uint32_t *ss = reinterpret_cast<uint32_t *>(smem_raw);  // [q][nout]
  for (int i = threadIdx.x; i < nq * nout; i += blockDim.x) {
    const int q = i / nout, o = i - q * nout;
    ss[i] = split[(int64_t)q * WOp + o_lo + o];
  }
  T *rows = reinterpret_cast<T *>(smem_raw + (((size_t)nq * nout * 4 + 15) & ~(size_t)15)) + (size_t)warp * (WA + WN);
  __syncthreads();
  const int64_t nw = (int64_t)gridDim.x * nwarp;
  int64_t v = (int64_t)blockIdx.x * nwarp + warp;
  T pa[PF], pn[PF];  // the next vertex's rows, lane-strided
  auto fetch = [&](int64_t u) {
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int x = lane + 32 * i;
      pa[i] = (u < n && x < WA) ? __ldg(A + u * ldA + x) : (T)0;
      pn[i] = (u < n && x < WN) ? __ldg(N + u * ldN + x) : (T)0;
    }
  };
  fetch(v);
  for (; v < n; v += nw) {
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int x = lane + 32 * i;
      if (x < WA) rows[x] = pa[i];
      if (x < WN) rows[WA + x] = pn[i];
    }
    __syncwarp();
    fetch(v + nw);  // the next vertex's rows are in flight during this one's split walk
    for (int o = lane; o < nout; o += 32) {
      T acc = (T)0;
      for (int q = 0; q < nq; ++q) {
        const uint32_t sp = ss[q * nout + o];
        acc = fma(rows[sp & 0xFFFF], rows[WA + (sp >> 16)], acc);
      }
      out[v * ldO + o_lo + o] = acc;
    }
    __syncwarp();
  }
}

// Lane-per-vertex combine (persistent, one CTA of 8 warps per SM): tiles of
// 32 vertices' A' and N'' rows are staged TRANSPOSED in shared memory as
// [column][33] by cp.async (double-buffered: tile i+1 streams in while tile i
// is computed); the split table sits in shared memory when it fits.  Each
// warp takes groups of 8 output colour sets; per split q one warp-uniform
// 32-byte read of the table gives 8 (x, y) pairs, and every lane accumulates
// its own vertex: 2 conflict-free LDS per FMA (shared-memory bound, not HBM).
template <typename T>
__device__ __forceinline__ void cp_async_elem(T *smem, const T *gmem, bool ok) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 4 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
}

template <typename T, int V>
struct LaneVec;
template <typename T>
struct LaneVec<T, 1> {
  using type = T;
  __device__ static T at(const T &x, int) { return x; }
};
template <>
struct LaneVec<float, 2> {
  using type = float2;
  __device__ static float at(const float2 &x, int i) { return i ? x.y : x.x; }
};
template <>
struct LaneVec<double, 2> {
  using type = double2;
  __device__ static double at(const double2 &x, int i) { return i ? x.y : x.x; }
};

// V vertices per lane (tile = 32 V vertices): element (v, c) of the staged
// tile sits at [c][v / V][v % V] with a row stride of 33 vectors, so a lane
// reads its V vertices of column c with one conflict-free V-wide LDS and one
// address computation serves V FMAs.
// One launch covers the output colour sets [o0, o0 + WOc): the split table
// slice of those outputs is staged in shared memory (wide steps whose whole
// table does not fit run several launches, re-staging the tiles).
template <typename T, int OUT, int V>
__global__ void __launch_bounds__(512, 1) k_combine_lane(const T *__restrict__ A, int64_t ldA, int WA,
                                                         const T *__restrict__ N, int64_t ldN, int WN,
                                                         const uint32_t *__restrict__ split, int nq, int64_t n,
                                                         T *__restrict__ out, int64_t ldO, int WO, int nbuf, int o0,
                                                         int WOc) {
  constexpr int S = 33;       // row stride in V-vectors
  constexpr int TV = 32 * V;  // vertices per tile
  using LV = typename LaneVec<T, V>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int W = WA + WN;
  const size_t bstride = ((size_t)S * V * W * sizeof(T) + 15) / 16 * 16 / sizeof(T);  // 16-byte aligned buffers
  T *bufs = reinterpret_cast<T *>(smem_raw);  // nbuf x [W][33][V]: A' columns then N'' columns
  const int WOp = (WO + 7) & ~7, WOcp = (WOc + 7) & ~7;
  const int o_end = min(WO, o0 + WOc);
  // the split-table slice [q][WOcp] of this launch's outputs, in shared memory
  uint32_t *ss = reinterpret_cast<uint32_t *>(bufs + (size_t)nbuf * bstride);
  for (int i = threadIdx.x; i < nq * WOcp; i += blockDim.x) {
    const int q = i / WOcp, o = o0 + i - q * WOcp;
    ss[i] = o < WOp ? split[(int64_t)q * WOp + o] : 0u;
  }
  const int64_t ntiles = (n + TV - 1) / TV;
  auto stage = [&](int64_t tile, T *b) {
    const int64_t v0 = tile * TV;
    for (int r = warp; r < TV; r += nwarp) {
      const bool ok = v0 + r < n;
      const int64_t vr = ok ? v0 + r : 0;
      T *dst = b + (r / V) * V + (r % V);
      for (int x = lane; x < WA; x += 32) cp_async_elem(dst + (size_t)x * S * V, A + vr * ldA + x, ok);
      for (int y = lane; y < WN; y += 32) cp_async_elem(dst + (size_t)(WA + y) * S * V, N + vr * ldN + y, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) stage(tile, bufs);
  __syncthreads();  // split table staged
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    T *cur = bufs + (size_t)(nbuf == 2 ? (it & 1) : 0) * bstride;
    if (nbuf == 2) {
      if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, bufs + (size_t)((it + 1) & 1) * bstride);
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    // byte bases of the lane's vectors: one IMAD per operand address
    const char *Ab = reinterpret_cast<const char *>(reinterpret_cast<const LV *>(cur) + lane);
    const char *Nb = reinterpret_cast<const char *>(reinterpret_cast<const LV *>(cur) + (size_t)WA * S + lane);
    constexpr uint32_t CB = S * sizeof(LV);  // bytes per staged column
    const int64_t vb = tile * TV + (int64_t)lane * V;
    for (int g = warp; g < (WOc + OUT - 1) / OUT; g += nwarp) {
      T acc[OUT][V];
#pragma unroll
      for (int j = 0; j < OUT; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[j][i] = (T)0;
      const uint4 *e = reinterpret_cast<const uint4 *>(ss) + (OUT / 4) * g;
#pragma unroll 2
      for (int q = 0; q < nq; ++q) {
        uint32_t xy[OUT];
#pragma unroll
        for (int h = 0; h < OUT / 4; ++h) {
          const uint4 eh = e[q * (WOcp / 4) + h];
          xy[4 * h + 0] = eh.x;
          xy[4 * h + 1] = eh.y;
          xy[4 * h + 2] = eh.z;
          xy[4 * h + 3] = eh.w;
        }
#pragma unroll
        for (int j = 0; j < OUT; ++j) {
          const LV av = *reinterpret_cast<const LV *>(Ab + (xy[j] & 0xFFFF) * CB);
          const LV nv = *reinterpret_cast<const LV *>(Nb + (xy[j] >> 16) * CB);
#pragma unroll
          for (int i = 0; i < V; ++i)
            acc[j][i] = fma(LaneVec<T, V>::at(av, i), LaneVec<T, V>::at(nv, i), acc[j][i]);
        }
      }
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (vb + i < n) {
#pragma unroll
          for (int j = 0; j < OUT; ++j)
            if (o0 + OUT * g + j < o_end) out[(vb + i) * ldO + o0 + OUT * g + j] = acc[j][i];
        }
    }
    __syncthreads();  // the buffer is refilled two tiles later (or next tile when single-buffered)
    if (nbuf == 1 && tile + gridDim.x < ntiles) stage(tile + gridDim.x, bufs);
  }
}

// Z-block combine.  For a block Z of t'+1 colours, every split (X, Y) of
// every output S = Z \ {z} uses only the C(t'+1, a') active sets and the
// C(t'+1, p') passive sets of Z.  A lane (one vertex, or V vertices) loads
// Z's passive values into registers once, then streams Z's active values:
// each active value X feeds the p'+1 outputs Z \ {z}, z not in X, with the
// passive value Z \ X \ {z} -- register indices fixed at compile time by
// ZTab.  Shared-memory reads per FMA drop from 2 to ~0.4 (config 3's
// (9;6,3): 25 blocks cover its 165 outputs).
constexpr int cbinom(int n, int r) {
  if (r < 0 || r > n) return 0;
  int c = 1;
  for (int i = 1; i <= r; ++i) c = c * (n - r + i) / i;
  return c;
}
constexpr int clocal_rank(unsigned m) {  // colex rank of a subset of {0..31}
  int r = 0, i = 0;
  for (int c = 0; c < 32; ++c)
    if (m >> c & 1u) r += cbinom(c, ++i);
  return r;
}
constexpr unsigned clocal_unrank(int s, int r) {
  unsigned m = 0;
  int hi = 31;
  for (int i = s; i >= 1; --i) {
    int c = i - 1;
    while (c + 1 <= hi && cbinom(c + 1, i) <= r) ++c;
    r -= cbinom(c, i);
    m |= 1u << c;
    hi = c - 1;
  }
  return m;
}
template <int ZS, int AS>
struct ZTab {
  static constexpr int PS = ZS - 1 - AS;
  static constexpr int NA = cbinom(ZS, AS), NN = cbinom(ZS, PS);
  int z[NA][PS + 1];  // outputs (local z) fed by active set a
  int y[NA][PS + 1];  // the passive set's local index for that output
  constexpr ZTab() : z(), y() {
    for (int a = 0; a < NA; ++a) {
      const unsigned X = clocal_unrank(AS, a);
      int q = 0;
      for (int zz = 0; zz < ZS; ++zz) {
        if (X >> zz & 1u) continue;
        z[a][q] = zz;
        y[a][q] = clocal_rank(((1u << ZS) - 1) & ~X & ~(1u << zz));
        ++q;
      }
    }
  }
};

// GT (global table): the cover stays in global memory (L1-cached, warp-uniform
// 16-byte loads at each block's start) when it does not fit next to the tile --
// configs[4]'s (7;4,3) at k = 15: 627 blocks x 160 B = 100 KB.
template <typename T, int ZS, int AS, int V, bool GT = false>
__global__ void __launch_bounds__(512, 1) k_combine_z(const T *__restrict__ A, int64_t ldA, int WA,
                                                      const T *__restrict__ N, int64_t ldN, int WN,
                                                      const uint16_t *__restrict__ ztab, int nblocks, int zld, int64_t n,
                                                      T *__restrict__ out, int64_t ldO, int nbuf,
                                                      const uint16_t *__restrict__ comp, double *__restrict__ per_vertex) {
  constexpr ZTab<ZS, AS> tab{};
  constexpr int PS = ZS - 1 - AS, NA = ZTab<ZS, AS>::NA, NN = ZTab<ZS, AS>::NN;
  constexpr int S = 33;
  constexpr int TV = 32 * V;
  using LV = typename LaneVec<T, V>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int W = WA + WN;
  const size_t bstride = ((size_t)S * V * W * sizeof(T) + 15) / 16 * 16 / sizeof(T);
  T *bufs = reinterpret_cast<T *>(smem_raw);
  // the cover in shared memory as 32-bit entries: the staged-tile byte
  // offset (column x CB) of each active / passive set, then the raw output
  // columns -- one LDS.128 gives 4 ready addresses
  constexpr uint32_t CB = S * sizeof(LV);
  uint32_t *zs = reinterpret_cast<uint32_t *>(bufs + (size_t)nbuf * bstride);
  if constexpr (!GT)
    for (int i = threadIdx.x; i < nblocks * zld; i += blockDim.x) {
      const uint32_t x = ztab[i];
      zs[i] = (i % zld) < NA + NN ? x * CB : x;
    }
  // fused root (per_vertex != nullptr): the outputs are not stored; each
  // output T'(v, X') (rounded to the storage type, as the stored table would
  // be) is multiplied in fp64 by the staged N''(v, comp X') -- the root step
  // (Eq. 2 at the root) shares this step's passive -- and the per-warp sums
  // are added in warp order into X_v (Eq. 3's summand)
  double *red = reinterpret_cast<double *>(smem_raw + ((size_t)nbuf * bstride * sizeof(T) + (GT ? 0 : (size_t)nblocks * zld * 4) + 7) / 8 * 8);
  const int64_t ntiles = (n + TV - 1) / TV;
  // GT: each warp's next cover block is prefetched by cp.async into a
  // per-warp double buffer of zld raw entries, then turned into the ready
  // 32-bit byte offsets of the shared-memory path (behind the fused root's sums)
  uint16_t *wtab = reinterpret_cast<uint16_t *>(red + (per_vertex ? nwarp * TV : 0)) + (size_t)warp * 4 * zld;
  uint32_t *woff = reinterpret_cast<uint32_t *>(wtab + 2 * zld);
  int jt = 0;  // this warp's running block count (buffer parity)
  auto tprefetch = [&](int zb, int buf) {
    if (lane * 8 < zld) {
      const unsigned d = (unsigned)__cvta_generic_to_shared(wtab + (size_t)buf * zld + lane * 8);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(ztab + (size_t)zb * zld + lane * 8)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (GT && warp < nblocks) tprefetch(warp, 0);
  auto stage = [&](int64_t tile, T *b) {
    const int64_t v0 = tile * TV;
    for (int r = warp; r < TV; r += nwarp) {
      const bool ok = v0 + r < n;
      const int64_t vr = ok ? v0 + r : 0;
      T *dst = b + (r / V) * V + (r % V);
      for (int x = lane; x < WA; x += 32) cp_async_elem(dst + (size_t)x * S * V, A + vr * ldA + x, ok);
      for (int y = lane; y < WN; y += 32) cp_async_elem(dst + (size_t)(WA + y) * S * V, N + vr * ldN + y, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) stage(tile, bufs);
  __syncthreads();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    T *cur = bufs + (size_t)(nbuf == 2 ? (it & 1) : 0) * bstride;
    if (nbuf == 2) {
      if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, bufs + (size_t)((it + 1) & 1) * bstride);
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const char *Ab = reinterpret_cast<const char *>(reinterpret_cast<const LV *>(cur) + lane);
    const char *Nb = reinterpret_cast<const char *>(reinterpret_cast<const LV *>(cur) + (size_t)WA * S + lane);
    const int64_t vb = tile * TV + (int64_t)lane * V;
    double rsum[V];
#pragma unroll
    for (int i = 0; i < V; ++i) rsum[i] = 0.0;
    T *orow[V];  // the stored outputs' rows (nullptr past n)
#pragma unroll
    for (int i = 0; i < V; ++i) orow[i] = vb + i < n && out ? out + (vb + i) * ldO : nullptr;
    for (int zb = warp; zb < nblocks; zb += nwarp) {
      const uint32_t *e = zs + (size_t)zb * zld;
      if constexpr (GT) {
        const int nxt = zb + nwarp < nblocks ? zb + nwarp : warp;  // wraps to the next tile's first block
        __syncwarp();  // the previous block's offsets are read
        tprefetch(nxt, (jt + 1) & 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncwarp();
        const uint16_t *raw = wtab + (size_t)(jt & 1) * zld;
        for (int i = lane; i < zld; i += 32) {
          const uint32_t x = raw[i];
          woff[i] = i < NA + NN ? x * CB : x;
        }
        __syncwarp();
        e = woff;
        ++jt;
      }
      // block entries read 4 at a time (one 16-byte broadcast load per 4
      // ready byte offsets)
      const uint4 *e4 = reinterpret_cast<const uint4 *>(e);
      auto off = [&](int i) -> uint32_t {
        const uint4 w = e4[i >> 2];
        return (i & 3) == 0 ? w.x : (i & 3) == 1 ? w.y : (i & 3) == 2 ? w.z : w.w;
      };
      LV nv[NN];
#pragma unroll
      for (int j = 0; j < NN; ++j) nv[j] = *reinterpret_cast<const LV *>(Nb + off(NA + j));
      T acc[ZS][V];
#pragma unroll
      for (int zz = 0; zz < ZS; ++zz)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[zz][i] = (T)0;
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const LV av = *reinterpret_cast<const LV *>(Ab + off(a));
#pragma unroll
        for (int q = 0; q <= PS; ++q)
#pragma unroll
          for (int i = 0; i < V; ++i)
            acc[tab.z[a][q]][i] = fma(LaneVec<T, V>::at(av, i), LaneVec<T, V>::at(nv[tab.y[a][q]], i),
                                      acc[tab.z[a][q]][i]);
      }
#pragma unroll
      for (int zz = 0; zz < ZS; ++zz) {
        const uint32_t oc = e[NA + NN + zz];
        if (oc != 0xFFFFu) {
          if (per_vertex) {
            const LV ny = *reinterpret_cast<const LV *>(Nb + (uint32_t)__ldg(comp + oc) * CB);
#pragma unroll
            for (int i = 0; i < V; ++i) rsum[i] += (double)acc[zz][i] * (double)LaneVec<T, V>::at(ny, i);
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i)
              if (orow[i]) orow[i][oc] = acc[zz][i];
          }
        }
      }
    }
    if (per_vertex) {
#pragma unroll
      for (int i = 0; i < V; ++i) red[warp * TV + lane * V + i] = rsum[i];
    }
    __syncthreads();
    if (per_vertex) {
      for (int r = threadIdx.x; r < TV; r += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < nwarp; ++w) x += red[w * TV + r];
        if (tile * TV + r < n) per_vertex[tile * TV + r] = x;
      }
    }
    if (nbuf == 1 && tile + gridDim.x < ntiles) stage(tile + gridDim.x, bufs);
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

// A single column (A' = the root vertex alone, or X_v formed in an
// epilogue): thread per vertex, then a fixed-order block reduction.
template <typename T>
__global__ void __launch_bounds__(256) k_vsum(const T *__restrict__ N, int64_t ldN, int64_t n,
                                              double *__restrict__ partials, double *__restrict__ per_vertex) {
  __shared__ double wsum_s[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)N[v * ldN];
    if (per_vertex) per_vertex[v] = x;
    s += x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) wsum_s[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) b += wsum_s[i];
    partials[blockIdx.x] = b;
  }
}

// X_v = sum of the root table's row (templates with fewer vertices than colours)
template <typename T>
__global__ void __launch_bounds__(256) k_rowsum(const T *__restrict__ R, int64_t ld, int W, int64_t n,
                                                double *__restrict__ partials, double *__restrict__ per_vertex) {
  __shared__ double wsum_s[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  double wsum = 0.0;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; v < n; v += nwarps) {
    double s = 0.0;
    for (int x = lane; x < W; x += 32) s += (double)R[v * ld + x];
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
__global__ void __launch_bounds__(256) k_pack(const T *__restrict__ src, int64_t ld, int64_t c0, int64_t w,
                                              const int32_t *__restrict__ idx, int64_t rows, T *__restrict__ out,
                                              int64_t ldo) {
  using VT = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const int64_t nvec = (w + VW - 1) / VW;  // a ragged chunk's last vector reads the row's padding
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; i < rows; i += nwarps) {
    const VT *s = reinterpret_cast<const VT *>(src + (int64_t)idx[i] * ld + c0);
    VT *o = reinterpret_cast<VT *>(out + i * ldo);
    for (int64_t j = lane; j < nvec; j += 32) o[j] = __ldg(s + j);
  }
}

template <typename T, int V>
void combine_go(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint32_t *split,
                int nq, int64_t n, void *out, int64_t ldO, int WO, int o_lo, int o_hi, int num_sms, cudaStream_t s) {
  auto kern = k_combine<T, V>;
  const size_t smem = (size_t)(V == Vec<T>::W ? V : V + Vec<T>::W) * (WA + WN) * sizeof(T);
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = std::min(256, (o_hi - o_lo + 31) / 32 * 32);  // one thread per output column
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  kern<<<grid, threads, smem, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, split, nq,
                                   n, static_cast<T *>(out), ldO, WO, o_lo, o_hi);
}

// Output colour sets [o_lo, o_hi) only (a column chunk of the output table;
// out is then the chunk's virtual base: column o of row v at out[v * ldO + o]).
template <typename T>
int combine_typed(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint32_t *split,
                   int nq, int64_t n, void *out, int64_t ldO, int WO, int o_lo, int o_hi, const Knobs &kn,
                   int num_sms, cudaStream_t s) {
  const size_t split_bytes = (size_t)nq * ((WO + 7) & ~7) * 4;
  const size_t cap = 227 * 1024;
  // V = 2 vertices per lane (one address per 2 FMAs, single-buffered
  // 64-vertex tiles) when that tile plus the whole split table fits; else
  // V = 1 double-buffered with the whole table; else V = 1 single-buffered
  // with the outputs in chunks whose table slices fit (configs[4]'s (7;4,3)).
  const size_t tile2 = ((size_t)(WA + WN) * 33 * 2 * sizeof(T) + 15) / 16 * 16;
  const size_t tile1 = ((size_t)(WA + WN) * 33 * sizeof(T) + 15) / 16 * 16;
  int V = 1, nbuf = 1, chunk = WO;
  if (tile2 + split_bytes <= cap) V = 2;
  else if (2 * tile1 + split_bytes <= cap) nbuf = 2;
  else if (tile1 + (size_t)nq * 4 * 64 <= cap) chunk = (int)((cap - tile1) / ((size_t)nq * 4) / 8 * 8);
  else chunk = 0;  // even 64 outputs do not fit: V-tile kernel
  const size_t tile_bytes = V == 2 ? tile2 : tile1;
  // the lane kernel pays a staging pass per tile: it wins only when the
  // split walk does enough FMAs per staged entry (measured: (9;6,3) of
  // config 3 at 11.7 FMA/entry wins, config 2's (7;4,3) at 6.7 and (4;3,1)
  // at 2.1 lose)
  const double intensity = (double)(o_hi - o_lo) * nq / (double)(WA + WN + (o_hi - o_lo));
  const bool lane_ok = kn.combine_impl >= 2 ? kn.combine_impl == 2 : intensity >= 8.0;
  if (lane_ok && chunk > 0) {
    const int WOcp = (std::min(chunk, o_hi - o_lo) + 7) & ~7;
    const size_t smem = nbuf * tile_bytes + (size_t)nq * WOcp * 4;
    // 16 warps; output groups of 4 or 8 colour sets, whichever balances the warps better
    const int r8 = ((WOcp + 7) / 8 + 15) / 16, r4 = ((WOcp + 3) / 4 + 15) / 16;
    const bool o8 = 2 * r8 <= r4;
    auto kern = V == 2 ? (o8 ? k_combine_lane<T, 8, 2> : k_combine_lane<T, 4, 2>)
                       : (o8 ? k_combine_lane<T, 8, 1> : k_combine_lane<T, 4, 1>);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = persistent_grid(kern, 512, smem, num_sms);
    int launches = 0;
    for (int o0 = o_lo; o0 < o_hi; o0 += chunk, ++launches)
      kern<<<grid, 512, smem, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, split, nq,
                                   n, static_cast<T *>(out), ldO, WO, nbuf, o0, std::min(chunk, o_hi - o0));
    return launches;
  }
  // low-intensity steps with short rows: warp per vertex (knob combine_impl 4;
  // auto when the rows fit a warp's prefetch registers and the split slice fits)
  {
    const int nout = o_hi - o_lo;
    const size_t ssb = ((size_t)nq * nout * 4 + 15) & ~(size_t)15;
    const size_t smem = ssb + (size_t)8 * (WA + WN) * sizeof(T);
    const bool warp_ok = kn.combine_impl == 4 || (kn.combine_impl == 0 && WA <= 128 && WN <= 128);
    if (warp_ok && WA <= 128 && WN <= 128 && (nq == 2 || nq == 3) && nout <= 256 && kn.combine_wreg) {
      const size_t rsm = (size_t)8 * (WA + WN) * sizeof(T);
      // (outputs per lane NO = 2, 6 or 8; rows per lane PF = 1, 2 or 4)
      const int pf = (WA <= 32 && WN <= 32) ? 1 : (WA <= 64 && WN <= 64) ? 2 : 4;
      const int no = nout <= 64 ? 2 : nout <= 192 ? 6 : 8;
      using KW = decltype(&k_combine_wreg<T, 1, 2, 2>);
      KW tab[3][2][3] = {{{k_combine_wreg<T, 1, 2, 2>, k_combine_wreg<T, 1, 2, 6>, k_combine_wreg<T, 1, 2, 8>},
                          {k_combine_wreg<T, 1, 3, 2>, k_combine_wreg<T, 1, 3, 6>, k_combine_wreg<T, 1, 3, 8>}},
                         {{k_combine_wreg<T, 2, 2, 2>, k_combine_wreg<T, 2, 2, 6>, k_combine_wreg<T, 2, 2, 8>},
                          {k_combine_wreg<T, 2, 3, 2>, k_combine_wreg<T, 2, 3, 6>, k_combine_wreg<T, 2, 3, 8>}},
                         {{k_combine_wreg<T, 4, 2, 2>, k_combine_wreg<T, 4, 2, 6>, k_combine_wreg<T, 4, 2, 8>},
                          {k_combine_wreg<T, 4, 3, 2>, k_combine_wreg<T, 4, 3, 6>, k_combine_wreg<T, 4, 3, 8>}}};
      KW kern = tab[pf == 1 ? 0 : pf == 2 ? 1 : 2][nq - 2][no == 2 ? 0 : no == 6 ? 1 : 2];
      const int grid = persistent_grid(kern, 256, rsm, num_sms);
      kern<<<grid, 256, rsm, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, split, n,
                                  static_cast<T *>(out), ldO, WO, o_lo, o_hi);
      return 1;
    }
    if (warp_ok && WA <= 128 && WN <= 128 && smem <= 200 * 1024) {
      auto kern = (WA <= 32 && WN <= 32)   ? k_combine_warp<T, 1>
                  : (WA <= 64 && WN <= 64) ? k_combine_warp<T, 2>
                                           : k_combine_warp<T, 4>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = persistent_grid(kern, 256, smem, num_sms);
      kern<<<grid, 256, smem, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, split, nq,
                                   n, static_cast<T *>(out), ldO, WO, o_lo, o_hi);
      return 1;
    }
  }
  // wide rows: tile of V vertices (padded rows); k <= 16 bounds a row by
  // 2 x C(15,7) entries, so the smallest tile always fits in 227 KB
  const size_t row = (size_t)(WA + WN) * sizeof(T);
  const size_t budget = 100 * 1024;
  if (row * 20 <= budget) { combine_go<T, 16>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, num_sms, s); return 1; }
  else if (row * 12 <= budget) { combine_go<T, 8>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, num_sms, s); return 1; }
  else if (sizeof(T) == 4 || row * 6 <= 220 * 1024)
    combine_go<T, 4>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, num_sms, s);
  else combine_go<T, sizeof(T) == 8 ? 2 : 4>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, num_sms, s);
  return 1;
}

}  // namespace

int root_partials_blocks(int num_sms) { return num_sms * 8; }

int launch_color(const int32_t *orig, int64_t n, uint64_t seed, int k, uint8_t *out, cudaStream_t s) {
  if (n == 0) return 0;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_color<<<grid, 256, 0, s>>>(orig, n, seed, k, out);
  return 1;
}

int launch_permute_colors(const uint8_t *by_orig, const int32_t *orig, int64_t n, int k, uint8_t *out, unsigned *bad,
                          cudaStream_t s) {
  if (n == 0) return 0;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_permute_colors<<<grid, 256, 0, s>>>(by_orig, orig, n, k, out, bad);
  return 1;
}

bool combine_z_supported(int elem, int ts, int as) {
  // instantiated shapes: (t'; a') = (8; 5) -- configs[3]'s (9;6,3) -- and
  // (6; 3) -- configs[2] and [4]'s (7;4,3); fp64 only for (6; 3) (registers)
  if (ts == 8 && as == 5) return elem == 4;
  return ts == 6 && as == 3;
}

namespace {
template <typename T, int ZS, int AS>
int z_go(const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, const uint16_t *ztab, int nblocks,
         int zld, int64_t n, void *out, int64_t ldO, int num_sms, cudaStream_t s, const uint16_t *comp = nullptr,
         double *per_vertex = nullptr, bool kn_zglobal = true) {
  const size_t cap = 227 * 1024;
  const size_t tile = ((size_t)(WA + WN) * 33 * sizeof(T) + 15) / 16 * 16;
  // (+ the fused root's per-warp vertex sums: 16 warps x 32 doubles)
  const size_t zbytes = ((size_t)nblocks * zld * 4 + 7) / 8 * 8 + (per_vertex ? 16 * 32 * 8 : 0);
  if (tile + zbytes > cap) {
    // the cover in global memory (16-byte aligned blocks of zld entries): two
    // single-buffered CTAs of 8 warps per SM when two tiles fit
    if (!kn_zglobal || (zld * 2) % 16 != 0) return 0;
    const size_t tb = (size_t)16 * 4 * zld * 2;  // per-warp raw double buffer + ready offsets
    const size_t gz = (per_vertex ? 16 * 32 * 8 : 0) + tb;
    if (tile + gz > cap) return 0;
    const int threads = 2 * (tile + gz) <= cap ? 256 : 512;
    auto kern = k_combine_z<T, ZS, AS, 1, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(tile + gz));
    const int grid = persistent_grid(kern, threads, tile + gz, num_sms);
    kern<<<grid, threads, tile + gz, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, ztab,
                                          nblocks, zld, n, static_cast<T *>(out), ldO, 1, comp, per_vertex);
    return 1;
  }
  // two single-buffered CTAs of 8 warps per SM when they fit (one computes
  // while the other stages or waits at its barrier; measured 5% faster on
  // config 3), else one CTA of 16 warps, double-buffered when it fits
  int nbuf = 2 * tile + zbytes <= cap ? 2 : 1, threads = 512;
  if (2 * (tile + zbytes) <= cap) {
    nbuf = 1;
    threads = 256;
  }
  const size_t smem = nbuf * tile + zbytes;
  auto kern = k_combine_z<T, ZS, AS, 1>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, threads, smem, num_sms);
  kern<<<grid, threads, smem, s>>>(static_cast<const T *>(A), ldA, WA, static_cast<const T *>(N), ldN, WN, ztab,
                                   nblocks, zld, n, static_cast<T *>(out), ldO, nbuf, comp, per_vertex);
  return 1;
}
}  // namespace

int launch_combine_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                        const uint16_t *ztab, int nblocks, int zld, int ts, int as, const uint16_t *comp, int64_t n,
                        double *per_vertex, const Knobs &kn, int num_sms, cudaStream_t s) {
  if (n == 0 || !ztab || !comp || !per_vertex) return 0;
  if (kn.combine_impl >= 2) return 0;
  if (const int l = launch_combine_static(elem, A, ldA, WA, N, ldN, WN, ts, as, n, nullptr, 0, per_vertex, kn, num_sms, s))
    return l;
  if (elem == 4 && ts == 8 && as == 5)
    return z_go<float, 9, 5>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, nullptr, 0, num_sms, s, comp, per_vertex, kn.combine_zglobal);
  if (elem == 4 && ts == 6 && as == 3)
    return z_go<float, 7, 3>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, nullptr, 0, num_sms, s, comp, per_vertex, kn.combine_zglobal);
  if (elem == 8 && ts == 6 && as == 3)
    return z_go<double, 7, 3>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, nullptr, 0, num_sms, s, comp, per_vertex, kn.combine_zglobal);
  return 0;
}

int launch_combine(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                   const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, const uint16_t *ztab,
                   int nblocks, int zld, int ts, int as, const Knobs &kn, int num_sms, cudaStream_t s) {
  if (n == 0) return 0;
  if (ztab && kn.combine_impl <= 1) {  // the Z-block kernel when the shape has one
    int l = launch_combine_static(elem, A, ldA, WA, N, ldN, WN, ts, as, n, out, ldO, nullptr, kn, num_sms, s);
    if (l) return l;
    if (elem == 4 && ts == 8 && as == 5) l = z_go<float, 9, 5>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, out, ldO, num_sms, s, nullptr, nullptr, kn.combine_zglobal);
    else if (elem == 4 && ts == 6 && as == 3) l = z_go<float, 7, 3>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, out, ldO, num_sms, s, nullptr, nullptr, kn.combine_zglobal);
    else if (elem == 8 && ts == 6 && as == 3) l = z_go<double, 7, 3>(A, ldA, WA, N, ldN, WN, ztab, nblocks, zld, n, out, ldO, num_sms, s, nullptr, nullptr, kn.combine_zglobal);
    if (l) return l;
  }
  if (elem == 8)
    return combine_typed<double>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, 0, WO, kn, num_sms, s);
  return combine_typed<float>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, 0, WO, kn, num_sms, s);
}

int launch_combine_cols(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                        const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, int o_lo, int o_hi,
                        const Knobs &kn, int num_sms, cudaStream_t s) {
  if (n == 0 || o_lo >= o_hi) return 0;
  if (elem == 8)
    return combine_typed<double>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, kn, num_sms, s);
  return combine_typed<float>(A, ldA, WA, N, ldN, WN, split, nq, n, out, ldO, WO, o_lo, o_hi, kn, num_sms, s);
}

int launch_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, const uint16_t *comp,
                int64_t n, double *partials, int n_partials, double *per_vertex, double *result, cudaStream_t s) {
  if (!A && elem == 8)
    k_vsum<double><<<n_partials, 256, 0, s>>>(static_cast<const double *>(N), ldN, n, partials, per_vertex);
  else if (!A)
    k_vsum<float><<<n_partials, 256, 0, s>>>(static_cast<const float *>(N), ldN, n, partials, per_vertex);
  else if (elem == 8)
    k_root<double><<<n_partials, 256, 0, s>>>(static_cast<const double *>(A), ldA, WA, static_cast<const double *>(N),
                                               ldN, comp, n, partials, per_vertex);
  else
    k_root<float><<<n_partials, 256, 0, s>>>(static_cast<const float *>(A), ldA, WA, static_cast<const float *>(N),
                                              ldN, comp, n, partials, per_vertex);
  k_reduce<<<1, 32, 0, s>>>(partials, n_partials, result);
  return 2;
}

int launch_rowsum(int elem, const void *R, int64_t ld, int W, int64_t n, double *partials, int n_partials,
                  double *per_vertex, double *result, cudaStream_t s) {
  if (elem == 8)
    k_rowsum<double><<<n_partials, 256, 0, s>>>(static_cast<const double *>(R), ld, W, n, partials, per_vertex);
  else
    k_rowsum<float><<<n_partials, 256, 0, s>>>(static_cast<const float *>(R), ld, W, n, partials, per_vertex);
  k_reduce<<<1, 32, 0, s>>>(partials, n_partials, result);
  return 2;
}

int launch_pack(int elem, const void *src, int64_t ld, int64_t c0, int64_t w, const int32_t *idx, int64_t rows,
                void *out, int64_t ldo, cudaStream_t s) {
  if (rows == 0 || w == 0) return 0;
  const int grid = (int)std::min<int64_t>((rows + 7) / 8, 148 * 8);
  if (elem == 8)
    k_pack<double><<<grid, 256, 0, s>>>(static_cast<const double *>(src), ld, c0, w, idx, rows,
                                        static_cast<double *>(out), ldo);
  else
    k_pack<float><<<grid, 256, 0, s>>>(static_cast<const float *>(src), ld, c0, w, idx, rows,
                                       static_cast<float *>(out), ldo);
  return 1;
}

}  // namespace dev
}  // namespace cc
