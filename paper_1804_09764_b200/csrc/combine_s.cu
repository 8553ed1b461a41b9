// combine_s.cu -- the split sum of Eq. 1 for the combine
// shapes whose outputs are the (K-3)-colour sets of the compressed K = k-1
// colour universe, with the whole cover fixed at compile time (sm_100a).
//
//   T'(v, S') = sum_{X' u Y'' = S', |X'| = AS} A'(v, X') N''(v, Y'')
//
// k_combine_z (kernels.cu) reads its Z-block cover from a table at run time:
// every shared-memory load costs an address add and a quarter of a table
// load, and 36% of its FMAs recompute outputs another block owns.  Here the
// colour sets are colex-ranked at compile time, so:
//
//   * the blocks are Z = [K] \ {i, j} for the pairs {i, j} inside one half of
//     the universe ({0..K/2-1} or {K/2..K-1}).  An output S' misses exactly
//     three colours; two of them share a half, so some block contains S'
//     (the complement of a triangle-free Turan graph: C(K/2,2)+C(K-K/2,2)
//     blocks, 25 for K = 11 -- the Schoenheim lower bound, so the cover is
//     minimum).
//   * every output is OWNED by one block (the least loaded candidate, in
//     colex order of the missing triples): no redundant FMA, exactly
//     C(K,TS) x C(TS,AS) per vertex.
//   * every shared-memory load is [lane base + immediate] (no address math,
//     no table), the register indices of the Z-block passives are immediates
//     too, and loops over unowned outputs vanish at compile time.
//   * the blocks are dealt to NW warps by longest-processing-time over their
//     FMA + load counts (K = 11: 5 warps x 5 blocks, exactly balanced); a
//     warp runs straight-line code for its own blocks (~3 K instructions,
//     well inside the measured instruction-prefetch regime).
//
// Tiles of 32 vertices' A' and N'' rows are staged TRANSPOSED ([column][33])
// by cp.async as in k_combine_z; two CTAs per SM, so one stages while the
// other computes.  With ROOT the output is not stored: each T'(v, S') is
// multiplied in fp64 by N''(v, [K] \ S') and summed into X_v in a fixed
// order (fused root, reading C-15); otherwise T' is stored.  fp32 tables only
// (the Z-block passives of one block live in registers).
#include <cstdint>

#include "dev_common.cuh"

namespace cc {
namespace dev {

namespace {

__host__ __device__ constexpr int sbin(int n, int r) {
  if (r < 0 || n < 0 || r > n) return 0;
  int c = 1;
  for (int i = 1; i <= r; ++i) c = c * (n - r + i) / i;
  return c;
}

constexpr uint32_t kCB = 33 * sizeof(float);  // bytes per staged column ([column][33 lanes])

// the per-warp straight-line block code (gen_combine_s.py, emitted into build/gen at build time)
#include "combine_s_gen.cuh"

template <int K, int AS, bool ROOT>
__device__ __forceinline__ void s_dispatch(int warp, const char *Ab, const char *Nb, double &rsum, float *orow, bool ok) {
  if constexpr (K == 11 && AS == 5) s_dispatch_11_5<ROOT>(warp, Ab, Nb, rsum, orow, ok);
  else s_dispatch_9_3<ROOT>(warp, Ab, Nb, rsum, orow, ok);
}

template <int K, int AS, int NW, int MINB, bool ROOT>
__global__ void __launch_bounds__(32 * NW) __maxnreg__(65536 / (32 * NW * MINB) / 8 * 8) k_combine_s(const float *__restrict__ A, int64_t ldA,
                                                             const float *__restrict__ N, int64_t ldN, int64_t n,
                                                             float *__restrict__ out, int64_t ldO,
                                                             double *__restrict__ per_vertex) {
  constexpr int WA = sbin(K, AS), WN = sbin(K, K - 3 - AS);  // NOLINT
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float *tile = reinterpret_cast<float *>(smem_raw);
  double *red = reinterpret_cast<double *>(smem_raw + ((size_t)(WA + WN) * kCB + 15) / 16 * 16);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntiles = (n + 31) / 32;
  const char *Ab = reinterpret_cast<const char *>(tile + lane);
  const char *Nb = Ab + (size_t)WA * kCB;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t v0 = tl * 32;
    for (int r = warp; r < 32; r += NW) {
      const bool ok = v0 + r < n;
      const int64_t vr = ok ? v0 + r : 0;
      const float *ar = A + vr * ldA, *nr = N + vr * ldN;
      const unsigned d = (unsigned)__cvta_generic_to_shared(tile + r);
      for (int x = lane; x < WA; x += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d + x * kCB), "l"(ar + x), "r"(ok ? 4 : 0)
                     : "memory");
      for (int x = lane; x < WN; x += 32)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d + (WA + x) * kCB), "l"(nr + x),
                     "r"(ok ? 4 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    double rsum = 0.0;
    const bool ok = v0 + lane < n;
    float *orow = ROOT ? nullptr : out + (ok ? v0 + lane : 0) * ldO;
    s_dispatch<K, AS, ROOT>(warp, Ab, Nb, rsum, orow, ok);
    if constexpr (ROOT) red[warp * 32 + lane] = rsum;
    __syncthreads();  // the tile is restaged next iteration; red is complete
    if constexpr (ROOT) {
      if (threadIdx.x < 32 && v0 + threadIdx.x < n) {
        double x = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) x += red[w * 32 + threadIdx.x];
        per_vertex[v0 + threadIdx.x] = x;
      }
    }
  }
}

template <int K, int AS, int NW, int MINB>
int s_go(const float *A, int64_t ldA, const float *N, int64_t ldN, int64_t n, float *out, int64_t ldO,
         double *per_vertex, int num_sms, cudaStream_t s) {
  constexpr int WA = sbin(K, AS), WN = sbin(K, K - 3 - AS);
  const size_t smem = ((size_t)(WA + WN) * kCB + 15) / 16 * 16 + (size_t)NW * 32 * sizeof(double);
  auto kern = per_vertex ? k_combine_s<K, AS, NW, MINB, true> : k_combine_s<K, AS, NW, MINB, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = persistent_grid(kern, 32 * NW, smem, num_sms);
  kern<<<grid, 32 * NW, smem, s>>>(A, ldA, N, ldN, n, out, ldO, per_vertex);
  return 1;
}

}  // namespace

// The compile-time cover exists for (K; TS = K - 3, AS) = (9; 6, 3) (configs[2]'s
// (7;4,3) at k = 10: 16 blocks, ~50 KB of code; measured 0.33 -> 0.25 ms for the
// combine phase) and (11; 8, 5) (configs[3]'s (9;6,3) at k = 12), fp32 tables
// stored in colex column order (layout knob 0).  The (11; 8, 5) kernel runs
// only with combine_static = 2: its 25 blocks are ~240 KB of straight-line
// code, 5 different streams per CTA, and the warps starve on instruction
// fetch (ncu: 8.8 warps stalled on no_instruction per issue, issue active
// 20%): 16.4 ms against 8.8 ms for k_combine_z's 2 KB loop
// (profiles/r2/SUMMARY.md).
int launch_combine_static(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, int ts,
                          int as, int64_t n, void *out, int64_t ldO, double *per_vertex, const Knobs &kn, int num_sms,
                          cudaStream_t s) {
  if (n == 0 || elem != 4 || kn.layout != 0 || !kn.combine_static || kn.combine_impl >= 2) return 0;
  const float *a = static_cast<const float *>(A), *nn = static_cast<const float *>(N);
  float *o = static_cast<float *>(out);
  if (ts == 8 && as == 5 && WA == sbin(11, 5) && WN == sbin(11, 3) && kn.combine_static == 2)
    return s_go<11, 5, kSWarps_11_5, 2>(a, ldA, nn, ldN, n, o, ldO, per_vertex, num_sms, s);
  if (ts == 6 && as == 3 && WA == sbin(9, 3) && WN == sbin(9, 3))
    return s_go<9, 3, kSWarps_9_3, 4>(a, ldA, nn, ldN, n, o, ldO, per_vertex, num_sms, s);
  return 0;
}

}  // namespace dev
}  // namespace cc
