// kernels.cuh -- device kernels of the colour-coding DP (sm_100a) and their
// host launchers.  All kernels are templated on the table storage type T
// (double for CC_FP64, float for CC_FP32); neighbour sums and root products
// accumulate in double.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cc {
namespace dev {

// Work list of one aggregation pass (Alg. 4: the
// neighbour list of a vertex is cut into tasks of at most s neighbours).
//   light[i]       vertices whose [beg, end) range has <= s neighbours
//   seg_*          segments of heavy vertices, grouped per heavy vertex
//   hv_first/nseg  first segment and segment count of heavy vertex h
struct AggWork {
  const int32_t *light = nullptr;
  int64_t n_light = 0;
  const int32_t *seg_v = nullptr;
  const int64_t *seg_b = nullptr, *seg_e = nullptr;
  const int32_t *seg_hv = nullptr;
  const int32_t *hv_first = nullptr, *hv_nseg = nullptr;
  int64_t n_seg = 0, n_hv = 0;
};

struct AggArgs {
  const int64_t *beg;    // per vertex: first neighbour position
  const int64_t *end;    // per vertex: one past the last
  const int32_t *col;    // neighbour row ids into src
  const void *src;       // passive table P (rows x ld_src)
  int64_t ld_src;
  void *dst;             // N (rows x ld_dst)
  int64_t ld_dst;
  int W;                 // valid columns
  int accumulate;        // 0: dst = sum; 1: dst += sum
  double *scratch;       // n_seg x W_pad doubles (heavy partials)
  int64_t ld_scratch;
  unsigned int *arrive;  // n_hv x nchunks counters (zeroed before launch)
  AggWork work;
};

// Launchers.  `elem` = sizeof(T) (8 or 4).  Return the number of launches.
int launch_color(const int32_t *orig, int64_t n, uint64_t seed, int k, uint8_t *out, cudaStream_t s);
int launch_hist(int elem, const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                const AggWork &work, int64_t n, int k, void *out, int64_t ld, int num_sms, cudaStream_t s);
// Aggregation: chooses group width / chunking from W and chunk_cols.
int launch_agg(int elem, const AggArgs &a, int64_t chunk_cols, int num_sms, int *nchunks_out,
               cudaStream_t s);
int launch_lift(int elem, const void *N, int64_t ldN, const uint8_t *colors, const uint16_t *drop,
                int64_t n, int Wt, void *out, int64_t ldO, int num_sms, cudaStream_t s);
int launch_combine(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                   const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, int num_sms,
                   cudaStream_t s);
// Root step + deterministic reduction into result[0] (double).  A == nullptr
// means the single-vertex active part (a = 1): sum_v N(v, comp1[col v]).
int launch_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN,
                const uint16_t *comp, const uint8_t *colors, int64_t n, double *partials,
                int n_partials, double *per_vertex, double *result, cudaStream_t s);
// Halo pack: out[i, :] = src[idx[i], :] for i < rows (whole padded rows).
int launch_pack(int elem, const void *src, int64_t ld, const int32_t *idx, int64_t rows, void *out,
                cudaStream_t s);

int agg_partials_blocks(int num_sms);  // grid size used by launch_root partials
int agg_nchunks(int elem, int W, int64_t chunk_cols);  // column chunks launch_agg will use

}  // namespace dev
}  // namespace cc
