// Microbenchmark (not product code): random row gathers through TMA
// tile::gather4 (4 rows per request into a shared-memory stage ring, mbarrier
// completion) against plain LDG.128 rows, on a table >> L2.  Decides whether
// the lean neighbour-sum gathers should land their rows by TMA (VERDICT r1
// "next round" 5).  Prints GB/s of row bytes per variant.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, int c0, int r0, int r1, int r2, int r3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

// warp 0 lane 0: producer; warps 1..C: consumers (stage i -> consumer (i mod C))
template <int S, int NREQ, int CW, int C>
__global__ void __launch_bounds__(32 * (C + 1)) k_tma4(const __grid_constant__ CUtensorMap tm,
                                                       const int32_t *__restrict__ idx, int64_t ngroups, float *out) {
  constexpr int STAGE = NREQ * 4 * CW * 4;  // bytes
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)S * STAGE);
  uint64_t *empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int64_t i = 0;
      for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++i) {
        const int st = (int)(i % S);
        const uint32_t use = (uint32_t)(i / S);
        if (use) mbar_wait(empty + st, (use - 1) & 1);
        const int4 r = __ldg(reinterpret_cast<const int4 *>(idx) + g);
        mbar_expect_tx(full + st, STAGE);
#pragma unroll
        for (int q = 0; q < NREQ; ++q)
          tma_gather4(sm + (size_t)st * STAGE + q * 4 * CW * 4, &tm, q * CW, r.x, r.y, r.z, r.w, full + st);
      }
    }
    return;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  int64_t i = warp - 1;
  for (int64_t g = blockIdx.x + (int64_t)(warp - 1) * gridDim.x; g < ngroups; g += (int64_t)C * gridDim.x, i += C) {
    const int st = (int)(i % S);
    mbar_wait(full + st, (uint32_t)(i / S) & 1);
    const float4 *p = reinterpret_cast<const float4 *>(sm + (size_t)st * STAGE);
    for (int v = lane; v < STAGE / 16; v += 32) {
      const float4 x = p[v];
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// Each warp issues its own gather4 requests into a private ring of S stages
// (lane 0 issues, the warp consumes in order and re-issues into the freed
// stage): the layout the short-list gather would use.
template <int S, int NREQ, int CW, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_tma_self(const __grid_constant__ CUtensorMap tm,
                                                         const int32_t *__restrict__ idx, int64_t ngroups, float *out) {
  constexpr int STAGE = NREQ * 4 * CW * 4;
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *ring = sm + (size_t)warp * S * STAGE;
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)WARPS * S * STAGE) + warp * S;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nwg = (int64_t)gridDim.x * WARPS;
  const int64_t per = (ngroups + nwg - 1) / nwg, g0 = gw * per, g1 = g0 + per < ngroups ? g0 + per : ngroups;
  auto issue = [&](int64_t g) {
    const int st = (int)((g - g0) % S);
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int4 r = __ldg(reinterpret_cast<const int4 *>(idx) + g);
      mbar_expect_tx(full + st, STAGE);
#pragma unroll
      for (int q = 0; q < NREQ; ++q)
        tma_gather4(ring + (size_t)st * STAGE + q * 4 * CW * 4, &tm, q * CW, r.x, r.y, r.z, r.w, full + st);
    }
  };
  for (int64_t g = g0; g < g1 && g < g0 + S; ++g) issue(g);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t g = g0; g < g1; ++g) {
    const int st = (int)((g - g0) % S);
    mbar_wait(full + st, (uint32_t)((g - g0) / S) & 1);
    const float4 *p = reinterpret_cast<const float4 *>(ring + (size_t)st * STAGE);
    for (int v = lane; v < STAGE / 16; v += 32) {
      const float4 x = p[v];
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
    }
    __syncwarp();
    if (g + S < g1) issue(g + S);
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

template <int NV, int U>
__global__ void __launch_bounds__(256) k_rows(const float4 *__restrict__ tab, int64_t ld_vec, int nvec,
                                              const int32_t *__restrict__ idx, int64_t nreads, float *out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t r0 = w * U; r0 < nreads; r0 += nw * U) {
    float4 x[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u < nreads ? r0 + u : r0;
      const float4 *row = tab + (int64_t)__ldg(idx + r) * ld_vec + lane;
#pragma unroll
      for (int j = 0; j < NV; ++j) x[u][j] = lane + 32 * j < nvec ? __ldg(row + 32 * j) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        acc.x += x[u][j].x;
        acc.y += x[u][j].y;
        acc.z += x[u][j].z;
        acc.w += x[u][j].w;
      }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int S, int NREQ, int CW, int C>
void run_tma(EncodeTiled enc, float4 *tab, int64_t rows, int64_t ld, const int32_t *idx, int64_t nreads, float *out,
             int sms, int ctas_per_sm, const char *name) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {CW, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("{\"variant\": \"%s\", \"encode_error\": %d}\n", name, (int)r);
    return;
  }
  constexpr int STAGE = NREQ * 4 * CW * 4;
  const size_t smem = (size_t)S * STAGE + 2 * S * 8;
  auto kern = k_tma4<S, NREQ, CW, C>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    kern<<<sms * ctas_per_sm, 32 * (C + 1), smem>>>(tm, idx, nreads / 4, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2)
      printf("{\"variant\": \"%s\", \"row_bytes\": %d, \"smem_kb\": %.1f, \"ctas_per_sm\": %d, \"ms\": %.3f, "
             "\"row_GBs\": %.1f, \"err\": \"%s\"}\n",
             name, NREQ * CW * 4, smem / 1024.0, ctas_per_sm, ms, (double)nreads * NREQ * CW * 4 / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
  }
}

template <int S, int NREQ, int CW, int WARPS>
void run_self(EncodeTiled enc, float4 *tab, int64_t rows, int64_t ld, const int32_t *idx, int64_t nreads, float *out,
              int sms, int ctas_per_sm, const char *name) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {CW, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("{\"variant\": \"%s\", \"encode_error\": %d}\n", name, (int)r);
    return;
  }
  constexpr int STAGE = NREQ * 4 * CW * 4;
  const size_t smem = (size_t)WARPS * S * STAGE + (size_t)WARPS * S * 8;
  auto kern = k_tma_self<S, NREQ, CW, WARPS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    kern<<<sms * ctas_per_sm, 32 * WARPS, smem>>>(tm, idx, nreads / 4, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep == 2)
      printf("{\"variant\": \"%s\", \"row_bytes\": %d, \"smem_kb\": %.1f, \"ctas_per_sm\": %d, \"ms\": %.3f, "
             "\"row_GBs\": %.1f, \"err\": \"%s\"}\n",
             name, NREQ * CW * 4, smem / 1024.0, ctas_per_sm, ms, (double)nreads * NREQ * CW * 4 / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  const int64_t rows = 5351589;
  const int64_t nreads = 464000000;
  std::vector<int32_t> h(nreads);
  std::mt19937_64 rng(7);
  for (auto &x : h) x = (int32_t)(rng() % rows);
  int32_t *idx;
  cudaMalloc(&idx, nreads * 4);
  cudaMemcpy(idx, h.data(), nreads * 4, cudaMemcpyHostToDevice);
  float *out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeTiled enc = (EncodeTiled)fn;
  // p = 5 rows of configs[3]: 330 fp32 columns (1320 B), ld 336
  {
    const int64_t ld = 336;
    float4 *tab;
    cudaMalloc(&tab, rows * ld * 4);
    cudaMemset(tab, 0, rows * ld * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_rows<3, 4><<<sms * 8, 256>>>(tab, ld / 4, 83, idx, nreads, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("{\"variant\": \"ldg U4\", \"row_bytes\": 1328, \"ms\": %.3f, \"row_GBs\": %.1f, \"err\": \"%s\"}\n", ms,
               (double)nreads * 1328 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    run_tma<8, 2, 168, 4>(enc, tab, rows, ld, idx, nreads, out, sms, 4, "tma4 S8 2x168 C4 x4");
    run_tma<16, 2, 168, 4>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "tma4 S16 2x168 C4 x2");
    run_tma<32, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "tma4 S32 2x168 C8 x1");
    run_tma<24, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "tma4 S24 2x168 C8 x1");
    run_tma<12, 2, 168, 4>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "tma4 S12 2x168 C4 x2");
    run_self<4, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "self S4 2x168 W8 x1");
    run_self<5, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "self S5 2x168 W8 x1");
    run_self<3, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "self S3 2x168 W8 x1");
    run_self<2, 2, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "self S2 2x168 W8 x2");
    run_self<5, 2, 168, 4>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "self S5 2x168 W4 x2");
    cudaFree(tab);
  }
  // p = 4 rows: 165 columns (660 B), ld 168
  {
    const int64_t ld = 168;
    float4 *tab;
    cudaMalloc(&tab, rows * ld * 4);
    cudaMemset(tab, 0, rows * ld * 4);
    run_tma<16, 1, 168, 4>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "tma4 p4 S16 1x168 C4 x2");
    run_tma<32, 1, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "tma4 p4 S32 1x168 C8 x1");
    run_tma<48, 1, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "tma4 p4 S48 1x168 C8 x1");
    run_self<8, 1, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 1, "self p4 S8 1x168 W8 x1");
    run_self<5, 1, 168, 8>(enc, tab, rows, ld, idx, nreads, out, sms, 2, "self p4 S5 1x168 W8 x2");
    cudaFree(tab);
  }
  return 0;
}
