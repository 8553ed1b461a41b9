// Microbenchmark (not product code): the practical DRAM ceiling of a random
// row gather on this GPU.  A table of R rows x B bytes (>> L2) is read in a
// uniformly random row order, one warp per row, 16-byte loads, and summed.
// Prints GB/s of row bytes.  Used to judge the gather kernels' DRAM fraction
// against what random ~1 KB row reads can reach (profiles/r1/SUMMARY.md).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

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
        acc.x += x[u][j].x; acc.y += x[u][j].y; acc.z += x[u][j].z; acc.w += x[u][j].w;
      }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

int main(int argc, char **argv) {
  const int64_t rows = 5351589;
  const int nvec_list[] = {83, 42, 14};  // p = 5, 4, 3 rows of configs[3] (16-byte vectors)
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
  for (int nvec : nvec_list) {
    const int64_t ld_vec = (nvec + 1) / 2 * 2;  // 32-byte padded rows
    float4 *tab;
    cudaMalloc(&tab, rows * ld_vec * 16);
    cudaMemset(tab, 0, rows * ld_vec * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (nvec > 64) k_rows<3, 4><<<sms * 8, 256>>>(tab, ld_vec, nvec, idx, nreads, out);
      else if (nvec > 32) k_rows<2, 8><<<sms * 8, 256>>>(tab, ld_vec, nvec, idx, nreads, out);
      else k_rows<1, 8><<<sms * 8, 256>>>(tab, ld_vec, nvec, idx, nreads, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)nreads * nvec * 16;
      if (rep == 2)
        printf("{\"row_bytes\": %d, \"reads\": %lld, \"ms\": %.3f, \"row_GBs\": %.1f, \"err\": \"%s\"}\n", nvec * 16,
               (long long)nreads, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(tab);
  }
  return 0;
}
