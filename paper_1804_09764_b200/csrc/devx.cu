// devx.cu -- the device-initiated halo exchange (CC_EXCHANGE_DEVICE; SURVEY
// F2): the pack kernel stores each boundary row straight into the peer's
// halo window (NCCL >= 2.28 device API: a symmetric window registered by
// every rank, ncclGetLsaPointer to the peer's copy over NVLink), with an LSA
// barrier before (every rank has finished reading its window) and after
// (every rank's stores are visible).  No send buffer, no ncclSend/ncclRecv:
// PAPER.md Alg. 2 line 15 (exchange the boundary rows) as one kernel.
#include <nccl_device.h>

#include <cuda/atomic>
#include <cstring>
#include <vector>

#include "dev_common.cuh"
#include "devx.h"

namespace cc {
namespace dev {

namespace {

// One CTA per barrier slot (the grid is the same on every rank: kPutCtas).
// Rows of peer q: send positions [send_off[q], send_off[q + 1]); row i goes to
// row dst_row[q] + (i - send_off[q]) of q's window (stride ldH), columns
// [c0, c0 + w) of the source row (stride ld) to columns [0, w).
template <typename T>
__global__ void __launch_bounds__(256) k_pack_put(ncclDevComm comm, ncclWindow_t win, size_t win_off,
                                                  const T *__restrict__ src, int64_t ld, int64_t c0, int64_t w,
                                                  const int32_t *__restrict__ send_idx,
                                                  const int64_t *__restrict__ send_off,
                                                  const int64_t *__restrict__ dst_row, int world, int me,
                                                  int64_t ldH) {
  using VT = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x);
  bar.sync(ncclCoopCta(), cuda::memory_order_acquire);  // every peer is done reading its window
  const int lane = threadIdx.x & 31;
  const int64_t nvec = (w + VW - 1) / VW;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int q = 0; q < world; ++q) {
    if (q == me) continue;
    const int peer = ncclTeamRankToLsa(comm, ncclTeamWorld(comm), q);
    for (int64_t i = send_off[q] + gw; i < send_off[q + 1]; i += nw) {
      const VT *s = reinterpret_cast<const VT *>(src + (int64_t)send_idx[i] * ld + c0);
      const size_t off = win_off + (size_t)(dst_row[q] + (i - send_off[q])) * ldH * sizeof(T);
      VT *d = static_cast<VT *>(ncclGetLsaPointer(win, off, peer));
      for (int64_t j = lane; j < nvec; j += 32) d[j] = __ldg(s + j);
    }
  }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);  // my stores are out; the peers' stores to me are in
}

// One-rank self test: CTA b stores 4 values into the window through the LSA
// pointer of rank 0 (itself), syncs the barrier, and reads them back locally.
__global__ void k_put_selftest(ncclDevComm comm, ncclWindow_t win, double *out) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x);
  bar.sync(ncclCoopCta(), cuda::memory_order_acquire);
  double *d = static_cast<double *>(ncclGetLsaPointer(win, (size_t)blockIdx.x * 4 * sizeof(double), 0));
  if (threadIdx.x < 4) d[threadIdx.x] = 1000.0 * blockIdx.x + threadIdx.x;
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  const double *l = static_cast<const double *>(ncclGetLocalPointer(win, (size_t)blockIdx.x * 4 * sizeof(double)));
  if (threadIdx.x < 4) out[blockIdx.x * 4 + threadIdx.x] = l[threadIdx.x];
}

}  // namespace

int launch_pack_put(int elem, const ncclDevComm &comm, ncclWindow_t win, size_t win_off, const void *src, int64_t ld,
                    int64_t c0, int64_t w, const int32_t *send_idx, const int64_t *send_off, const int64_t *dst_row,
                    int world, int me, int64_t ldH, cudaStream_t s) {
  if (elem == 8)
    k_pack_put<double><<<kPutCtas, 256, 0, s>>>(comm, win, win_off, static_cast<const double *>(src), ld, c0, w,
                                                 send_idx, send_off, dst_row, world, me, ldH);
  else
    k_pack_put<float><<<kPutCtas, 256, 0, s>>>(comm, win, win_off, static_cast<const float *>(src), ld, c0, w,
                                                send_idx, send_off, dst_row, world, me, ldH);
  return 1;
}

int launch_put_selftest(const ncclDevComm &comm, ncclWindow_t win, double *out, cudaStream_t s) {
  k_put_selftest<<<kPutCtas, 128, 0, s>>>(comm, win, out);
  return 1;
}

}  // namespace dev
}  // namespace cc

// ---------------------------------------------------------------- host side
#include "ctx.h"

namespace cc {

struct DevX {
  ncclDevComm comm{};
  bool comm_ok = false;
  ncclWindow_t win = nullptr;
  void *buf = nullptr;
  size_t bytes = 0;
  int64_t *d_dst_row = nullptr, *d_send_off = nullptr;
};

void devx_init(cc_ctx *c, const std::vector<int64_t> &dst_row) {
  auto &api = nccl();
  if (!api.dev_ok) throw Error(CC_ERR_NCCL, "CC_EXCHANGE_DEVICE needs the NCCL >= 2.28 device API (symmetric windows)");
  if (!c->comm) throw Error(CC_ERR_ARG, "CC_EXCHANGE_DEVICE needs a NCCL communicator (not the loopback transport)");
  devx_free(c);
  c->devx = new DevX();
  ncclDevCommRequirements reqs;
  std::memset(&reqs, 0, sizeof(reqs));
  reqs.lsaBarrierCount = dev::kPutCtas;
  NCCL_OK(api.DevCommCreate(c->comm, &reqs, &c->devx->comm));
  c->devx->comm_ok = true;
  c->devx->d_dst_row = c->pupload(dst_row);
  c->devx->d_send_off = c->pupload(c->part.send_off);
}

void devx_free(cc_ctx *c) {
  if (!c->devx) return;
  auto &api = nccl();
  DevX *d = c->devx;
  cudaStreamSynchronize(c->s_comm);
  cudaStreamSynchronize(c->s_main);
  if (d->win) api.CommWindowDeregister(c->comm, d->win);
  if (d->buf) api.MemFree(d->buf);
  if (d->comm_ok) api.DevCommDestroy(c->comm, &d->comm);
  delete d;
  c->devx = nullptr;
}

// The halo window (collective: every rank asks for the same size at the same
// point of the same plan): at least `bytes`, symmetric, registered once.
void *devx_window(cc_ctx *c, size_t bytes) {
  DevX *d = c->devx;
  if (d->bytes >= bytes) return d->buf;
  auto &api = nccl();
  CUDA_OK(cudaStreamSynchronize(c->s_comm));
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  if (d->win) NCCL_OK(api.CommWindowDeregister(c->comm, d->win));
  if (d->buf) NCCL_OK(api.MemFree(d->buf));
  d->win = nullptr;
  d->buf = nullptr;
  d->bytes = 0;
  const size_t b = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
  NCCL_OK(api.MemAlloc(&d->buf, b));
  NCCL_OK(api.CommWindowRegister(c->comm, d->buf, b, &d->win, NCCL_WIN_COLL_SYMMETRIC));
  d->bytes = b;
  return d->buf;
}

// Device-initiated exchange of columns [c0, c0 + w) of P's boundary rows into
// the peers' windows at byte offset win_off (on the comm stream).
void devx_put(cc_ctx *c, const void *P, int64_t ldP, int64_t c0, int64_t w, size_t win_off, int64_t ldH) {
  DevX *d = c->devx;
  c->stats[3] += dev::launch_pack_put(c->elem(), d->comm, d->win, win_off, P, ldP, c0, w, c->d_send_idx,
                                      d->d_send_off, d->d_dst_row, c->pworld(), c->opt.rank, ldH, c->s_comm);
  c->check_launch();
}

cc_status device_selftest(int32_t device) {
  auto &api = nccl();
  if (!api.ok || !api.dev_ok) return CC_ERR_NCCL;
  ncclComm_t comm = nullptr;
  cudaStream_t s = nullptr;
  double *out = nullptr;
  void *buf = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dc{};
  bool dc_ok = false;
  cc_status st = CC_OK;
  try {
    CUDA_OK(cudaSetDevice(device));
    ncclUniqueId id;
    NCCL_OK(api.GetUniqueId(&id));
    NCCL_OK(api.CommInitRank(&comm, 1, id, 0));
    CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    NCCL_OK(api.MemAlloc(&buf, NCCL_WIN_REQUIRED_ALIGNMENT));
    NCCL_OK(api.CommWindowRegister(comm, buf, NCCL_WIN_REQUIRED_ALIGNMENT, &win, NCCL_WIN_COLL_SYMMETRIC));
    ncclDevCommRequirements reqs;
    std::memset(&reqs, 0, sizeof(reqs));
    reqs.lsaBarrierCount = dev::kPutCtas;
    NCCL_OK(api.DevCommCreate(comm, &reqs, &dc));
    dc_ok = true;
    CUDA_OK(cudaMalloc(&out, dev::kPutCtas * 4 * sizeof(double)));
    dev::launch_put_selftest(dc, win, out, s);
    CUDA_OK(cudaGetLastError());
    std::vector<double> h(dev::kPutCtas * 4);
    CUDA_OK(cudaMemcpyAsync(h.data(), out, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    for (int b = 0; b < dev::kPutCtas; ++b)
      for (int j = 0; j < 4; ++j)
        if (h[b * 4 + j] != 1000.0 * b + j) st = CC_ERR_NCCL;
  } catch (const Error &e) {
    st = e.status;
  }
  if (s) cudaStreamSynchronize(s);
  if (dc_ok) api.DevCommDestroy(comm, &dc);
  if (win) api.CommWindowDeregister(comm, win);
  if (buf) api.MemFree(buf);
  if (out) cudaFree(out);
  if (s) cudaStreamDestroy(s);
  if (comm) api.CommDestroy(comm);
  return st;
}

}  // namespace cc
