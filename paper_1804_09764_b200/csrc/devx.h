// devx.h -- the device-initiated halo exchange (devx.cu): launchers.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>

struct ncclDevComm;

namespace cc {
namespace dev {

// CTAs of the put kernel = LSA barrier slots (the same on every rank).
constexpr int kPutCtas = 16;

// Columns [c0, c0 + w) of the send rows of src (stride ld) stored into the
// peers' windows: row i of peer q's rows lands at window row dst_row[q] +
// (i - send_off[q]) (stride ldH, byte offset win_off); LSA barriers before
// and after (collective over the ranks).
int launch_pack_put(int elem, const ncclDevComm &comm, ncclWindow_t win, size_t win_off, const void *src, int64_t ld,
                    int64_t c0, int64_t w, const int32_t *send_idx, const int64_t *send_off, const int64_t *dst_row,
                    int world, int me, int64_t ldH, cudaStream_t s);
// One-rank check of the window + LSA pointer + barrier machinery: out[b * 4 + j] = 1000 b + j.
int launch_put_selftest(const ncclDevComm &comm, ncclWindow_t win, double *out, cudaStream_t s);

}  // namespace dev
}  // namespace cc
