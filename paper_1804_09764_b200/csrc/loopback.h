// loopback.h -- an in-process transport standing in for NCCL so that the
// 1D-partition path (pack kernel, halo placement, local / remote gather
// passes, cross-rank reduction) can run with several ranks -- one host
// thread and one cc_ctx each -- on a single GPU.  Test infrastructure for
// the multi-rank device path when fewer GPUs than ranks are available.
//
// No kernel ever waits for another rank: the ranks meet on the HOST
// (rendezvous with a timeout), halo rows move with cudaMemcpyAsync ordered by
// events recorded on the sender's stream, and the sender's stream waits for
// the receivers' copy events before its send buffer is released.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

namespace cc {

struct LoopbackGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int64_t generation = 0;
  int arrived = 0;
  // per-rank slots published at the current rendezvous
  std::vector<const void *> ptr;
  std::vector<const int64_t *> offs;
  std::vector<cudaEvent_t> ev, ev2;
  std::vector<std::vector<double>> vec;
  explicit LoopbackGroup(int w) : world(w), ptr(w), offs(w), ev(w), ev2(w), vec(w) {}
  // Every rank calls with its slot filled; returns when all ranks arrived
  // (CC_ERR_NCCL after 300 s: a rank failed or diverged).
  void rendezvous();
};

}  // namespace cc
