// Staged transfers of pageable host buffers and the pageable host-cloud cache (hostio.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

namespace gsct_dev {

// true when p is ordinary (pageable) host memory, not page-locked / device memory
bool host_pageable(const void* p);
// fn(k) for k in [0, n_tasks) on the process-wide host worker pool (the caller helps)
void host_parallel_for(int64_t n_tasks, const std::function<void(int64_t)>& fn);

struct CloudArrays {
  const void* p[4];  // pos, log_scale, quat, raw_density
};

class HostIO {
 public:
  ~HostIO();
  // Enqueue on st. Pageable buffers >= kMinStaged go through the pinned arena (H2D: parallel
  // host copy now; D2H: parallel copy-out at finish()); anything else is a plain
  // cudaMemcpyAsync.
  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
  cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t st);
  // Deferred D2H copy-outs (each piece as soon as its DMA has landed, so the copy-out of one
  // piece overlaps the DMA of the next), then the arena reset. Called before the call's
  // stream synchronisation; returns the first error an awaited DMA reported.
  cudaError_t finish();
  // Drop deferred copies (error path; the arena is reset).
  void discard();
  bool has_pending() const { return !pending_.empty(); }
  // Pageable host cloud -> device replica `dev`: only chunks that differ from the pinned
  // shadow of the previous call (same host/device pointers and n) are uploaded.
  cudaError_t cloud_to_device(const CloudArrays& host, const CloudArrays& dev, int64_t n, int device,
                              cudaStream_t st, int64_t* bytes_uploaded);
  void invalidate_cloud();

  static constexpr size_t kMinStaged = size_t(256) << 10;
  // GSCT_HOSTIO_STATS=1: host-side milliseconds per activity, printed when the context dies
  double ms_replica = 0, ms_h2d = 0, ms_copyout = 0, ms_sync = 0, ms_api = 0, ms_replica_dirty = 0;
  int64_t n_replica = 0, bytes_replica_up = 0, n_api = 0, n_replica_dirty = 0;
  // host-side split of the forward call (GSCT_HOSTIO_STATS): cloud upload, set-up enqueue +
  // pair-count wait, binning + raster enqueue, final sync + copy-out
  double ms_fwd[4] = {0, 0, 0, 0};

 private:
  void* stage(size_t bytes);
  struct Block {
    void* p = nullptr;
    size_t cap = 0, used = 0;
  };
  struct Pending {
    void* dst;
    const void* staged;
    size_t bytes;
    cudaEvent_t landed;  // recorded behind the piece's DMA
  };
  cudaEvent_t next_event();
  std::vector<cudaEvent_t> events_;
  size_t n_events_used_ = 0;
  int device_ = 0;
  std::vector<Block> blocks_;
  size_t cur_ = 0;
  std::vector<Pending> pending_;
  double* shadow_ = nullptr;
  size_t shadow_cap_ = 0;
  bool key_valid_ = false;
  CloudArrays key_host_{}, key_dev_{};
  int64_t key_n_ = 0;
};

}  // namespace gsct_dev
