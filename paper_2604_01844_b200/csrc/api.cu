// C-ABI implementation (include/gsct_cuda.h): device context, grow-only workspace,
// host<->device staging, per-call orchestration of the set-up / sort / pair / tail kernels,
// error mapping to the reference's contract_error messages, and RenderStats.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "../../include/gsct_cuda.h"
#include "group.h"
#include "hostio.h"
#include "gsct_internal.cuh"

using namespace gsct_dev;

namespace gsct_dev {
thread_local int64_t* g_launch_counter = nullptr;
}

namespace {

enum Slot {
  S_POS, S_LS, S_Q, S_RAW, S_FRAMES, S_REC, S_COUNT, S_OFFSET, S_KEYS, S_VALS, S_KEYS2, S_VALS2,
  S_CUB, S_START, S_END, S_IMAGES, S_GRADIMG, S_MOMENTS, S_GPOS, S_GLS, S_GQ, S_GRAW, S_GPGN,
  S_GVIS, S_VREC, S_VOLUME, S_GRADVOL, S_DBG0, S_DBG1, S_DBG2, S_DBG3, S_DBG4, S_PRE, S_PRE_AOS, S_ACC, S_SAVED, S_LOSS_IN, S_LOSS_TGT, S_LOSS_GRAD, S_LOSS_COEF, S_LOSS_PART, S_ADAM_SKIP, S_VLOSS_SCR, S_CTRL, S_CTRL_RNG, S_FGSC, S_FGSC_LOG, S_FGSC_CNT, S_VTCOUNT,
  S_TOTAL64, S_VIEWPAIRS, S_WCOUNT, S_WSLOT, S_WSUMS, S_WSTART, S_MOMENTS64, S_BSUMS, S_FSCHED, S_GFLAG, S_GPOSN, S_GSUMS, S_GROWS, S_GIDX, S_GCNT,
  S_COUNT_SLOTS
};

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

struct CallError {
  int code;
  std::string msg;
};

}  // namespace

struct gsct_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  // host<->device image traffic of the C-ABI host-buffer path runs here, chunk by chunk,
  // overlapped with the compute stream (event-ordered both ways)
  cudaStream_t copy_stream = nullptr;
  // second compute stream: the host-image forward alternates its view sub-ranges between
  // this and `stream`, so consecutive sub-range kernels fill each other's tails
  cudaStream_t aux_stream = nullptr;
  bool own_stream = false;
  bool async = false;
  std::string err;
  int64_t launches = 0;
  Buf bufs[S_COUNT_SLOTS];
  DevStats* dstats = nullptr;   // device
  DevStats* hstats = nullptr;   // pinned host mirror
  uint32_t* hscratch = nullptr; // pinned 128 B: scan totals / small result words
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  gsct_stats pending{};          // async-mode stats accumulated at synchronize
  // per-phase event timing (gsct_ctx_set_profiling)
  bool profiling = false;
  std::vector<cudaEvent_t> event_pool;
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks;
  double phase_ms[GSCT_NUM_PHASES] = {};
  int64_t phase_count[GSCT_NUM_PHASES] = {};
  // save-for-backward: forward set-up records kept for the matching backward call
  bool save_fb = false;
  bool saved_valid = false;
  std::string saved_key;
  bool fgsc_table_ready = false;  // S_FGSC_LOG holds the binary16 log table
  // the saved forward's walk-order buckets (S_WCOUNT / S_WSLOT, all views of the call)
  bool walk_valid = false;
  gsct_dev::WalkLayout walk_L;
  // multi-GPU group (gsct_ctx_set_group): collectives of the backward / voxel calls
  gsct_group group = nullptr;
  // staged transfers of pageable host buffers + the pageable host-cloud replica (hostio.cu)
  gsct_dev::HostIO hio;
};

namespace gsct_dev {
double run_microbench(int kind, cudaStream_t st);
}

namespace {

void throw_cuda(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw CallError{GSCT_ERR_OOM, std::string(what) + ": out of device memory"};
  }
  throw CallError{GSCT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(call)                              \
  do {                                        \
    cudaError_t e_ = (call);                  \
    if (e_ != cudaSuccess) throw_cuda(e_, #call); \
  } while (0)

void contract(bool ok, const std::string& msg) {
  if (!ok) throw CallError{GSCT_ERR_CONTRACT, msg};
}

// Host <-> device copies of caller buffers: pageable memory is staged (hostio.cu) in
// synchronous mode; async calls (whose completion the caller owns) use plain copies.
void h2d(gsct_ctx c, void* dst, const void* src, size_t bytes, cudaStream_t st);
void d2h(gsct_ctx c, void* dst, const void* src, size_t bytes, cudaStream_t st);

// group.cu calls: empty string = success
void GK(const std::string& err) {
  if (!err.empty()) throw CallError{GSCT_ERR_CUDA, err};
}

void h2d(gsct_ctx c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (c->async)
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  else
    CK(c->hio.h2d(dst, src, bytes, st));
}

void d2h(gsct_ctx c, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (c->async)
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
  else
    CK(c->hio.d2h(dst, src, bytes, st));
}

template <class T>
T* ws(gsct_ctx c, Slot s, size_t count) {
  Buf& b = c->bufs[s];
  const size_t bytes = count * sizeof(T) + 16;
  if (b.cap < bytes) {
    if (b.p) CK(cudaFreeAsync(b.p, c->stream));
    b.p = nullptr;
    b.cap = 0;
    size_t want = bytes + bytes / 4;
    CK(cudaMallocAsync(&b.p, want, c->stream));
    b.cap = want;
  }
  return static_cast<T*>(b.p);
}

cudaEvent_t pooled_event(gsct_ctx c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// `waiter` waits for the work enqueued so far on `signaller` (pooled event, recycled once
// the wait is enqueued: re-recording a pooled event later does not affect that wait).
void stream_after(gsct_ctx c, cudaStream_t waiter, cudaStream_t signaller) {
  cudaEvent_t e = pooled_event(c);
  CK(cudaEventRecord(e, signaller));
  CK(cudaStreamWaitEvent(waiter, e, 0));
  c->event_pool.push_back(e);
}

// Records CUDA events around one phase's launches when profiling is on.
struct Phase {
  gsct_ctx c;
  int phase;
  cudaEvent_t a = nullptr;
  Phase(gsct_ctx ctx, int ph) : c(ctx), phase(ph) {
    if (c->profiling) {
      a = pooled_event(c);
      CK(cudaEventRecord(a, c->stream));
    }
  }
  ~Phase() {
    if (!a) return;
    cudaEvent_t b = pooled_event(c);
    cudaEventRecord(b, c->stream);
    c->marks.push_back({phase, a, b});
  }
};

void resolve_marks(gsct_ctx c) {
  if (c->marks.empty()) return;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& m : c->marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
      c->phase_ms[m.phase] += ms;
      c->phase_count[m.phase] += 1;
    }
    c->event_pool.push_back(m.a);
    c->event_pool.push_back(m.b);
  }
  c->marks.clear();
}

struct Guard {  // sets the launch counter for the duration of an API call
  explicit Guard(gsct_ctx c) {
    g_launch_counter = &c->launches;
    cudaSetDevice(c->device);
  }
  ~Guard() { g_launch_counter = nullptr; }
};

// error path: in-flight DMAs may still target the staging arena (and the cloud replica
// is suspect), so wait for them before the arena is reused
void drop_staged(gsct_ctx c) {
  cudaStreamSynchronize(c->copy_stream);
  cudaStreamSynchronize(c->aux_stream);
  cudaStreamSynchronize(c->stream);
  cudaGetLastError();
  c->hio.discard();
  c->hio.invalidate_cloud();
}

template <class F>
int run(gsct_ctx c, F&& f) {
  if (!c) return GSCT_ERR_CONTRACT;
  Guard guard(c);
  const auto t0 = std::chrono::steady_clock::now();
  try {
    f();
    c->hio.ms_api += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ++c->hio.n_api;
    c->err.clear();
    return GSCT_OK;
  } catch (const CallError& e) {
    c->err = e.msg;
    drop_staged(c);
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    drop_staged(c);
    return GSCT_ERR_CUDA;
  }
}

void validate_geometry(const gsct_geometry* g, const double* angles, int n_views) {
  contract(g != nullptr, "ScanGeometry: null geometry");
  contract(g->n_u >= 1 && g->n_v >= 1, "ScanGeometry: detector must be at least 1x1");
  contract(g->s_u > 0.0 && g->s_v > 0.0, "ScanGeometry: pixel spacing must be positive");
  contract(n_views >= 0, "ScanGeometry: negative view count");
  for (int i = 0; i < n_views; ++i) contract(std::isfinite(angles[i]), "ScanGeometry: non-finite angle");
  if (g->cone)
    contract(g->source_to_origin > 0.0 && g->origin_to_detector > 0.0,
             "ScanGeometry: cone distances must be positive");
  contract(g->n_u <= 65535 && g->n_v <= 65535, "ScanGeometry: detector side above 65535 unsupported");
}

Frame make_frame(const gsct_geometry* g, double angle) {
  double f[16];
  gsct_host_view_frame(g, angle, f);
  Frame fr;
  for (int k = 0; k < 3; ++k) {
    fr.u[k] = f[k];
    fr.v[k] = f[3 + k];
    fr.d[k] = f[6 + k];
    fr.dc[k] = f[9 + k];
    fr.src[k] = f[12 + k];
  }
  fr.focal = f[15];
  return fr;
}

Geo make_geo(const gsct_geometry* g) { return Geo{g->cone, g->n_u, g->n_v, g->s_u, g->s_v}; }

RSet make_rs(const gsct_raster_settings* r) {
  return RSet{r->tau_cut, r->sigma_cap, r->dilation_px2, r->tile_size, r->dilate, r->bounding};
}

// Device view of a cloud; host arrays get device copies (allocated here; the copy is
// enqueued on `st` unless `copy` is false -- then copy_cloud() does it later). A pageable
// host cloud in synchronous mode is kept as a device replica refreshed chunk-wise
// (hostio.cu), whatever `copy` says.
Cloud upload_cloud(gsct_ctx c, const gsct_cloud* cl, cudaStream_t st = nullptr, bool copy = true);

// GSCT_HOST_ZEROED outputs have host semantics; *zeroed tells a sparse-capable call that the
// caller's buffers are already zero-filled
gsct_grads host_norm(const gsct_grads* g, bool* zeroed) {
  gsct_grads o = *g;
  *zeroed = o.location == GSCT_HOST_ZEROED;
  if (*zeroed) o.location = GSCT_HOST;
  return o;
}

bool replica_applies(gsct_ctx c, const gsct_cloud* cl) {
  return !c->async && cl->location == GSCT_HOST && cl->n > 0 && host_pageable(cl->pos) &&
         host_pageable(cl->log_scale) && host_pageable(cl->quat) && host_pageable(cl->raw_density);
}

void copy_cloud(gsct_ctx c, const gsct_cloud* cl, const Cloud& d, cudaStream_t st) {
  const size_t n = static_cast<size_t>(cl->n);
  c->hio.invalidate_cloud();  // the device buffers no longer hold the pageable replica
  if (st != c->stream) stream_after(c, st, c->stream);  // after the (re)allocation and prior readers
  CK(cudaMemcpyAsync(const_cast<double*>(d.pos), cl->pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(const_cast<double*>(d.ls), cl->log_scale, 3 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(const_cast<double*>(d.q), cl->quat, 4 * n * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(const_cast<double*>(d.raw), cl->raw_density, n * sizeof(double), cudaMemcpyHostToDevice, st));
}

Cloud upload_cloud(gsct_ctx c, const gsct_cloud* cl, cudaStream_t st, bool copy) {
  if (!st) st = c->stream;
  contract(cl != nullptr && cl->n >= 0, "GaussianCloud: invalid cloud");
  contract(cl->n < (int64_t(1) << 31), "GaussianCloud: more than 2^31 splats unsupported");
  Cloud d{cl->n, cl->pos, cl->log_scale, cl->quat, cl->raw_density};
  if (cl->n == 0) return d;
  contract(cl->pos && cl->log_scale && cl->quat && cl->raw_density,
           "GaussianCloud: parameter arrays out of lockstep");
  if (cl->location == GSCT_HOST) {
    const size_t n = static_cast<size_t>(cl->n);
    d.pos = ws<double>(c, S_POS, 3 * n);
    d.ls = ws<double>(c, S_LS, 3 * n);
    d.q = ws<double>(c, S_Q, 4 * n);
    d.raw = ws<double>(c, S_RAW, n);
    if (replica_applies(c, cl)) {
      // pageable host cloud (the C++ drop-in): chunks changed since the last call only
      const CloudArrays h{{cl->pos, cl->log_scale, cl->quat, cl->raw_density}};
      const CloudArrays dv{{d.pos, d.ls, d.q, d.raw}};
      if (st != c->stream) stream_after(c, st, c->stream);
      CK(c->hio.cloud_to_device(h, dv, cl->n, c->device, st, nullptr));
    } else if (copy) {
      copy_cloud(c, cl, d, st);
    }
  }
  return d;
}

// Device address of a page-locked, device-mapped host buffer (cudaHostAlloc'd / registered
// memory under UVA, e.g. torch pinned tensors), else nullptr. Host outputs in such memory are
// written by the kernels directly over PCIe ("zero-copy"): the transfer overlaps the kernel
// instead of following it as a D2H copy.
#ifndef GSCT_ZEROCOPY
#define GSCT_ZEROCOPY 1
#endif
template <class T>
T* mapped_host(gsct_ctx c, T* host) {
  if (!GSCT_ZEROCOPY || host == nullptr) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  // only memory pinned under this context's device (portable allocations made elsewhere
  // take the staged path: their mapping into this device cannot be told from here)
  return a.type == cudaMemoryTypeHost && a.devicePointer && a.device == c->device ? static_cast<T*>(a.devicePointer)
                                                                                   : nullptr;
}

void reset_stats(gsct_ctx c) {
  if (c->async) return;  // async: accumulate until gsct_ctx_synchronize
  DevStats z{0, 0, 0, 0, ~0ull};
  CK(cudaMemcpyAsync(c->dstats, &z, sizeof z, cudaMemcpyHostToDevice, c->stream));
}

// Reads device stats, maps device-side contract errors, accumulates RenderStats.
void finish_sync(gsct_ctx c, gsct_stats* stats, bool counters, double* ms_slot) {
  if (c->async) return;
  CK(cudaMemcpyAsync(c->hstats, c->dstats, sizeof(DevStats), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->ev1, c->stream));
  // deferred copy-outs of staged D2H into pageable caller buffers, each piece as it lands
  const cudaError_t landed = c->hio.finish();
  {
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(c->stream));
    c->hio.ms_sync += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  CK(landed);
  CK(cudaGetLastError());
  const DevStats& h = *c->hstats;
  if (h.error_key != ~0ull) {
    const unsigned long long idx = h.error_key >> 2;
    const int code = static_cast<int>(h.error_key & 3);
    throw CallError{GSCT_ERR_CONTRACT, std::string(code == 1 ? "activate: non-finite parameter in splat "
                                                             : "activate: zero quaternion in splat ") +
                                           std::to_string(idx)};
  }
  if (stats) {
    if (counters) {
      stats->culled += static_cast<int64_t>(h.culled);
      stats->degenerate += static_cast<int64_t>(h.degenerate);
      stats->tile_pairs += static_cast<int64_t>(h.tile_pairs);
      stats->pixel_pairs += static_cast<int64_t>(h.pixel_pairs);
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (ms_slot == &stats->forward_ms) stats->forward_ms += ms;
    if (ms_slot == &stats->backward_ms) stats->backward_ms += ms;
  }
}

// Exact 64-bit sum of per-item pair counts (the u32 scan could wrap); pairs beyond what one
// radix sort takes are a contract error rather than a wrapped workspace.
int64_t count_total(gsct_ctx c, const uint32_t* counts, int64_t n) {
  unsigned long long* d = ws<unsigned long long>(c, S_TOTAL64, 1);
  CK(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
  launch_sum_u32(counts, n, d, c->stream);
  CK(cudaMemcpyAsync(c->hscratch, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  unsigned long long t = 0;
  std::memcpy(&t, c->hscratch, sizeof t);
  contract(t <= static_cast<unsigned long long>(INT32_MAX), "bin: more than 2^31 pairs (" + std::to_string(t) + ")");
  return static_cast<int64_t>(t);
}

int bits_for(uint64_t n_keys) {
  int b = 1;
  while ((uint64_t(1) << b) < n_keys) ++b;
  return b;
}

// Exclusive scan of counts + pair emission + stable radix sort by key + key ranges.
// Returns the number of pairs; sorted values end up in *vals_out, start/end per key.
// sort_bits > 0: the emitted pairs are already ordered by the key bits above sort_bits
// (view-major emission, key = view << sort_bits | tile), so a stable sort on the low
// sort_bits alone leaves every (view, tile) run contiguous -- ordered (tile, view, splat)
// rather than (view, tile, splat), with the splats of a run still ascending -- in one
// radix pass instead of two or three; ranges by binary search in (tile, view) order.
template <class Emit>
int64_t bin_and_sort(gsct_ctx c, const uint32_t* counts, int64_t n_items, uint32_t n_keys,
                     Emit&& emit, uint32_t** keys_out, uint32_t** vals_out, uint32_t** start,
                     uint32_t** end, int sort_bits = 0, int64_t known_total = -1) {
  uint32_t* offsets = ws<uint32_t>(c, S_OFFSET, static_cast<size_t>(n_items));
  size_t tmp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, offsets, static_cast<int>(n_items), c->stream));
  void* tmp = ws<uint8_t>(c, S_CUB, tmp_bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offsets, static_cast<int>(n_items), c->stream));
  const int64_t total = known_total >= 0 ? known_total : count_total(c, counts, n_items);
  *start = ws<uint32_t>(c, S_START, n_keys);
  *end = ws<uint32_t>(c, S_END, n_keys);
  if (total == 0) {
    CK(cudaMemsetAsync(*start, 0, n_keys * sizeof(uint32_t), c->stream));
    CK(cudaMemsetAsync(*end, 0, n_keys * sizeof(uint32_t), c->stream));
    *keys_out = *vals_out = nullptr;
    return 0;
  }
  uint32_t* k1 = ws<uint32_t>(c, S_KEYS, total);
  uint32_t* v1 = ws<uint32_t>(c, S_VALS, total);
  uint32_t* k2 = ws<uint32_t>(c, S_KEYS2, total);
  uint32_t* v2 = ws<uint32_t>(c, S_VALS2, total);
  emit(offsets, k1, v1);
  cub::DoubleBuffer<uint32_t> kb(k1, k2), vb(v1, v2);
  const int end_bit = sort_bits > 0 ? sort_bits : bits_for(n_keys);
  tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<int>(total), 0, end_bit, c->stream));
  tmp = ws<uint8_t>(c, S_CUB, tmp_bytes);
  CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<int>(total), 0, end_bit, c->stream));
  *keys_out = kb.Current();
  *vals_out = vb.Current();
  if (sort_bits > 0) {
    launch_ranges_swapped(*keys_out, total, n_keys, sort_bits, *start, *end, c->stream);
  } else {
    launch_ranges(*keys_out, total, n_keys, *start, *end, c->stream);
  }
  return total;
}

// Forward binning plan (one place decides, for chunk sizing and for the binning itself):
//  narrow packed: <= 256 super-tiles (one 8-bit pass), 256 <= n < 2^24: key = tile << 24 | splat
//  wide packed:   <= 4096 super-tiles, n >= kWideMinItems, n < 2^(32 - tile_bits):
//                 key = tile << (32 - tile_bits) | splat
//  otherwise:     key + value pairs (view * stride + tile, splat)
#ifndef GSCT_BIN_PACKED
#define GSCT_BIN_PACKED 1  // keys-only packed binning when it applies (see bin_packed)
#endif
#ifndef GSCT_BIN_PACKED_WIDE
#define GSCT_BIN_PACKED_WIDE 1  // packed keys also beyond 8 tile bits (2048^2: tile << 20 | splat)
#endif
#ifndef GSCT_BIN_ONEPASS
#define GSCT_BIN_ONEPASS 1
#endif
struct BinPlan {
  int tile_bits = 0;
  bool onepass = false;  // key stride a power of two; the sort covers the tile bits only
  int stride = 0;        // (view, tile) key stride
  bool packed = false, wide = false;
  int shift = 24;        // packed: tile bits start here
  uint32_t vmask = 0xFFFFFFFFu;  // packed: splat index = key & vmask
};
BinPlan fwd_bin_plan(int64_t n, int n_tiles) {
  BinPlan p;
  p.tile_bits = bits_for(static_cast<uint32_t>(n_tiles));
  // key = view * stride + super-tile; stride a power of two for the one-pass sort, used when
  // the tile bits fit one 8-bit radix pass (A/B: C2 bin 0.94 -> 0.74 ms; at C5, 12 tile bits,
  // the two-pass tile-only sort was 1.1 ms slower than the full key)
  p.onepass = GSCT_BIN_ONEPASS && p.tile_bits <= 8;
  p.stride = p.onepass ? (1 << p.tile_bits) : n_tiles;
  const bool narrow = GSCT_BIN_PACKED && p.onepass && n >= 256 && n < (int64_t(1) << 24) && n_tiles <= 256;
  const bool wide = GSCT_BIN_PACKED && GSCT_BIN_PACKED_WIDE && !narrow && p.tile_bits >= 1 && p.tile_bits <= 12 &&
                    n >= kWideMinItems && n < (int64_t(1) << (32 - p.tile_bits)) && n_tiles <= 4096;
  p.packed = narrow || wide;
  p.wide = wide;
  p.shift = wide ? 32 - p.tile_bits : 24;
  p.vmask = !p.packed ? 0xFFFFFFFFu : (wide ? (0xFFFFFFFFu >> p.tile_bits) : 0x00FFFFFFu);
  return p;
}

// pairs per binning pass: int-sized for the radix sort, and a bounded key workspace
constexpr int64_t kMaxBinPairs = int64_t(1) << 30;

// Packed keys-only forward binning (see k_emit_tile_keys): scan of the per-item counts,
// emission of the packed keys with (view, tile) counts, ONE stable radix pass over the tile
// bits (two for the wide layout; 4 bytes per pair moved), ranges from the counts. `total` is
// the exact pair count (the set-up's per-view sums, <= kMaxBinPairs).
void bin_packed(gsct_ctx c, const BinPlan& pl, const RasterRec* rec, const uint32_t* counts, int64_t n, int n_views,
                int tiles_u, int n_tiles, int64_t total, uint32_t** keys_out, uint32_t** start, uint32_t** end) {
  const int64_t n_items = n * n_views;
  const uint32_t n_keys = static_cast<uint32_t>(n_views) * static_cast<uint32_t>(pl.stride);
  *start = ws<uint32_t>(c, S_START, n_keys);
  *end = ws<uint32_t>(c, S_END, n_keys);
  if (total == 0) {
    CK(cudaMemsetAsync(*start, 0, n_keys * sizeof(uint32_t), c->stream));
    CK(cudaMemsetAsync(*end, 0, n_keys * sizeof(uint32_t), c->stream));
    *keys_out = nullptr;
    return;
  }
  uint32_t* offsets = ws<uint32_t>(c, S_OFFSET, static_cast<size_t>(n_items));
  uint32_t* k1 = ws<uint32_t>(c, S_KEYS, static_cast<size_t>(total));
  uint32_t* k2 = ws<uint32_t>(c, S_KEYS2, static_cast<size_t>(total));
  uint32_t* vt = ws<uint32_t>(c, S_VTCOUNT, static_cast<size_t>(n_views) * n_tiles);
  CK(cudaMemsetAsync(vt, 0, static_cast<size_t>(n_views) * n_tiles * sizeof(uint32_t), c->stream));
  // item offsets: the hand-written u32 scan (order.cu)
  launch_exclusive_scan_u32(counts, offsets, n_items,
                            ws<uint32_t>(c, S_BSUMS, static_cast<size_t>(scan_workspace_u32(n_items))), c->stream);
#ifndef GSCT_EMIT_WIDE_ALL
#define GSCT_EMIT_WIDE_ALL 1  // 4096-item emitting CTAs for the narrow layout too (A/B C2 emit 0.234 -> 0.176 ms)
#endif
  if (pl.wide || (GSCT_EMIT_WIDE_ALL && n >= kWideItems))
    launch_emit_tile_keys_wide(rec, offsets, counts, n, n_views, kBinTile, tiles_u, n_tiles, pl.shift, k1, vt,
                               c->stream);
  else
    launch_emit_tile_keys(rec, offsets, counts, n, n_views, kBinTile, tiles_u, n_tiles, k1, vt, c->stream);
  cub::DoubleBuffer<uint32_t> kb(k1, k2);
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, kb, static_cast<int>(total), pl.shift,
                                    pl.shift + pl.tile_bits, c->stream));
  void* tmp = ws<uint8_t>(c, S_CUB, tmp_bytes);
  CK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, kb, static_cast<int>(total), pl.shift, pl.shift + pl.tile_bits,
                                    c->stream));
  *keys_out = kb.Current();
  if (pl.wide)
    launch_ranges_from_counts_wide(vt, n_views, n_tiles, pl.stride, *start, *end, c->stream);
  else
    launch_ranges_from_counts(vt, n_views, n_tiles, pl.stride, *start, *end, c->stream);
}

// The forward's binning of views [0, n_views) of one chunk's records (view-major, `counts`
// their super-tile counts, `total` the exact pair count): sorted splat lists per (view,
// super-tile) in [start, end) of `vals` (splat = vals[k] & plan.vmask). Shared by
// gsct_rasterize_fwd and the parity export gsct_debug_fwd_bins.
struct FwdBins {
  const uint32_t* vals = nullptr;
  const uint32_t* start = nullptr;
  const uint32_t* end = nullptr;
};
FwdBins fwd_bin(gsct_ctx c, const BinPlan& pl, const RasterRec* rec, const uint32_t* cnt, int64_t n, int n_views,
                int tiles_u, int n_tiles, int64_t total) {
  uint32_t *keys = nullptr, *vals = nullptr, *start = nullptr, *end = nullptr;
  if (pl.packed) {
    bin_packed(c, pl, rec, cnt, n, n_views, tiles_u, n_tiles, total, &vals, &start, &end);
  } else {
    const uint32_t n_keys = static_cast<uint32_t>(n_views) * static_cast<uint32_t>(pl.stride);
    bin_and_sort(
        c, cnt, n * n_views, n_keys,
        [&](const uint32_t* offsets, uint32_t* k, uint32_t* v) {
          launch_emit_tile_pairs(rec, offsets, cnt, n, n_views, kBinTile, tiles_u, pl.stride, k, v, c->stream);
        },
        &keys, &vals, &start, &end, pl.onepass ? pl.tile_bits : 0, total);
  }
  return FwdBins{vals, start, end};
}

// Splits a chunk's views into consecutive binning ranges of at most kMaxBinPairs pairs each
// (per-view pair counts from the set-up); a single view above the bound is a contract error.
std::vector<int> bin_ranges(const unsigned long long* view_pairs, int n_views) {
  std::vector<int> cut{0};
  unsigned long long acc = 0;
  for (int v = 0; v < n_views; ++v) {
    const unsigned long long p = view_pairs[v];
    contract(p <= static_cast<unsigned long long>(kMaxBinPairs),
             "rasterize: more than 2^30 (super-tile, splat) pairs in one view (" + std::to_string(p) + ")");
    if (acc + p > static_cast<unsigned long long>(kMaxBinPairs)) {
      cut.push_back(v);
      acc = 0;
    }
    acc += p;
  }
  cut.push_back(n_views);
  return cut;
}

// Walk order of the lane-per-item backward over views [0, n_views) of `rec`: the chain kernel
// (32 B-aligned rows) uses the hand-written spatial counting sort (order.cu: buckets from the
// records here; the forward's set-up produces them directly when it saves its records); the
// other row widths keep the shape keys + radix sort of the lane kernel.
#ifndef GSCT_BWD_COUNTSORT
#define GSCT_BWD_COUNTSORT 1
#endif
const uint32_t* walk_order(gsct_ctx c, const RasterRec* rec, int64_t n, int n_views, int n_u, int n_v, int vec,
                           uint32_t* k1, uint32_t* v1, uint32_t* k2, uint32_t* v2) {
  const int64_t items = n * n_views;
  if (GSCT_BWD_COUNTSORT && bwd_chain_applies(vec)) {
    c->walk_valid = false;  // S_WCOUNT / S_WSLOT reused below
    const WalkLayout L = walk_layout(n_views, n_u, n_v);
    const int64_t nb = walk_buckets(L, n_views);
    uint32_t* counts = ws<uint32_t>(c, S_WCOUNT, static_cast<size_t>(nb));
    uint32_t* starts = ws<uint32_t>(c, S_WSTART, static_cast<size_t>(nb));
    uint2* slots = ws<uint2>(c, S_WSLOT, static_cast<size_t>(items));
    uint32_t* sums = ws<uint32_t>(c, S_WSUMS, static_cast<size_t>(scan_workspace_u32(nb)));
    CK(cudaMemsetAsync(counts, 0, static_cast<size_t>(nb) * sizeof(uint32_t), c->stream));
    launch_walk_count(rec, n, n_views, L, counts, slots, c->stream);
    launch_walk_scatter(counts, starts, nb, slots, items, sums, v1, c->stream);
    return v1;
  }
  const int kbits = launch_bwd_shape_keys(rec, n, n_views, n_u, n_v, vec, k1, v1, c->stream);
  cub::DoubleBuffer<uint32_t> kb(k1, k2), vb(v1, v2);
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<int>(items), 0, kbits, c->stream));
  void* tmp = ws<uint8_t>(c, S_CUB, tmp_bytes);
  CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<int>(items), 0, kbits, c->stream));
  return vb.Current();
}

// Identity of a rasterizer call for save-for-backward: cloud buffers and size, geometry,
// angles and settings, field by field (no struct padding).
std::string raster_call_key(const gsct_cloud* cl, const gsct_geometry* g, const double* angles, int n_views,
                            const gsct_raster_settings* rs) {
  std::string k;
  auto put = [&k](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  put(&cl->n, sizeof cl->n);
  put(&cl->pos, sizeof cl->pos);
  put(&cl->log_scale, sizeof cl->log_scale);
  put(&cl->quat, sizeof cl->quat);
  put(&cl->raw_density, sizeof cl->raw_density);
  put(&cl->location, sizeof cl->location);
  put(&g->cone, sizeof g->cone);
  put(&g->n_u, sizeof g->n_u);
  put(&g->n_v, sizeof g->n_v);
  put(&g->s_u, sizeof g->s_u);
  put(&g->s_v, sizeof g->s_v);
  put(&g->source_to_origin, sizeof g->source_to_origin);
  put(&g->origin_to_detector, sizeof g->origin_to_detector);
  put(&n_views, sizeof n_views);
  if (n_views > 0) put(angles, sizeof(double) * static_cast<size_t>(n_views));
  put(&rs->tau_cut, sizeof rs->tau_cut);
  put(&rs->sigma_cap, sizeof rs->sigma_cap);
  put(&rs->dilation_px2, sizeof rs->dilation_px2);
  put(&rs->tile_size, sizeof rs->tile_size);
  put(&rs->dilate, sizeof rs->dilate);
  put(&rs->bounding, sizeof rs->bounding);
  return k;
}

// Views per chunk: bounded (view, splat) items, and view*n_tiles + tile keys of at most
// 16 bits so the stable radix sort needs two 8-bit passes.
int views_per_chunk(int64_t n, int n_views, int64_t n_tiles) {
  const int64_t budget = int64_t(1) << 25;  // (view, splat) items per chunk
  int64_t v = n > 0 ? budget / n : n_views;
  if (n_tiles > 0 && n_tiles <= 65536) v = std::min<int64_t>(v, 65536 / n_tiles);
  if (v < 1) v = 1;
  if (v > n_views) v = n_views;
  // balance the chunks (e.g. 75 views -> 38 + 37, not 64 + 11) so no launch has a short tail
  if (v > 0 && n_views > 0) {
    const int64_t n_chunks = (n_views + v - 1) / v;
    v = (n_views + n_chunks - 1) / n_chunks;
  }
  return static_cast<int>(v);
}

}  // namespace

extern "C" {

int gsct_abi_version(void) { return GSCT_ABI_VERSION; }

int gsct_ctx_create(int device, gsct_ctx* out) {
  if (!out) return GSCT_ERR_CONTRACT;
  *out = nullptr;
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || device < 0 || device >= n_dev) {
    cudaGetLastError();
    return GSCT_ERR_CUDA;
  }
  auto* c = new gsct_ctx_s();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->dstats, sizeof(DevStats)) != cudaSuccess ||
      cudaMallocHost(&c->hstats, sizeof(DevStats)) != cudaSuccess ||
      cudaMallocHost(&c->hscratch, 16 * sizeof(uint64_t)) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return GSCT_ERR_CUDA;
  }
  c->own_stream = true;
  DevStats z{0, 0, 0, 0, ~0ull};
  cudaMemcpy(c->dstats, &z, sizeof z, cudaMemcpyHostToDevice);
  *out = c;
  return GSCT_OK;
}

void gsct_ctx_destroy(gsct_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (Buf& b : c->bufs)
    if (b.p) cudaFreeAsync(b.p, c->stream);
  cudaStreamSynchronize(c->stream);
  cudaFree(c->dstats);
  cudaFreeHost(c->hstats);
  cudaFreeHost(c->hscratch);
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  for (auto& m : c->marks) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  }
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* gsct_ctx_last_error(gsct_ctx c) { return c ? c->err.c_str() : "null context"; }

int gsct_ctx_set_stream(gsct_ctx c, void* stream) {
  return run(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    if (c->own_stream) CK(cudaStreamDestroy(c->stream));
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
  });
}

void* gsct_ctx_stream(gsct_ctx c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int gsct_ctx_set_async(gsct_ctx c, int async) {
  return run(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    c->async = async != 0;
    DevStats z{0, 0, 0, 0, ~0ull};
    CK(cudaMemcpyAsync(c->dstats, &z, sizeof z, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int gsct_ctx_synchronize(gsct_ctx c, gsct_stats* stats_accum) {
  return run(c, [&] {
    CK(cudaMemcpyAsync(c->hstats, c->dstats, sizeof(DevStats), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGetLastError());
    const DevStats h = *c->hstats;
    DevStats z{0, 0, 0, 0, ~0ull};
    CK(cudaMemcpyAsync(c->dstats, &z, sizeof z, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (stats_accum) {
      stats_accum->culled += static_cast<int64_t>(h.culled);
      stats_accum->degenerate += static_cast<int64_t>(h.degenerate);
      stats_accum->tile_pairs += static_cast<int64_t>(h.tile_pairs);
      stats_accum->pixel_pairs += static_cast<int64_t>(h.pixel_pairs);
    }
    if (h.error_key != ~0ull) {
      const unsigned long long idx = h.error_key >> 2;
      const int code = static_cast<int>(h.error_key & 3);
      throw CallError{GSCT_ERR_CONTRACT, std::string(code == 1 ? "activate: non-finite parameter in splat "
                                                               : "activate: zero quaternion in splat ") +
                                             std::to_string(idx)};
    }
  });
}

size_t gsct_ctx_workspace_bytes(gsct_ctx c) {
  if (!c) return 0;
  size_t s = 0;
  for (const Buf& b : c->bufs) s += b.cap;
  return s;
}

int64_t gsct_ctx_launch_count(gsct_ctx c) { return c ? c->launches : 0; }

int gsct_ctx_set_save_for_backward(gsct_ctx c, int save) {
  return run(c, [&] {
    c->save_fb = save != 0;
    c->saved_valid = false;
  });
}

int gsct_ctx_set_profiling(gsct_ctx c, int on) {
  return run(c, [&] {
    resolve_marks(c);
    c->profiling = on != 0;
  });
}

int gsct_ctx_phase_times(gsct_ctx c, double ms[GSCT_NUM_PHASES], int64_t counts[GSCT_NUM_PHASES]) {
  return run(c, [&] {
    resolve_marks(c);
    for (int k = 0; k < GSCT_NUM_PHASES; ++k) {
      if (ms) ms[k] = c->phase_ms[k];
      if (counts) counts[k] = c->phase_count[k];
      c->phase_ms[k] = 0.0;
      c->phase_count[k] = 0;
    }
  });
}

int gsct_microbench(gsct_ctx c, int kind, double* ops_per_second) {
  return run(c, [&] {
    contract(ops_per_second != nullptr && (kind == 0 || kind == 1), "microbench: bad arguments");
    CK(cudaStreamSynchronize(c->stream));
    *ops_per_second = run_microbench(kind, c->stream);
    CK(cudaGetLastError());
  });
}

// ---------------------------------------------------------------------------------------
// Multi-GPU group (group.cu)
// ---------------------------------------------------------------------------------------

int gsct_group_new_id(gsct_ctx c, gsct_group_id* out) {
  return run(c, [&] {
    contract(out != nullptr, "gsct_group_new_id: null output");
    GK(group_new_id(out->bytes));
  });
}

int gsct_group_create(gsct_ctx c, const gsct_group_id* id, int n_ranks, int rank, gsct_group* out) {
  return run(c, [&] {
    contract(id != nullptr && out != nullptr, "gsct_group_create: null argument");
    contract(n_ranks >= 1 && rank >= 0 && rank < n_ranks, "gsct_group_create: rank outside [0, n_ranks)");
    *out = nullptr;
    CK(cudaStreamSynchronize(c->stream));
    GK(group_create(c->device, id->bytes, n_ranks, rank, out));
  });
}

int gsct_ctx_set_group(gsct_ctx c, gsct_group g) {
  return run(c, [&] {
    contract(g == nullptr || group_device(g) == c->device, "gsct_ctx_set_group: group made on another device");
    c->group = g;
  });
}

int gsct_group_info(gsct_group g, int* rank, int* n_ranks) {
  if (!g) return GSCT_ERR_CONTRACT;
  if (rank) *rank = group_rank(g);
  if (n_ranks) *n_ranks = group_size(g);
  return GSCT_OK;
}

void gsct_group_destroy(gsct_group g) { group_destroy(g); }

// ---------------------------------------------------------------------------------------
// Rasterizer
// ---------------------------------------------------------------------------------------

int gsct_rasterize_fwd(gsct_ctx c, const gsct_cloud* cloud, const gsct_geometry* geom,
                       const double* angles, int n_views, const gsct_raster_settings* rs,
                       float* images, int images_location, gsct_stats* stats) {
  return run(c, [&] {
    validate_geometry(geom, angles, n_views);
    contract(rs != nullptr, "RasterSettings: null");
    contract(rs->tile_size >= 1, "bin_tiles: tile size must be at least 1");
    contract(images != nullptr || n_views == 0, "rasterize: null image buffer");
    if (!c->async) CK(cudaEventRecord(c->ev0, c->stream));
    reset_stats(c);
#ifndef GSCT_CLOUD_PIECES
#define GSCT_CLOUD_PIECES 2  // host cloud uploaded in splat ranges, each range's set-up starting
                             // as soon as its bytes are in (single view chunk only; A/B C2 e2e:
                             // 1 / 2 / 3 / 4 / 8 pieces -> 7.63 / 7.55 / 7.63 / 7.74 / 7.82 ms)
#endif
    const int64_t n_in = cloud ? cloud->n : 0;
    const int cloud_pieces = cloud && cloud->location == GSCT_HOST && !replica_applies(c, cloud) && n_in >= 16384 &&
                                     n_views > 0 &&
                                     views_per_chunk(n_in, n_views, 0) >= n_views
                                 ? GSCT_CLOUD_PIECES
                                 : 1;
    auto fwd_t = std::chrono::steady_clock::now();
    auto fwd_mark = [&](int k) {
      const auto t = std::chrono::steady_clock::now();
      c->hio.ms_fwd[k] += std::chrono::duration<double, std::milli>(t - fwd_t).count();
      fwd_t = t;
    };
    const Cloud d = upload_cloud(c, cloud, c->stream, cloud_pieces == 1);
    fwd_mark(0);
    std::vector<cudaEvent_t> piece_up;
    if (cloud_pieces > 1) {
      c->hio.invalidate_cloud();
      stream_after(c, c->copy_stream, c->stream);  // after the (re)allocation and prior readers
      for (int k = 0; k < cloud_pieces; ++k) {
        const size_t a = static_cast<size_t>(n_in * k / cloud_pieces), b = static_cast<size_t>(n_in * (k + 1) / cloud_pieces);
        const size_t m = b - a;
        CK(cudaMemcpyAsync(const_cast<double*>(d.pos) + 3 * a, cloud->pos + 3 * a, 3 * m * sizeof(double),
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(const_cast<double*>(d.ls) + 3 * a, cloud->log_scale + 3 * a, 3 * m * sizeof(double),
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(const_cast<double*>(d.q) + 4 * a, cloud->quat + 4 * a, 4 * m * sizeof(double),
                           cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaMemcpyAsync(const_cast<double*>(d.raw) + a, cloud->raw_density + a, m * sizeof(double),
                           cudaMemcpyHostToDevice, c->copy_stream));
        piece_up.push_back(pooled_event(c));
        CK(cudaEventRecord(piece_up.back(), c->copy_stream));
      }
    }
    const int64_t n = d.n;
    const int64_t npx = static_cast<int64_t>(geom->n_u) * geom->n_v;
    // binned at 32x32 super-tiles (kBinTile); RenderStats::tile_pairs stays at rs->tile_size
    const int tiles_u = (geom->n_u + kBinTile - 1) / kBinTile, tiles_v = (geom->n_v + kBinTile - 1) / kBinTile;
    const int n_tiles = tiles_u * tiles_v;
    std::vector<Frame> frames(static_cast<size_t>(n_views));
    for (int v = 0; v < n_views; ++v) frames[static_cast<size_t>(v)] = make_frame(geom, angles[v]);
    Frame* dframes = ws<Frame>(c, S_FRAMES, frames.size() + 1);
    if (n_views)
      CK(cudaMemcpyAsync(dframes, frames.data(), frames.size() * sizeof(Frame), cudaMemcpyHostToDevice, c->stream));
    float* out = images;
    float* zc_images = images_location == GSCT_HOST && n > 0 ? mapped_host(c, images) : nullptr;
    if (zc_images)
      out = zc_images;  // the forward kernel stores straight into the pinned host images
    else if (images_location == GSCT_HOST && n_views)
      out = ws<float>(c, S_IMAGES, static_cast<size_t>(npx) * n_views);
    const bool stage_images = images_location == GSCT_HOST && !zc_images;
    const Geo g = make_geo(geom);
    const RSet r = make_rs(rs);
    c->saved_valid = false;
    PreSplat* pre = ws<PreSplat>(c, S_PRE, static_cast<size_t>(n) + 1);
    PreSplat* pre_aos = ws<PreSplat>(c, S_PRE_AOS, static_cast<size_t>(n) + 1);
    if (n > 0 && cloud_pieces == 1) {
      Phase ph(c, GSCT_PH_RASTER_SETUP);
      launch_splat_prepare(d, pre, pre_aos, c->dstats, c->stream);
    }
    // save-for-backward keeps every view's records in one buffer for the backward call
    RasterRec* saved = c->save_fb && n > 0 ? ws<RasterRec>(c, S_SAVED, static_cast<size_t>(n) * n_views) : nullptr;
#ifndef GSCT_FWD_TILECAP
#define GSCT_FWD_TILECAP 1  // 1: <= 65536 (view, tile) keys per forward chunk (16-bit sorts)
#endif
    // the packed keys-only binning has no per-chunk key limit; the key + value fallback keeps
    // (view, tile) keys within 16 bits (A/B at C5 with packed keys: uncapped 25-view chunks
    // bin + forward 42.2 ms vs 43.2 capped)
    const BinPlan plan = fwd_bin_plan(n, n_tiles);
    int chunk = views_per_chunk(n, n_views, GSCT_FWD_TILECAP && !plan.packed ? n_tiles : 0);
    // saved records: the set-up also files every item into the backward's walk-order buckets
    c->walk_valid = false;
    WalkOut walk;
    const bool walk_out = GSCT_BWD_COUNTSORT && saved != nullptr && geom->n_u % 8 == 0;
    if (walk_out) {
      walk.L = walk_layout(n_views, geom->n_u, geom->n_v);
      const int64_t nb = walk_buckets(walk.L, n_views);
      walk.count = ws<uint32_t>(c, S_WCOUNT, static_cast<size_t>(nb));
      walk.slot = ws<uint2>(c, S_WSLOT, static_cast<size_t>(n) * n_views);
      CK(cudaMemsetAsync(walk.count, 0, static_cast<size_t>(nb) * sizeof(uint32_t), c->stream));
    }
    unsigned long long* dpairs = ws<unsigned long long>(c, S_VIEWPAIRS, static_cast<size_t>(chunk) + 1);
    std::vector<unsigned long long> hpairs(static_cast<size_t>(chunk));
    for (int v0 = 0; v0 < n_views; v0 += chunk) {
      const int cv = std::min(chunk, n_views - v0);
      float* img = out + static_cast<int64_t>(v0) * npx;
      if (n == 0) {
        CK(cudaMemsetAsync(img, 0, static_cast<size_t>(npx) * cv * sizeof(float), c->stream));
        if (images_location == GSCT_HOST) {
          stream_after(c, c->copy_stream, c->stream);
          d2h(c, images + static_cast<int64_t>(v0) * npx, img, static_cast<size_t>(npx) * cv * sizeof(float),
              c->copy_stream);
        }
        continue;
      }
      RasterRec* rec = saved ? saved + static_cast<int64_t>(v0) * n : ws<RasterRec>(c, S_REC, static_cast<size_t>(n) * cv);
      uint32_t* cnt = ws<uint32_t>(c, S_COUNT, static_cast<size_t>(n) * cv);
      CK(cudaMemsetAsync(dpairs, 0, static_cast<size_t>(cv) * sizeof(unsigned long long), c->stream));
      {
        Phase ph(c, GSCT_PH_RASTER_SETUP);
        if (cloud_pieces > 1) {  // one view chunk: per splat range, wait for its bytes, set up
          for (int k = 0; k < cloud_pieces; ++k) {
            const int64_t i0 = n * k / cloud_pieces, i1 = n * (k + 1) / cloud_pieces;
            CK(cudaStreamWaitEvent(c->stream, piece_up[static_cast<size_t>(k)], 0));
            launch_splat_prepare(d, pre, pre_aos, c->dstats, c->stream, i0, i1);
            WalkOut wk = walk;
            if (walk_out) wk.slot = walk.slot + static_cast<int64_t>(v0) * n, wk.view_base = v0;
            launch_raster_preprocess(pre, n, dframes + v0, cv, g, r, kBinTile, rec, cnt, c->dstats, c->stream, i0,
                                     i1, dpairs, walk_out ? &wk : nullptr);
          }
          for (cudaEvent_t e : piece_up) c->event_pool.push_back(e);
          piece_up.clear();
        } else {
          WalkOut wk = walk;
          if (walk_out) wk.slot = walk.slot + static_cast<int64_t>(v0) * n, wk.view_base = v0;
          launch_raster_preprocess(pre, n, dframes + v0, cv, g, r, kBinTile, rec, cnt, c->dstats, c->stream, 0, -1,
                                   dpairs, walk_out ? &wk : nullptr);
        }
      }
      CK(cudaGetLastError());
      // exact 64-bit (super-tile, splat) pair count per view: binning ranges of <= 2^30 pairs
      CK(cudaMemcpyAsync(hpairs.data(), dpairs, static_cast<size_t>(cv) * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      fwd_mark(1);
      const std::vector<int> cut = bin_ranges(hpairs.data(), cv);
      for (size_t bi = 0; bi + 1 < cut.size(); ++bi) {
        const int b0 = cut[bi], bv = cut[bi + 1] - cut[bi];  // views [v0 + b0, v0 + b0 + bv)
        int64_t total = 0;
        for (int v = b0; v < b0 + bv; ++v) total += static_cast<int64_t>(hpairs[static_cast<size_t>(v)]);
        const RasterRec* brec = rec + static_cast<int64_t>(b0) * n;
        float* bimg = img + static_cast<int64_t>(b0) * npx;
        FwdBins bins;
        {
          Phase ph(c, GSCT_PH_RASTER_BIN);
          bins = fwd_bin(c, plan, brec, cnt + static_cast<int64_t>(b0) * n, n, bv, tiles_u, n_tiles, total);
        }
        const int stride = plan.stride;
        // host output: launch in view sub-ranges so each one's images go down while the next
        // computes (the kernel indexes keys/records/images by its own view range)
#ifndef GSCT_FWD_SPLIT
#define GSCT_FWD_SPLIT 4  // staged host images: view sub-ranges (single stream A/B: 1 -> +1.74 ms, 2 -> +1.50,
                          // 4 -> +2.28; alternating two streams: 2/4/6/8 -> fwd 4.82/4.65/4.79/5.15 ms
                          // at C2, zero-copy 4.61)
#endif
#ifndef GSCT_FWD_MINPIECE
#define GSCT_FWD_MINPIECE 0  // > 0: halving sub-ranges (38, 19, 9, ...) down to this many views
#endif
#ifndef GSCT_FWD_BULKSTORE
#define GSCT_FWD_BULKSTORE 1  // zero-copy images leave the forward kernel as TMA bulk row stores
#endif
#ifndef GSCT_FWD_BULK_DEVICE
#define GSCT_FWD_BULK_DEVICE 0  // 1: device-memory images through the TMA bulk stores as well
                                // (A/B: C2 fwd 2.51 vs 2.48 ms, C5 37.1 vs 36.8 -- plain stores)
#endif
#ifndef GSCT_FWD_DUAL
#define GSCT_FWD_DUAL 1  // staged host images: sub-range kernels alternate between two streams
#endif
        const bool dual = stage_images && GSCT_FWD_DUAL && GSCT_FWD_SPLIT > 1;
        if (dual) stream_after(c, c->aux_stream, c->stream);  // after the binning
        const int sub = stage_images ? std::max(1, (bv + GSCT_FWD_SPLIT - 1) / GSCT_FWD_SPLIT) : bv;
        for (int vs = 0, nvs = 0, k = 0; vs < bv; vs += nvs, ++k) {
          const int rem = bv - vs;
          if (stage_images && GSCT_FWD_MINPIECE > 0)
            nvs = rem <= 2 * GSCT_FWD_MINPIECE ? rem : (rem + 1) / 2;
          else
            nvs = std::min(sub, rem);
          cudaStream_t fs = dual && (k & 1) ? c->aux_stream : c->stream;
          {
            Phase ph(c, GSCT_PH_RASTER_FWD);
            // warp schedule scratch: a disjoint slice per view sub-range (they may run concurrently)
            uint32_t* fsched = ws<uint32_t>(c, S_FSCHED, static_cast<size_t>(bv) * (2 * n_tiles + 2048)) +
                               static_cast<int64_t>(vs) * (2 * n_tiles + 2048);
            launch_raster_fwd_super(brec + static_cast<int64_t>(vs) * n, bins.vals,
                                    bins.start + static_cast<int64_t>(vs) * stride,
                                    bins.end + static_cast<int64_t>(vs) * stride, n, nvs, geom->n_u, geom->n_v,
                                    tiles_u, tiles_v, stride, bimg + static_cast<int64_t>(vs) * npx, fs,
                                    (zc_images || GSCT_FWD_BULK_DEVICE) && GSCT_FWD_BULKSTORE ? 1 : 0, plan.vmask,
                                    fsched);
          }
          CK(cudaGetLastError());
          if (stage_images) {
            stream_after(c, c->copy_stream, fs);
            d2h(c, images + static_cast<int64_t>(v0 + b0 + vs) * npx, bimg + static_cast<int64_t>(vs) * npx,
                static_cast<size_t>(npx) * nvs * sizeof(float), c->copy_stream);
          }
        }
        if (dual) stream_after(c, c->stream, c->aux_stream);
      }
    }
    if (stage_images && n_views) stream_after(c, c->stream, c->copy_stream);
    fwd_mark(2);
    finish_sync(c, stats, true, stats ? &stats->forward_ms : nullptr);
    fwd_mark(3);
    if (saved) {
      c->saved_key = raster_call_key(cloud, geom, angles, n_views, rs);
      c->saved_valid = true;
      c->walk_valid = walk_out;
      c->walk_L = walk.L;
    }
  });
}

int gsct_rasterize_bwd(gsct_ctx c, const gsct_cloud* cloud, const gsct_geometry* geom,
                       const double* angles, int n_views, const gsct_raster_settings* rs,
                       const float* grad_images, int grad_location, gsct_grads* out,
                       gsct_stats* stats) {
  return run(c, [&] {
    validate_geometry(geom, angles, n_views);
    contract(rs != nullptr, "RasterSettings: null");
    contract(rs->tile_size >= 1, "bin_tiles: tile size must be at least 1");
    contract(out != nullptr, "rasterize_backward: null gradient output");
    contract(grad_images != nullptr || n_views == 0, "rasterize_backward: grad image dims must match detector");
    bool zeroed = false;  // dense output: written in full either way
    gsct_grads out_n = host_norm(out, &zeroed);
    out = &out_n;
    if (!c->async) CK(cudaEventRecord(c->ev0, c->stream));
    reset_stats(c);
    // reuse the forward's set-up (PreSplat + records) when save-for-backward matched; then
    // the cloud itself is only needed by the final covariance_backward, so a host cloud
    // goes up on the copy stream, overlapped with the pixel walk
    const bool reuse = c->save_fb && c->saved_valid && cloud != nullptr && cloud->n > 0 &&
                       c->saved_key == raster_call_key(cloud, geom, angles, n_views, rs);
    const bool late_cloud = reuse && cloud->location == GSCT_HOST && !replica_applies(c, cloud);
    const Cloud d = upload_cloud(c, cloud, c->stream, !late_cloud);
    cudaEvent_t cloud_up = nullptr;
    const int64_t n = d.n;
    const size_t un = static_cast<size_t>(n);
    const int64_t npx = static_cast<int64_t>(geom->n_u) * geom->n_v;
    double *gp = out->pos, *gl = out->log_scale, *gq = out->quat, *gr = out->raw_density, *gn = out->pos_grad_norm;
    uint8_t* gv = out->visible;
    // host gradients in mapped pinned memory: the tail / finalize kernels store into them
    // directly (no trailing D2H); otherwise staged in the workspace and copied down
#ifndef GSCT_ZEROCOPY_GRADS
#define GSCT_ZEROCOPY_GRADS 0  // 1: the finalize leaves host-mapped gradients as TMA bulk stores
                               // (A/B C2 e2e 9.46 ms vs 9.28 for the staged 4-piece D2H, which
                               // overlaps the tail; plain strided stores over PCIe: +1.9 ms)
#endif
    bool zc_grads = false;
    if (GSCT_ZEROCOPY_GRADS && out->location == GSCT_HOST && n > 0 && n_views > 0) {
      double *mp = mapped_host(c, out->pos), *ml = mapped_host(c, out->log_scale), *mq = mapped_host(c, out->quat),
             *mr = mapped_host(c, out->raw_density), *mn = mapped_host(c, out->pos_grad_norm);
      const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
      if (mp && ml && mq && mr && mn && a16(mp) && a16(ml) && a16(mq) && a16(mr) && a16(mn)) {
        gp = mp, gl = ml, gq = mq, gr = mr, gn = mn;
        zc_grads = true;
      }
    }
    if (out->location == GSCT_HOST) {
      if (!zc_grads) {
        gp = ws<double>(c, S_GPOS, 3 * un);
        gl = ws<double>(c, S_GLS, 3 * un);
        gq = ws<double>(c, S_GQ, 4 * un);
        gr = ws<double>(c, S_GRAW, un);
        gn = ws<double>(c, S_GPGN, un);
      }
      gv = ws<uint8_t>(c, S_GVIS, un);  // visibility bytes always staged (N bytes)
    }
    if (n > 0 && n_views == 0 && !c->group) {
      CK(cudaMemsetAsync(gp, 0, 3 * un * sizeof(double), c->stream));
      CK(cudaMemsetAsync(gl, 0, 3 * un * sizeof(double), c->stream));
      CK(cudaMemsetAsync(gq, 0, 4 * un * sizeof(double), c->stream));
      CK(cudaMemsetAsync(gr, 0, un * sizeof(double), c->stream));
      CK(cudaMemsetAsync(gn, 0, un * sizeof(double), c->stream));
      CK(cudaMemsetAsync(gv, 0, un, c->stream));
    }
    std::vector<Frame> frames(static_cast<size_t>(n_views));
    for (int v = 0; v < n_views; ++v) frames[static_cast<size_t>(v)] = make_frame(geom, angles[v]);
    Frame* dframes = ws<Frame>(c, S_FRAMES, frames.size() + 1);
    if (n_views)
      CK(cudaMemcpyAsync(dframes, frames.data(), frames.size() * sizeof(Frame), cudaMemcpyHostToDevice, c->stream));
    const Geo g = make_geo(geom);
    const RSet r = make_rs(rs);
    PreSplat* pre = ws<PreSplat>(c, S_PRE, un + 1);
    PreSplat* pre_aos = ws<PreSplat>(c, S_PRE_AOS, un + 1);
    double* acc = ws<double>(c, S_ACC, 11 * un + 1);
    if (n > 0 && !reuse) {
      Phase ph(c, GSCT_PH_RASTER_SETUP);
      launch_splat_prepare(d, pre, pre_aos, c->dstats, c->stream);
    }
    RasterRec* saved = reuse ? ws<RasterRec>(c, S_SAVED, un * n_views) : nullptr;
    const int tiles_u = (geom->n_u + kTile - 1) / kTile, tiles_v = (geom->n_v + kTile - 1) / kTile;
#ifndef GSCT_BWD_ONECHUNK
#define GSCT_BWD_ONECHUNK 1  // the lane backward has no tile keys: chunk by the item budget only
#endif
#ifndef GSCT_BWD_L2_MB
#define GSCT_BWD_L2_MB 96  // grad-image MB per walked view chunk (A/B C5: 48 / 64 / 96 / 128 / 192 MB
                           // within 0.1%)
#endif
    int chunk = views_per_chunk(n, n_views, GSCT_BWD_ONECHUNK ? 0 : static_cast<int64_t>(tiles_u) * tiles_v);
    {
      // keep one chunk's grad images L2-resident (126 MB L2): C2's 75 x 1 MB in one chunk,
      // C5's 16 MB images 6 at a time (A/B at C5: 8-view chunk 77.7 ms vs 4-view 74.2)
      const int64_t l2_views = std::max<int64_t>(1, (int64_t(GSCT_BWD_L2_MB) << 20) / (static_cast<int64_t>(npx) * 4));
      if (chunk > l2_views) {
        const int64_t nc = (n_views + l2_views - 1) / l2_views;
        chunk = static_cast<int>((n_views + nc - 1) / nc);
      }
    }
    // chunk boundaries. Host grad images: growing chunks (~n/20, then x1.4 of the views so
    // far) so only a small first upload is exposed before the pixel walk starts and every
    // later chunk's upload (2.5x faster than its walk at C2) is in before its turn
#ifndef GSCT_BWD_GROW
#define GSCT_BWD_GROW 1
#endif
#ifndef GSCT_BWD_FIRST_DIV
#define GSCT_BWD_FIRST_DIV 20  // first host grad-image chunk ~ n_views / this (A/B 10 / 20 / 40: within 0.3%)
#endif
#ifndef GSCT_BWD_GROW_X10
#define GSCT_BWD_GROW_X10 12  // next chunk = 1.2 x the views so far (A/B C2 e2e with the other two
                              // pipelining knobs: 1.1 / 1.2 / 1.4 / 1.7 -> 7.58 / 7.55 / 7.74 / 7.89 ms)
#endif
    std::vector<int> cb{0};
#ifndef GSCT_BWD_HOST_CHUNKS
#define GSCT_BWD_HOST_CHUNKS 1  // 0: host grad images in one chunk (upload fully exposed; A/B C2
                                // e2e 10.0 ms vs growing chunks 9.61, six equal chunks 9.65)
#endif
    if (grad_location == GSCT_HOST && !GSCT_BWD_HOST_CHUNKS) {
      cb.push_back(n_views);
    } else if (grad_location == GSCT_HOST && n_views >= 12 && GSCT_BWD_GROW) {
      const int s0 = std::max(1, (n_views + GSCT_BWD_FIRST_DIV - 1) / GSCT_BWD_FIRST_DIV);
      while (cb.back() < n_views) {
        const int done = cb.back(), rem = n_views - done;
        int sz = std::max(s0, (done * GSCT_BWD_GROW_X10 + 9) / 10);
        sz = std::min(sz, chunk);
        if (rem - sz < sz / 2) sz = std::min(rem, chunk);
        cb.push_back(done + std::min(sz, rem));
      }
    } else {
      if (grad_location == GSCT_HOST && n_views >= 12) chunk = std::min(chunk, (n_views + 5) / 6);
      for (int v0 = chunk; v0 < n_views; v0 += chunk) cb.push_back(v0);
      cb.push_back(n_views);
    }
    int max_chunk = 0;
    for (size_t k = 1; k < cb.size(); ++k) max_chunk = std::max(max_chunk, cb[k] - cb[k - 1]);
    // pixel-loop moments of every view, view-major [n_views][N] x 8 fp32
    float* mom = ws<float>(c, S_MOMENTS, un * static_cast<size_t>(n_views) * 8 + 1);
    // host grad images: every chunk is queued up front on the copy stream (after the work
    // already on the compute stream, which may still read the buffer), one event per chunk;
    // chunk k's pixel walk waits only for its own upload
    float* gdev = nullptr;
    std::vector<cudaEvent_t> up_done;
    if (grad_location == GSCT_HOST && n > 0 && n_views > 0) {
      gdev = ws<float>(c, S_GRADIMG, static_cast<size_t>(npx) * n_views);
      stream_after(c, c->copy_stream, c->stream);
      for (size_t k = 0; k + 1 < cb.size(); ++k) {
        const int v0 = cb[k], cv = cb[k + 1] - cb[k];
        h2d(c, gdev + static_cast<int64_t>(v0) * npx, grad_images + static_cast<int64_t>(v0) * npx,
            static_cast<size_t>(npx) * cv * sizeof(float), c->copy_stream);
        up_done.push_back(pooled_event(c));
        CK(cudaEventRecord(up_done.back(), c->copy_stream));
      }
    }
    if (late_cloud) {  // queued behind the grad images: needed only by the finalize
      copy_cloud(c, cloud, d, c->copy_stream);
      cloud_up = pooled_event(c);
      CK(cudaEventRecord(cloud_up, c->copy_stream));
    }
    // with the forward's records of every view at hand (save-for-backward) and several chunks,
    // the walk order of all views is sorted once up front (view-major keys: each chunk is a
    // contiguous range) instead of once per chunk
    const float* gbase_ = gdev ? gdev : grad_images;
    const bool saved_walk = reuse && n > 0 && c->walk_valid && bwd_chain_applies(bwd_vec(geom->n_u, gbase_));
    const bool one_sort = saved_walk || (reuse && n > 0 && cb.size() > 2 && bwd_view_major(geom->n_u, geom->n_v));
#ifndef GSCT_BWD_DUAL
#define GSCT_BWD_DUAL 1  // chunk walks alternate between two streams
#endif
    const uint32_t* all_order = nullptr;
    if (one_sort) {
      Phase ph(c, GSCT_PH_RASTER_ORDER);
      const int64_t items = n * n_views;
      uint32_t* k1 = ws<uint32_t>(c, S_KEYS, static_cast<size_t>(items));
      uint32_t* v1 = ws<uint32_t>(c, S_VALS, static_cast<size_t>(items));
      uint32_t* k2 = ws<uint32_t>(c, S_KEYS2, static_cast<size_t>(items));
      uint32_t* v2 = ws<uint32_t>(c, S_VALS2, static_cast<size_t>(items));
      const float* gbase = gdev ? gdev : grad_images;
      if (saved_walk) {  // the forward's set-up filed every item: scan the bucket counts, scatter
        const int64_t nb = walk_buckets(c->walk_L, n_views);
        uint32_t* starts = ws<uint32_t>(c, S_WSTART, static_cast<size_t>(nb));
        uint32_t* sums = ws<uint32_t>(c, S_WSUMS, static_cast<size_t>(scan_workspace_u32(nb)));
        launch_walk_scatter(ws<uint32_t>(c, S_WCOUNT, static_cast<size_t>(nb)), starts, nb,
                            ws<uint2>(c, S_WSLOT, static_cast<size_t>(items)), items, sums, v1, c->stream);
        all_order = v1;
      } else {
        all_order =
            walk_order(c, saved, n, n_views, geom->n_u, geom->n_v, bwd_vec(geom->n_u, gbase), k1, v1, k2, v2);
      }
      if (GSCT_BWD_DUAL) stream_after(c, c->aux_stream, c->stream);  // after the sort
    }
    for (int ci = 0; ci + 1 < static_cast<int>(cb.size()) && n > 0; ++ci) {
      const int v0 = cb[static_cast<size_t>(ci)], cv = cb[static_cast<size_t>(ci) + 1] - v0;
      const float* gimg = gdev ? gdev + static_cast<int64_t>(v0) * npx : grad_images + static_cast<int64_t>(v0) * npx;
      RasterRec* rec = reuse ? saved + static_cast<int64_t>(v0) * n : ws<RasterRec>(c, S_REC, un * max_chunk);
      if (!reuse) {
        Phase ph(c, GSCT_PH_RASTER_SETUP);
        launch_raster_preprocess(pre, n, dframes + v0, cv, g, r, kTile, rec, nullptr, c->dstats, c->stream);
      }
      {
        if (one_sort) {  // walk this chunk's contiguous range of the all-view order
          Phase ph(c, GSCT_PH_RASTER_BWD);
          // chunks alternate between two streams so a chunk's walk fills the previous one's tail
          cudaStream_t ws_ = GSCT_BWD_DUAL && (ci & 1) ? c->aux_stream : c->stream;
          if (gdev) {
            CK(cudaStreamWaitEvent(ws_, up_done[static_cast<size_t>(ci)], 0));
            c->event_pool.push_back(up_done[static_cast<size_t>(ci)]);
          }
          launch_raster_bwd_lanes(saved, all_order + static_cast<int64_t>(v0) * n, n, cv, geom->n_u, geom->n_v,
                                  gdev ? gdev : grad_images, mom, 0, ws_);
          continue;
        }
        const int64_t items = n * cv;
        uint32_t* k1 = ws<uint32_t>(c, S_KEYS, static_cast<size_t>(items));
        uint32_t* v1 = ws<uint32_t>(c, S_VALS, static_cast<size_t>(items));
        uint32_t* k2 = ws<uint32_t>(c, S_KEYS2, static_cast<size_t>(items));
        uint32_t* v2 = ws<uint32_t>(c, S_VALS2, static_cast<size_t>(items));
        const uint32_t* order = nullptr;
        {
          Phase po(c, GSCT_PH_RASTER_ORDER);
          order = walk_order(c, rec, n, cv, geom->n_u, geom->n_v, bwd_vec(geom->n_u, gimg), k1, v1, k2, v2);
        }
        if (gdev) {
          CK(cudaStreamWaitEvent(c->stream, up_done[static_cast<size_t>(ci)], 0));
          c->event_pool.push_back(up_done[static_cast<size_t>(ci)]);
        }
        Phase ph(c, GSCT_PH_RASTER_BWD);
        launch_raster_bwd_lanes(rec, order, n, cv, geom->n_u, geom->n_v, gimg, mom, v0, c->stream);
      }
      CK(cudaGetLastError());
    }
    if (one_sort && GSCT_BWD_DUAL) stream_after(c, c->stream, c->aux_stream);
#ifndef GSCT_TAIL_PIECES
#define GSCT_TAIL_PIECES 8  // staged host gradients: tail + finalize in splat ranges, each range's
                            // D2H overlapping the next range's tail (A/B e2e with two streams: 2 / 4 / 6
                            // pieces 8.85 / 8.69 / 8.63 ms; current kernels 2 / 6 / 8: 7.98 / 7.74 / 7.74,
                            // with 2 cloud pieces and 1.2x chunk growth 6 / 8: 7.57 / 7.54)
#endif
    const bool stage_grads = out->location == GSCT_HOST && n > 0 && !zc_grads;
    const int pieces = (stage_grads || zc_grads) && n_views > 0 && n >= 4096 ? GSCT_TAIL_PIECES : 1;
    bool grads_down = false;
    if (n > 0 && c->group) {
      // multi-GPU: this rank's view sums, one fp64 all-reduce of the [11][N] accumulators
      // (+ max of the visibility bytes) on the stream, then the chain rule on the total
      Phase ph(c, GSCT_PH_RASTER_TAIL);
      if (cloud_up) CK(cudaStreamWaitEvent(c->stream, cloud_up, 0));
      if (n_views > 0) {
        launch_raster_tail(pre_aos, n, 0, n, dframes, n_views, g, r, mom, acc, gv, c->stream);
      } else {
        CK(cudaMemsetAsync(acc, 0, 11 * un * sizeof(double), c->stream));
        CK(cudaMemsetAsync(gv, 0, un, c->stream));
      }
      GK(group_allreduce_sum_f64(c->group, acc, 11 * un, c->stream));
      GK(group_allreduce_max_u8(c->group, gv, un, c->stream));
      launch_raster_finalize(d, 0, n, acc, gp, gl, gq, gr, gn, c->stream, zc_grads ? 1 : 0);
    } else if (n > 0 && n_views > 0) {
      Phase ph(c, GSCT_PH_RASTER_TAIL);
      if (cloud_up) CK(cudaStreamWaitEvent(c->stream, cloud_up, 0));
#ifndef GSCT_TAIL_DUAL
#define GSCT_TAIL_DUAL 1  // tail pieces alternate between two streams
#endif
      const bool tdual = GSCT_TAIL_DUAL && pieces > 1;
      if (tdual) stream_after(c, c->aux_stream, c->stream);
      for (int k = 0; k < pieces; ++k) {
        const int64_t i0 = n * k / pieces, i1 = n * (k + 1) / pieces;
        cudaStream_t ts = tdual && (k & 1) ? c->aux_stream : c->stream;
        launch_raster_tail(pre_aos, n, i0, i1, dframes, n_views, g, r, mom, acc, gv, ts);
        launch_raster_finalize(d, i0, i1, acc, gp, gl, gq, gr, gn, ts, zc_grads ? 1 : 0);
        if (pieces > 1 && stage_grads) {
          const size_t a = static_cast<size_t>(i0), m = static_cast<size_t>(i1 - i0);
          stream_after(c, c->copy_stream, ts);
          d2h(c, out->pos + 3 * a, gp + 3 * a, 3 * m * sizeof(double), c->copy_stream);
          d2h(c, out->log_scale + 3 * a, gl + 3 * a, 3 * m * sizeof(double), c->copy_stream);
          d2h(c, out->quat + 4 * a, gq + 4 * a, 4 * m * sizeof(double), c->copy_stream);
          d2h(c, out->raw_density + a, gr + a, m * sizeof(double), c->copy_stream);
          d2h(c, out->pos_grad_norm + a, gn + a, m * sizeof(double), c->copy_stream);
          d2h(c, out->visible + a, gv + a, m, c->copy_stream);
        }
      }
      if (tdual) stream_after(c, c->stream, c->aux_stream);
      if (pieces > 1 && stage_grads) {
        stream_after(c, c->stream, c->copy_stream);
        grads_down = true;
      }
    }
    if (cloud_up) {
      CK(cudaStreamWaitEvent(c->stream, cloud_up, 0));  // also when n_views == 0
      c->event_pool.push_back(cloud_up);
    }
    if (zc_grads) d2h(c, out->visible, gv, un, c->stream);
    if (stage_grads && !grads_down) {
      d2h(c, out->pos, gp, 3 * un * sizeof(double), c->stream);
      d2h(c, out->log_scale, gl, 3 * un * sizeof(double), c->stream);
      d2h(c, out->quat, gq, 4 * un * sizeof(double), c->stream);
      d2h(c, out->raw_density, gr, un * sizeof(double), c->stream);
      d2h(c, out->pos_grad_norm, gn, un * sizeof(double), c->stream);
      d2h(c, out->visible, gv, un, c->stream);
    }
    finish_sync(c, stats, false, stats ? &stats->backward_ms : nullptr);
  });
}

// ---------------------------------------------------------------------------------------
// Voxelizer
// ---------------------------------------------------------------------------------------

namespace {

VoxGrid make_grid(const gsct_grid* g) {
  contract(g != nullptr, "GridRegion: null grid");
  contract(g->dims[0] >= 1 && g->dims[1] >= 1 && g->dims[2] >= 1, "GridRegion: dims must be at least 1");
  contract(g->spacing > 0.0, "Volume: spacing must be positive");
  VoxGrid v;
  for (int k = 0; k < 3; ++k) {
    v.dims[k] = g->dims[k];
    v.origin[k] = g->origin[k];
  }
  v.spacing = g->spacing;
  return v;
}

Window make_window(const gsct_grid* g, const gsct_window* w) {
  Window win;
  for (int k = 0; k < 3; ++k) {
    win.lo[k] = w ? w->lo[k] : 0;
    win.hi[k] = w ? w->hi[k] : g->dims[k];
    contract(win.lo[k] >= 0 && win.lo[k] < win.hi[k] && win.hi[k] <= g->dims[k],
             "GridRegion: region outside parent grid");
  }
  return win;
}

int64_t window_count(const Window& w) {
  return static_cast<int64_t>(w.hi[0] - w.lo[0]) * (w.hi[1] - w.lo[1]) * (w.hi[2] - w.lo[2]);
}

// Backward pixel loop into moments[10][N] (zero-filled) for one window.
void voxel_moments(gsct_ctx c, const Cloud& d, const VoxGrid& grid, const Window& win,
                   const gsct_voxel_settings* vs, const float* grad, int grad_location, float* mom) {
  const int64_t n = d.n;
  const int64_t nvox = window_count(win);
  if (grad_location == GSCT_HOST) {
    float* dst = ws<float>(c, S_GRADVOL, static_cast<size_t>(nvox));
    h2d(c, dst, grad, static_cast<size_t>(nvox) * sizeof(float), c->stream);
    grad = dst;
  }
  CK(cudaMemsetAsync(mom, 0, static_cast<size_t>(n) * 10 * sizeof(float), c->stream));
  if (n == 0) return;
  VoxelRec* rec = ws<VoxelRec>(c, S_VREC, static_cast<size_t>(n));
  {
    Phase ph(c, GSCT_PH_VOXEL_SETUP);
    launch_voxel_preprocess(d, grid, win, vs->tau_cut, vs->sigma_cap, rec, nullptr, nullptr, nullptr,
                            nullptr, c->dstats, c->stream);
  }
  uint32_t* order = nullptr;
  {
    // walk order: 64^3 region of the box corner, then box shape (k_voxel_lane_keys)
    Phase ph(c, GSCT_PH_VOXEL_BIN);
    uint32_t* k1 = ws<uint32_t>(c, S_KEYS, static_cast<size_t>(n));
    uint32_t* v1 = ws<uint32_t>(c, S_VALS, static_cast<size_t>(n));
    uint32_t* k2 = ws<uint32_t>(c, S_KEYS2, static_cast<size_t>(n));
    uint32_t* v2 = ws<uint32_t>(c, S_VALS2, static_cast<size_t>(n));
    int end_bit = launch_voxel_lane_keys(rec, n, win, voxel_bwd_vec(win, grad), k1, v1, c->stream);
    if (end_bit > 32) end_bit = 32;
    cub::DoubleBuffer<uint32_t> kb(k1, k2), vb(v1, v2);
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, static_cast<int>(n), 0, end_bit, c->stream));
    void* tmp = ws<uint8_t>(c, S_CUB, tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, static_cast<int>(n), 0, end_bit, c->stream));
    order = vb.Current();
  }
  {
    Phase ph(c, GSCT_PH_VOXEL_BWD);
    const double vps = static_cast<double>(grid.dims[0]) * grid.dims[1] * grid.dims[2] / static_cast<double>(n);
    launch_voxel_bwd_lanes(rec, order, n, win, static_cast<float>(grid.spacing), grad, mom, c->stream, vps);
  }
  CK(cudaGetLastError());
}

struct GradPtrs {
  double *gp, *gl, *gq, *gr, *gn;
  uint8_t* gv;
};

GradPtrs grad_targets(gsct_ctx c, gsct_grads* out, size_t un) {
  if (out->location == GSCT_HOST)
    return GradPtrs{ws<double>(c, S_GPOS, 3 * un), ws<double>(c, S_GLS, 3 * un), ws<double>(c, S_GQ, 4 * un),
                    ws<double>(c, S_GRAW, un),     ws<double>(c, S_GPGN, un),    ws<uint8_t>(c, S_GVIS, un)};
  return GradPtrs{out->pos, out->log_scale, out->quat, out->raw_density, out->pos_grad_norm, out->visible};
}

// Sparse transfer of the gradients (zero-filled host outputs): rows of the splats that are
// visible or have a non-zero entry, compacted on the device in splat order, brought down
// and scattered into the caller's arrays after the call's sync (scatter_sparse_grads).
struct SparseGrads {
  std::vector<double> rows;  // 13 per row
  std::vector<uint32_t> idx;
};
void stage_sparse_grads(gsct_ctx c, const GradPtrs& p, size_t un, SparseGrads& sg) {
  if (un == 0) return;
  const int64_t n = static_cast<int64_t>(un);
  uint32_t* flag = ws<uint32_t>(c, S_GFLAG, un);
  uint32_t* pos = ws<uint32_t>(c, S_GPOSN, un);
  uint32_t* sums = ws<uint32_t>(c, S_GSUMS, static_cast<size_t>(scan_workspace_u32(n)));
  double* rows = ws<double>(c, S_GROWS, un * 13);
  uint32_t* idx = ws<uint32_t>(c, S_GIDX, un);
  uint32_t* cnt = ws<uint32_t>(c, S_GCNT, 1);
  launch_grad_row_flags(p.gp, p.gl, p.gq, p.gr, p.gn, p.gv, n, flag, c->stream);
  launch_exclusive_scan_u32(flag, pos, n, sums, c->stream);
  launch_grad_rows(p.gp, p.gl, p.gq, p.gr, p.gn, p.gv, n, flag, pos, rows, idx, cnt, c->stream);
  CK(cudaMemcpyAsync(c->hscratch, cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  uint32_t m = 0;
  std::memcpy(&m, c->hscratch, sizeof m);
  sg.rows.resize(static_cast<size_t>(m) * 13);
  sg.idx.resize(m);
  if (m == 0) return;
  d2h(c, sg.rows.data(), rows, sg.rows.size() * sizeof(double), c->stream);
  d2h(c, sg.idx.data(), idx, sg.idx.size() * sizeof(uint32_t), c->stream);
}
void scatter_sparse_grads(const SparseGrads& sg, gsct_grads* out) {
  const int64_t m = static_cast<int64_t>(sg.idx.size());
  constexpr int64_t kRows = 4096;
  host_parallel_for((m + kRows - 1) / kRows, [&](int64_t t) {
    const int64_t a = t * kRows, b = std::min(m, a + kRows);
    for (int64_t r = a; r < b; ++r) {
      const int64_t i = sg.idx[static_cast<size_t>(r)];
      const double* o = sg.rows.data() + r * 13;
      for (int k = 0; k < 3; ++k) {
        out->pos[3 * i + k] = o[k];
        out->log_scale[3 * i + k] = o[3 + k];
      }
      for (int k = 0; k < 4; ++k) out->quat[4 * i + k] = o[6 + k];
      out->raw_density[i] = o[10];
      out->pos_grad_norm[i] = o[11];
      out->visible[i] = o[12] != 0.0 ? 1 : 0;
    }
  });
}

void grads_to_host(gsct_ctx c, gsct_grads* out, const GradPtrs& p, size_t un) {
  if (out->location != GSCT_HOST || un == 0) return;
  d2h(c, out->pos, p.gp, 3 * un * sizeof(double), c->stream);
  d2h(c, out->log_scale, p.gl, 3 * un * sizeof(double), c->stream);
  d2h(c, out->quat, p.gq, 4 * un * sizeof(double), c->stream);
  d2h(c, out->raw_density, p.gr, un * sizeof(double), c->stream);
  d2h(c, out->pos_grad_norm, p.gn, un * sizeof(double), c->stream);
  d2h(c, out->visible, p.gv, un, c->stream);
}

}  // namespace

namespace {

// first slice of rank r's z-slab of nz slices over p ranks (the first nz % p slabs one
// slice thicker; sharding.zslab_windows)
int slab_lo(int nz, int r, int p) { return r * (nz / p) + std::min(r, nz % p); }

// Forward of one window into outv (device, window dims).
void voxel_fwd_window(gsct_ctx c, const Cloud& d, const VoxGrid& vg, const Window& win,
                      const gsct_voxel_settings* vs, float* outv) {
  const int64_t n = d.n;
  const int64_t nvox = window_count(win);
  const int nbx = (win.hi[0] - win.lo[0] + kBrick - 1) / kBrick;
  const int nby = (win.hi[1] - win.lo[1] + kBrick - 1) / kBrick;
  const int nbz = (win.hi[2] - win.lo[2] + kBrickZ - 1) / kBrickZ;
  const uint64_t n_bricks = static_cast<uint64_t>(nbx) * nby * nbz;
  contract(n_bricks < (uint64_t(1) << 31), "voxelize: grid too large");
  if (n == 0) {
    CK(cudaMemsetAsync(outv, 0, static_cast<size_t>(nvox) * sizeof(float), c->stream));
    return;
  }
  VoxelRec* rec = ws<VoxelRec>(c, S_VREC, static_cast<size_t>(n));
  uint32_t* cnt = ws<uint32_t>(c, S_COUNT, static_cast<size_t>(n));
  {
    Phase ph(c, GSCT_PH_VOXEL_SETUP);
    launch_voxel_preprocess(d, vg, win, vs->tau_cut, vs->sigma_cap, rec, cnt, nullptr, nullptr, nullptr,
                            c->dstats, c->stream);
  }
  uint32_t *keys, *vals, *start, *end;
  {
    Phase ph(c, GSCT_PH_VOXEL_BIN);
    bin_and_sort(
        c, cnt, n, static_cast<uint32_t>(n_bricks),
        [&](const uint32_t* offsets, uint32_t* k, uint32_t* v) {
          launch_emit_brick_pairs(rec, offsets, cnt, n, win, nbx, nby, k, v, c->stream);
        },
        &keys, &vals, &start, &end);
  }
  {
    Phase ph(c, GSCT_PH_VOXEL_FWD);
    launch_voxel_fwd(rec, vals, start, end, win, nbx, nby, nbz, static_cast<float>(vg.spacing), outv, c->stream,
                     ws<uint32_t>(c, S_FSCHED, 2 * static_cast<size_t>(n_bricks) + 2048));
  }
  CK(cudaGetLastError());
}

}  // namespace

int gsct_voxelize_fwd(gsct_ctx c, const gsct_cloud* cloud, const gsct_grid* grid,
                      const gsct_window* window, const gsct_voxel_settings* vs, float* volume,
                      int volume_location, gsct_stats* stats) {
  return run(c, [&] {
    const VoxGrid vg = make_grid(grid);
    const Window win = make_window(grid, window);
    contract(vs != nullptr, "VoxelSettings: null");
    contract(volume != nullptr, "voxelize: null volume buffer");
    if (!c->async) CK(cudaEventRecord(c->ev0, c->stream));
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const int64_t nvox = window_count(win);
    float* outv = volume;
    if (volume_location == GSCT_HOST) outv = ws<float>(c, S_VOLUME, static_cast<size_t>(nvox));
    if (c->group && window == nullptr) {
      // multi-GPU voxelize_full: this rank's z-slab, then every slab broadcast to all ranks
      const int P = group_size(c->group), rk = group_rank(c->group), nz = grid->dims[2];
      const int64_t plane = static_cast<int64_t>(grid->dims[0]) * grid->dims[1];
      std::vector<size_t> off(static_cast<size_t>(P) + 1);
      for (int k = 0; k <= P; ++k) off[static_cast<size_t>(k)] = static_cast<size_t>(plane * slab_lo(nz, k, P));
      Window sw = win;
      sw.lo[2] = slab_lo(nz, rk, P);
      sw.hi[2] = slab_lo(nz, rk + 1, P);
      if (sw.hi[2] > sw.lo[2]) voxel_fwd_window(c, d, vg, sw, vs, outv + plane * sw.lo[2]);
      GK(group_allgather_slabs_f32(c->group, outv, off.data(), c->stream));
    } else {
      voxel_fwd_window(c, d, vg, win, vs, outv);
    }
    if (volume_location == GSCT_HOST)
      d2h(c, volume, outv, static_cast<size_t>(nvox) * sizeof(float), c->stream);
    finish_sync(c, stats, true, stats ? &stats->forward_ms : nullptr);
  });
}

namespace {

// This call's window (or, with a group and no window, this rank's z-slab of the full grid)
// walked into fp32 moments; with a group the moments are widened to fp64 and all-reduced.
// Returns the moments the finish reads: float* (single GPU) or double* (group).
struct VoxMoments {
  const float* f32 = nullptr;
  const double* f64 = nullptr;
};
VoxMoments voxel_bwd_moments(gsct_ctx c, const Cloud& d, const VoxGrid& vg, const gsct_grid* grid,
                             const gsct_window* window, const gsct_voxel_settings* vs, const float* grad_volume,
                             int grad_location, bool want_f64) {
  const size_t un = static_cast<size_t>(d.n);
  float* mom = ws<float>(c, S_MOMENTS, un * 10 + 1);
  Window win = make_window(grid, window);
  const float* gvol = grad_volume;
  bool empty = false;
  if (c->group && window == nullptr) {
    const int P = group_size(c->group), rk = group_rank(c->group), nz = grid->dims[2];
    const int64_t plane = static_cast<int64_t>(grid->dims[0]) * grid->dims[1];
    win.lo[2] = slab_lo(nz, rk, P);
    win.hi[2] = slab_lo(nz, rk + 1, P);
    gvol = grad_volume + plane * win.lo[2];
    empty = win.hi[2] <= win.lo[2];
  }
  if (empty)
    CK(cudaMemsetAsync(mom, 0, un * 10 * sizeof(float), c->stream));
  else
    voxel_moments(c, d, vg, win, vs, gvol, grad_location, mom);
  VoxMoments m;
  if (!want_f64 && !c->group) {
    m.f32 = mom;
    return m;
  }
  double* m64 = ws<double>(c, S_MOMENTS64, un * 10 + 1);
  launch_widen_f32(mom, m64, static_cast<int64_t>(un) * 10, c->stream);
  if (c->group) GK(group_allreduce_sum_f64(c->group, m64, un * 10, c->stream));
  m.f64 = m64;
  return m;
}

}  // namespace

int gsct_voxelize_bwd(gsct_ctx c, const gsct_cloud* cloud, const gsct_grid* grid,
                      const gsct_window* window, const gsct_voxel_settings* vs,
                      const float* grad_volume, int grad_location, gsct_grads* out,
                      gsct_stats* stats) {
  return run(c, [&] {
    const VoxGrid vg = make_grid(grid);
    make_window(grid, window);
    contract(vs != nullptr, "VoxelSettings: null");
    contract(out != nullptr, "voxelize_backward: null gradient output");
    contract(grad_volume != nullptr, "voxelize_backward: grad dims must match region");
    bool zeroed = false;
    gsct_grads out_n = host_norm(out, &zeroed);
    out = &out_n;
    if (!c->async) CK(cudaEventRecord(c->ev0, c->stream));
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const size_t un = static_cast<size_t>(d.n);
    const VoxMoments m = voxel_bwd_moments(c, d, vg, grid, window, vs, grad_volume, grad_location, false);
    const GradPtrs p = grad_targets(c, out, un);
    {
      Phase ph(c, GSCT_PH_VOXEL_TAIL);
      if (m.f64)
        launch_voxel_tail(d, vg, vs->tau_cut, vs->sigma_cap, m.f64, p.gp, p.gl, p.gq, p.gr, p.gn, p.gv, c->dstats,
                          c->stream);
      else
        launch_voxel_tail(d, vg, vs->tau_cut, vs->sigma_cap, m.f32, p.gp, p.gl, p.gq, p.gr, p.gn, p.gv, c->dstats,
                          c->stream);
    }
    CK(cudaGetLastError());
    if (zeroed && !c->async && out->location == GSCT_HOST) {  // sparse rows into the zero-filled buffers
      SparseGrads sg;
      stage_sparse_grads(c, p, un, sg);
      finish_sync(c, stats, false, stats ? &stats->backward_ms : nullptr);
      scatter_sparse_grads(sg, out);
      return;
    }
    grads_to_host(c, out, p, un);
    finish_sync(c, stats, false, stats ? &stats->backward_ms : nullptr);
  });
}

int gsct_voxelize_bwd_moments(gsct_ctx c, const gsct_cloud* cloud, const gsct_grid* grid,
                              const gsct_window* window, const gsct_voxel_settings* vs,
                              const float* grad_volume, int grad_location, double* moments_dev) {
  return run(c, [&] {
    const VoxGrid vg = make_grid(grid);
    const Window win = make_window(grid, window);
    contract(vs != nullptr && moments_dev != nullptr && grad_volume != nullptr, "voxelize_backward: null buffer");
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const size_t un = static_cast<size_t>(d.n);
    float* mom = ws<float>(c, S_MOMENTS, un * 10 + 1);
    voxel_moments(c, d, vg, win, vs, grad_volume, grad_location, mom);
    launch_widen_f32(mom, moments_dev, static_cast<int64_t>(un) * 10, c->stream);
    finish_sync(c, nullptr, false, nullptr);
  });
}

int gsct_voxelize_bwd_finish(gsct_ctx c, const gsct_cloud* cloud, const gsct_grid* grid,
                             const gsct_voxel_settings* vs, const double* moments_dev,
                             gsct_grads* out) {
  return run(c, [&] {
    const VoxGrid vg = make_grid(grid);
    contract(vs != nullptr && moments_dev != nullptr && out != nullptr, "voxelize_backward: null buffer");
    bool zeroed = false;
    gsct_grads out_n = host_norm(out, &zeroed);
    out = &out_n;
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const size_t un = static_cast<size_t>(d.n);
    const GradPtrs p = grad_targets(c, out, un);
    {
      Phase ph(c, GSCT_PH_VOXEL_TAIL);
      launch_voxel_tail(d, vg, vs->tau_cut, vs->sigma_cap, moments_dev, p.gp, p.gl, p.gq, p.gr, p.gn, p.gv,
                        c->dstats, c->stream);
    }
    CK(cudaGetLastError());
    grads_to_host(c, out, p, un);
    finish_sync(c, nullptr, false, nullptr);
  });
}

// ---------------------------------------------------------------------------------------
// Parity hooks
// ---------------------------------------------------------------------------------------

int gsct_debug_project(gsct_ctx c, const gsct_cloud* cloud, const gsct_geometry* geom, double angle,
                       const gsct_raster_settings* rs, int32_t* rect, uint8_t* flags, double* mean2d,
                       double* conic, double* amplitude) {
  return run(c, [&] {
    validate_geometry(geom, &angle, 1);
    contract(rs != nullptr, "RasterSettings: null");
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const size_t un = static_cast<size_t>(d.n);
    if (un == 0) return;
    const Frame fr = make_frame(geom, angle);
    Frame* df = ws<Frame>(c, S_FRAMES, 1);
    CK(cudaMemcpyAsync(df, &fr, sizeof fr, cudaMemcpyHostToDevice, c->stream));
    int32_t* drect = ws<int32_t>(c, S_DBG0, 4 * un);
    uint8_t* dflags = ws<uint8_t>(c, S_DBG1, un);
    double* dmean = ws<double>(c, S_DBG2, 2 * un);
    double* dconic = ws<double>(c, S_DBG3, 4 * un);
    double* damp = ws<double>(c, S_DBG4, un);
    c->saved_valid = false;  // S_PRE is reused below
    PreSplat* pre = ws<PreSplat>(c, S_PRE, un);
    launch_splat_prepare(d, pre, ws<PreSplat>(c, S_PRE_AOS, un), c->dstats, c->stream);
    launch_debug_project(pre, d.n, df, make_geo(geom), make_rs(rs), drect, dflags, dmean, dconic, damp,
                         c->stream);
    CK(cudaMemcpyAsync(rect, drect, 4 * un * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(flags, dflags, un, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(mean2d, dmean, 2 * un * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(conic, dconic, 4 * un * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(amplitude, damp, un * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    finish_sync(c, nullptr, false, nullptr);
  });
}

int gsct_debug_fwd_bins(gsct_ctx c, const gsct_cloud* cloud, const gsct_geometry* geom, const double* angles,
                        int n_views, const gsct_raster_settings* rs, int64_t* offsets, uint32_t* splats,
                        int64_t capacity, int64_t* n_pairs) {
  return run(c, [&] {
    validate_geometry(geom, angles, n_views);
    contract(rs != nullptr && rs->tile_size >= 1, "bin_tiles: tile size must be at least 1");
    contract(n_pairs != nullptr && offsets != nullptr, "debug_fwd_bins: null output");
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const int64_t n = d.n;
    const int tiles_u = (geom->n_u + kBinTile - 1) / kBinTile, tiles_v = (geom->n_v + kBinTile - 1) / kBinTile;
    const int n_tiles = tiles_u * tiles_v;
    *n_pairs = 0;
    std::fill(offsets, offsets + static_cast<int64_t>(n_views) * n_tiles + 1, int64_t(0));
    if (n == 0 || n_views == 0) {
      finish_sync(c, nullptr, false, nullptr);
      return;
    }
    std::vector<Frame> frames(static_cast<size_t>(n_views));
    for (int v = 0; v < n_views; ++v) frames[static_cast<size_t>(v)] = make_frame(geom, angles[v]);
    Frame* dframes = ws<Frame>(c, S_FRAMES, frames.size() + 1);
    CK(cudaMemcpyAsync(dframes, frames.data(), frames.size() * sizeof(Frame), cudaMemcpyHostToDevice, c->stream));
    c->saved_valid = false;
    PreSplat* pre = ws<PreSplat>(c, S_PRE, static_cast<size_t>(n) + 1);
    launch_splat_prepare(d, pre, ws<PreSplat>(c, S_PRE_AOS, static_cast<size_t>(n) + 1), c->dstats, c->stream);
    const Geo g = make_geo(geom);
    const RSet r = make_rs(rs);
    // same plan and chunking as gsct_rasterize_fwd
    const BinPlan plan = fwd_bin_plan(n, n_tiles);
    const int chunk = views_per_chunk(n, n_views, !plan.packed ? n_tiles : 0);
    unsigned long long* dpairs = ws<unsigned long long>(c, S_VIEWPAIRS, static_cast<size_t>(chunk) + 1);
    std::vector<unsigned long long> hpairs(static_cast<size_t>(chunk));
    std::vector<std::vector<uint32_t>> lists(static_cast<size_t>(n_views) * n_tiles);
    for (int v0 = 0; v0 < n_views; v0 += chunk) {
      const int cv = std::min(chunk, n_views - v0);
      RasterRec* rec = ws<RasterRec>(c, S_REC, static_cast<size_t>(n) * cv);
      uint32_t* cnt = ws<uint32_t>(c, S_COUNT, static_cast<size_t>(n) * cv);
      CK(cudaMemsetAsync(dpairs, 0, static_cast<size_t>(cv) * sizeof(unsigned long long), c->stream));
      launch_raster_preprocess(pre, n, dframes + v0, cv, g, r, kBinTile, rec, cnt, c->dstats, c->stream, 0, -1,
                               dpairs);
      CK(cudaMemcpyAsync(hpairs.data(), dpairs, static_cast<size_t>(cv) * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      const std::vector<int> cut = bin_ranges(hpairs.data(), cv);
      for (size_t bi = 0; bi + 1 < cut.size(); ++bi) {
        const int b0 = cut[bi], bv = cut[bi + 1] - cut[bi];
        int64_t total = 0;
        for (int v = b0; v < b0 + bv; ++v) total += static_cast<int64_t>(hpairs[static_cast<size_t>(v)]);
        const FwdBins bins = fwd_bin(c, plan, rec + static_cast<int64_t>(b0) * n, cnt + static_cast<int64_t>(b0) * n,
                                     n, bv, tiles_u, n_tiles, total);
        const size_t nk = static_cast<size_t>(bv) * plan.stride;
        std::vector<uint32_t> hs(nk), he(nk), hv(static_cast<size_t>(total));
        if (total > 0) {
          CK(cudaMemcpyAsync(hs.data(), bins.start, nk * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
          CK(cudaMemcpyAsync(he.data(), bins.end, nk * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
          CK(cudaMemcpyAsync(hv.data(), bins.vals, static_cast<size_t>(total) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaStreamSynchronize(c->stream));
        for (int v = 0; v < bv && total > 0; ++v)
          for (int t = 0; t < n_tiles; ++t) {
            const size_t k = static_cast<size_t>(v) * plan.stride + t;
            auto& L = lists[static_cast<size_t>(v0 + b0 + v) * n_tiles + t];
            for (uint32_t q = hs[k]; q < he[k]; ++q) L.push_back(hv[q] & plan.vmask);
          }
      }
    }
    int64_t acc = 0;
    for (size_t k = 0; k < lists.size(); ++k) {
      offsets[k] = acc;
      acc += static_cast<int64_t>(lists[k].size());
    }
    offsets[lists.size()] = acc;
    *n_pairs = acc;
    if (splats && acc <= capacity)
      for (size_t k = 0; k < lists.size(); ++k)
        std::copy(lists[k].begin(), lists[k].end(), splats + offsets[k]);
    finish_sync(c, nullptr, false, nullptr);
  });
}

int gsct_debug_tile_pairs(gsct_ctx c, const gsct_cloud* cloud, const gsct_geometry* geom, const double* angles,
                          int n_views, const gsct_raster_settings* rs, uint32_t* keys, uint32_t* values,
                          int64_t capacity, int64_t* n_pairs) {
  return run(c, [&] {
    validate_geometry(geom, angles, n_views);
    contract(rs != nullptr && rs->tile_size >= 1, "bin_tiles: tile size must be at least 1");
    contract(n_pairs != nullptr, "debug_tile_pairs: null count");
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const int64_t n = d.n;
    *n_pairs = 0;
    if (n == 0 || n_views == 0) {
      finish_sync(c, nullptr, false, nullptr);
      return;
    }
    const int ts = rs->tile_size;
    const int tiles_u = (geom->n_u + ts - 1) / ts, tiles_v = (geom->n_v + ts - 1) / ts;
    const int n_tiles = tiles_u * tiles_v;
    std::vector<Frame> frames(static_cast<size_t>(n_views));
    for (int v = 0; v < n_views; ++v) frames[static_cast<size_t>(v)] = make_frame(geom, angles[v]);
    Frame* dframes = ws<Frame>(c, S_FRAMES, frames.size());
    CK(cudaMemcpyAsync(dframes, frames.data(), frames.size() * sizeof(Frame), cudaMemcpyHostToDevice, c->stream));
    RasterRec* rec = ws<RasterRec>(c, S_REC, static_cast<size_t>(n) * n_views);
    uint32_t* cnt = ws<uint32_t>(c, S_COUNT, static_cast<size_t>(n) * n_views);
    c->saved_valid = false;  // S_PRE / S_REC are reused below
    PreSplat* pre = ws<PreSplat>(c, S_PRE, static_cast<size_t>(n));
    launch_splat_prepare(d, pre, ws<PreSplat>(c, S_PRE_AOS, static_cast<size_t>(n)), c->dstats, c->stream);
    launch_raster_preprocess(pre, n, dframes, n_views, make_geo(geom), make_rs(rs), ts, rec, cnt, c->dstats,
                             c->stream);
    uint32_t *dk, *dv, *start, *end;
    const int64_t total = bin_and_sort(
        c, cnt, n * n_views, static_cast<uint32_t>(n_views) * static_cast<uint32_t>(n_tiles),
        [&](const uint32_t* offsets, uint32_t* k, uint32_t* v) {
          launch_emit_tile_pairs(rec, offsets, cnt, n, n_views, ts, tiles_u, n_tiles, k, v, c->stream);
        },
        &dk, &dv, &start, &end);
    *n_pairs = total;
    if (total > 0 && total <= capacity && keys && values) {
      CK(cudaMemcpyAsync(keys, dk, static_cast<size_t>(total) * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(values, dv, static_cast<size_t>(total) * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    }
    finish_sync(c, nullptr, false, nullptr);
  });
}

// ---------------------------------------------------------------------------------------
// Next-row operators: image loss, Adam
// ---------------------------------------------------------------------------------------

namespace {
void ssim_window(double w[11]) {  // losses.hpp:85-98 on the host libm
  double sum = 0.0;
  for (int i = 0; i < 11; ++i) {
    const double d = i - 5;
    w[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
    sum += w[i];
  }
  for (int i = 0; i < 11; ++i) w[i] /= sum;
}
}  // namespace

int gsct_image_loss(gsct_ctx c, const float* rendered, const float* measured, int n_views, int n_u, int n_v,
                    double alpha_ssim, float* grad_images, int location, double* losses) {
  return run(c, [&] {
    contract(n_views >= 0, "image_loss: n_views must be >= 0");
    contract(n_u >= 11 && n_v >= 11, "ssim2d: image smaller than the 11x11 window");
    contract(std::isfinite(alpha_ssim) && alpha_ssim >= 0.0, "LossWeights: alpha_ssim invalid");
    contract(n_views == 0 || (rendered && measured && grad_images && losses), "image_loss: null buffer");
    if (n_views == 0) return;
    double w[11];  // the reference's normalised sigma-1.5 window (losses.hpp:85-98), host libm
    ssim_window(w);
    const size_t npx = static_cast<size_t>(n_u) * n_v * n_views;
    const float* p = rendered;
    const float* t = measured;
    float* g = grad_images;
    if (location == GSCT_HOST) {
      float* dp = ws<float>(c, S_LOSS_IN, npx);
      float* dt = ws<float>(c, S_LOSS_TGT, npx);
      CK(cudaMemcpyAsync(dp, rendered, npx * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(dt, measured, npx * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      p = dp, t = dt;
      g = ws<float>(c, S_LOSS_GRAD, npx);
    }
    const size_t nout = static_cast<size_t>(n_u - 10) * (n_v - 10) * n_views;
    float* coef = ws<float>(c, S_LOSS_COEF, 3 * nout);
    const int64_t nparts = image_loss_partials(n_views, n_u, n_v);
    double* parts = ws<double>(c, S_LOSS_PART, static_cast<size_t>(nparts) + 3 * static_cast<size_t>(n_views));
    const int64_t n_s = nparts - static_cast<int64_t>(n_views) * ((n_u + 31) / 32) * ((n_v + 15) / 16);
    double* out3 = parts + nparts;
    launch_image_loss(p, t, n_views, n_u, n_v, w, alpha_ssim, coef, parts, parts + n_s, g, out3, c->stream);
    CK(cudaGetLastError());
    if (location == GSCT_HOST)
      CK(cudaMemcpyAsync(grad_images, g, npx * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(losses, out3, 3 * static_cast<size_t>(n_views) * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}


int gsct_volume_loss(gsct_ctx c, const float* rendered, const float* target, const int dims[3], double alpha_ssim,
                     float* grad, int location, double* out3) {
  return run(c, [&] {
    contract(dims != nullptr && rendered && target && grad && out3, "volume_loss: null argument");
    contract(dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1, "l1: empty input");
    contract(std::isfinite(alpha_ssim) && alpha_ssim >= 0.0, "total_loss_fit: alpha_ssim invalid");
    if (alpha_ssim > 0.0)
      contract(dims[0] >= 11 && dims[1] >= 11 && dims[2] >= 11, "ssim3d: volume smaller than the 11^3 window");
    const size_t nvox = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
    const float* p = rendered;
    const float* t = target;
    float* g = grad;
    if (location == GSCT_HOST) {
      float* dp = ws<float>(c, S_LOSS_IN, nvox);
      float* dt = ws<float>(c, S_LOSS_TGT, nvox);
      CK(cudaMemcpyAsync(dp, rendered, nvox * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(dt, target, nvox * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      p = dp, t = dt;
      g = ws<float>(c, S_LOSS_GRAD, nvox);
    }
    double w[11];
    ssim_window(w);
    const int64_t ns = volume_loss_scratch_doubles(dims);
    double* scr = ws<double>(c, S_VLOSS_SCR, static_cast<size_t>(ns));
    launch_volume_loss(p, t, dims, w, alpha_ssim, scr, g, out3, c->stream);
    CK(cudaGetLastError());
    if (location == GSCT_HOST) CK(cudaMemcpyAsync(grad, g, nvox * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    double sums[2] = {0, 0};
    // {sum s, sum |d|} sit after the two 5-channel buffers and the two partial arrays
    const int64_t nb = (static_cast<int64_t>(nvox) + 255) / 256;
    CK(cudaMemcpyAsync(sums, scr + 10 * static_cast<int64_t>(nvox) + 2 * nb, sizeof sums, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const double nout = static_cast<double>(dims[0] - 10) * (dims[1] - 10) * (dims[2] - 10);
    out3[0] = sums[1] / static_cast<double>(nvox);
    out3[1] = alpha_ssim > 0.0 ? 1.0 - sums[0] / nout : 0.0;
    out3[2] = out3[0] + alpha_ssim * out3[1];
  });
}

int gsct_tv3d(gsct_ctx c, const float* volume, const int dims[3], float* grad, int location, double* value) {
  return run(c, [&] {
    contract(dims != nullptr && volume && grad && value, "tv3d: null argument");
    contract(dims[0] >= 2 && dims[1] >= 2 && dims[2] >= 2, "tv3d: dims must be at least 2 in every axis");
    const size_t nvox = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
    const float* v = volume;
    float* g = grad;
    if (location == GSCT_HOST) {
      float* dv = ws<float>(c, S_LOSS_IN, nvox);
      CK(cudaMemcpyAsync(dv, volume, nvox * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      v = dv;
      g = ws<float>(c, S_LOSS_GRAD, nvox);
    }
    const int64_t ns = tv3d_scratch_doubles(dims);
    double* scr = ws<double>(c, S_VLOSS_SCR, static_cast<size_t>(ns));
    launch_tv3d(v, dims, scr, g, c->stream);
    CK(cudaGetLastError());
    if (location == GSCT_HOST) CK(cudaMemcpyAsync(grad, g, nvox * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    const int64_t nint = static_cast<int64_t>(dims[0] - 1) * (dims[1] - 1) * (dims[2] - 1);
    double sum = 0.0;
    CK(cudaMemcpyAsync(&sum, scr + nint + (nint + 255) / 256, sizeof sum, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *value = sum / static_cast<double>(nint);
  });
}

int gsct_raymarch_project(gsct_ctx c, const float* volume, const gsct_grid* grid, int volume_location,
                          const gsct_geometry* geom, const double* angles, int n_views, float* images,
                          int images_location) {
  return run(c, [&] {
    validate_geometry(geom, angles, n_views);
    contract(grid != nullptr && volume != nullptr, "raymarch_project: null volume");
    contract(grid->dims[0] >= 1 && grid->dims[1] >= 1 && grid->dims[2] >= 1, "Volume: dims must be at least 1");
    contract(grid->spacing > 0.0, "Volume: spacing must be positive");
    contract(images != nullptr || n_views == 0, "raymarch_project: null image buffer");
    if (n_views == 0) return;
    const size_t nvox = static_cast<size_t>(grid->dims[0]) * grid->dims[1] * grid->dims[2];
    const float* v = volume;
    if (volume_location == GSCT_HOST) {
      float* dv = ws<float>(c, S_LOSS_IN, nvox);
      CK(cudaMemcpyAsync(dv, volume, nvox * sizeof(float), cudaMemcpyHostToDevice, c->stream));
      v = dv;
    }
    std::vector<Frame> frames(static_cast<size_t>(n_views));
    for (int k = 0; k < n_views; ++k) frames[static_cast<size_t>(k)] = make_frame(geom, angles[k]);
    Frame* df = ws<Frame>(c, S_FRAMES, frames.size());
    CK(cudaMemcpyAsync(df, frames.data(), frames.size() * sizeof(Frame), cudaMemcpyHostToDevice, c->stream));
    const size_t npx = static_cast<size_t>(geom->n_u) * geom->n_v * n_views;
    float* out = images_location == GSCT_HOST ? ws<float>(c, S_LOSS_GRAD, npx) : images;
    launch_raymarch(v, grid->dims, grid->spacing, grid->origin, df, make_geo(geom), n_views, out, c->stream);
    CK(cudaGetLastError());
    if (images_location == GSCT_HOST)
      CK(cudaMemcpyAsync(images, out, npx * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int gsct_adam_step(gsct_ctx c, gsct_cloud* params, gsct_adam_state* state, const gsct_grads* grads,
                   const gsct_learning_rates* lrs) {
  return run(c, [&] {
    contract(params && state && grads && lrs, "adam_step: null argument");
    contract(params->location == GSCT_DEVICE && grads->location == GSCT_DEVICE,
             "adam_step: parameters and gradients must be device-resident");
    contract(lrs->position > 0.0 && lrs->log_scale > 0.0 && lrs->rotation > 0.0 && lrs->density > 0.0,
             "lr_schedule: rates must be positive");
    state->step += 1;
    const double bias1 = 1.0 - std::pow(0.9, static_cast<double>(state->step));
    const double bias2 = 1.0 - std::pow(0.999, static_cast<double>(state->step));
    const int64_t n = params->n;
    if (n == 0) return;
    double* const mv[8] = {state->m_pos, state->v_pos, state->m_ls, state->v_ls,
                           state->m_rot, state->v_rot, state->m_dens, state->v_dens};
    const double lr[4] = {lrs->position, lrs->log_scale, lrs->rotation, lrs->density};
    unsigned long long* skipped = ws<unsigned long long>(c, S_ADAM_SKIP, 1);
    CK(cudaMemsetAsync(skipped, 0, sizeof(unsigned long long), c->stream));
    launch_adam_step(n, const_cast<double*>(params->pos), const_cast<double*>(params->log_scale),
                     const_cast<double*>(params->quat), const_cast<double*>(params->raw_density), mv, grads->pos,
                     grads->log_scale, grads->quat, grads->raw_density, lr, bias1, bias2, skipped, c->stream);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(c->hscratch, skipped, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::memcpy(&h, c->hscratch, sizeof h);
    state->skipped_updates += static_cast<int64_t>(h);
  });
}

int gsct_accumulate_control_stats(gsct_ctx c, int64_t n, const gsct_grads* grads, gsct_control_accum* acc) {
  return run(c, [&] {
    contract(grads && acc && n >= 0, "accumulate_control_stats: null argument");
    contract(grads->location == GSCT_DEVICE, "accumulate_control_stats: gradients must be device-resident");
    if (n == 0) return;
    contract(grads->visible && grads->pos_grad_norm && grads->pos && acc->grad_norm && acc->grad_dir && acc->count,
             "OptimState: arrays out of lockstep with the cloud");
    launch_ctrl_accumulate(n, grads->visible, grads->pos_grad_norm, grads->pos, acc->grad_norm, acc->grad_dir,
                           acc->count, c->stream);
    CK(cudaGetLastError());
    if (!c->async) CK(cudaStreamSynchronize(c->stream));
  });
}

int gsct_adaptive_control(gsct_ctx c, const gsct_cloud* cloud, const gsct_adam_state* state,
                          const gsct_control_accum* acc, const gsct_rng_state* rng,
                          const gsct_control_config* cfg, int64_t capacity, gsct_cloud* out_cloud,
                          gsct_adam_state* out_state, gsct_control_accum* out_acc, gsct_adaptive_report* report) {
  return run(c, [&] {
    contract(cloud && state && acc && rng && cfg && out_cloud && out_state && out_acc && report,
             "adaptive_control: null argument");
    contract(cloud->location == GSCT_DEVICE && out_cloud->location == GSCT_DEVICE,
             "adaptive_control: clouds must be device-resident");
    contract(rng->p <= 312, "Rng::restore_state: malformed engine state");
    const Cloud d = upload_cloud(c, cloud);
    const int64_t n = d.n;
    *report = gsct_adaptive_report{0, 0, 0, 0};
    if (n == 0) return;
    const size_t un = static_cast<size_t>(n);
    void* scratch = ws<char>(c, S_CTRL, ctrl_scratch_bytes(n) + 512);
    unsigned long long* small = reinterpret_cast<unsigned long long*>(c->hscratch);
    CK(launch_ctrl_classify(d, cfg->prune_density, cfg->grad_threshold,
                            cfg->split_scale_fraction * cfg->scene_extent, cfg->max_gaussians, acc->grad_norm,
                            acc->count, scratch, small, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const unsigned long long err = small[1];
    if (err != ~0ull) {
      const int64_t i = static_cast<int64_t>(err >> 2);
      contract(false, (err & 3) == 2 ? "activate: zero quaternion in splat " + std::to_string(i)
                                     : "activate: non-finite parameter in splat " + std::to_string(i));
    }
    const int64_t survivors = static_cast<int64_t>(small[2]);
    report->pruned = n - survivors;
    report->cloned = static_cast<int64_t>(small[3]);
    report->split = static_cast<int64_t>(small[4]);
    report->n_next = survivors + report->cloned + report->split;
    contract(report->n_next <= capacity, "adaptive_control: output capacity " + std::to_string(capacity) +
                                             " < " + std::to_string(report->n_next) + " rows");
    // the split children's engine draws, 12 per split, from a copy of the caller's state:
    // the reference draws from state.rng and then replaces the state with next_state, whose
    // rng was copied before the draws (optim.hpp:244, 301, 315), so the engine is unchanged
    const int64_t n_draws = 12 * report->split;
    unsigned long long* rs = ws<unsigned long long>(c, S_CTRL_RNG, 313 + static_cast<size_t>(n_draws));
    static_assert(sizeof(gsct_rng_state) == 313 * sizeof(uint64_t), "gsct_rng_state layout");
    if (n_draws > 0) {
      CK(cudaMemcpyAsync(rs, rng, sizeof(gsct_rng_state), cudaMemcpyHostToDevice, c->stream));
      launch_mt_generate(rs, rs + 313, n_draws, c->stream);
      CK(cudaGetLastError());
    }
    const double* mv_in[8] = {state->m_pos, state->v_pos, state->m_ls, state->v_ls,
                              state->m_rot, state->v_rot, state->m_dens, state->v_dens};
    double* const mv_out[8] = {out_state->m_pos, out_state->v_pos, out_state->m_ls, out_state->v_ls,
                               out_state->m_rot, out_state->v_rot, out_state->m_dens, out_state->v_dens};
    launch_ctrl_write(d, mv_in, acc->grad_dir, scratch, rs + 313, std::log(1.6), const_cast<double*>(out_cloud->pos),
                      const_cast<double*>(out_cloud->log_scale), const_cast<double*>(out_cloud->quat),
                      const_cast<double*>(out_cloud->raw_density), mv_out, c->stream);
    CK(cudaGetLastError());
    const size_t nn = static_cast<size_t>(report->n_next);
    CK(cudaMemsetAsync(out_acc->grad_norm, 0, nn * sizeof(double), c->stream));
    CK(cudaMemsetAsync(out_acc->grad_dir, 0, 3 * nn * sizeof(double), c->stream));
    CK(cudaMemsetAsync(out_acc->count, 0, nn * sizeof(int64_t), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    out_cloud->n = report->n_next;
    out_state->step = state->step;
    out_state->skipped_updates = state->skipped_updates;
    (void)un;
  });
}

namespace {
[[noreturn]] void parse_fail(const std::string& msg, size_t offset) {
  throw CallError{GSCT_ERR_PARSE, msg + " (byte offset " + std::to_string(offset) + ")"};
}
constexpr int kFgscHalfs = 0x7c00;  // binary16 patterns 0 .. 0x7bff (positive finite + zero)
}  // namespace

int gsct_compress_model(gsct_ctx c, const gsct_cloud* cloud, uint8_t* bytes, int location, int64_t* saturated) {
  return run(c, [&] {
    contract(cloud && bytes && saturated, "compress_model: null argument");
    contract((reinterpret_cast<uintptr_t>(bytes) & 1) == 0, "compress_model: byte buffer must be 2-byte aligned");
    const Cloud d = upload_cloud(c, cloud);
    const int64_t n = d.n;
    uint8_t header[16] = {'F', 'G', 'S', 'C', 1, 0, 0, 0};
    for (int k = 0; k < 8; ++k) header[8 + k] = static_cast<uint8_t>(static_cast<uint64_t>(n) >> (8 * k));
    const size_t body_bytes = 22 * static_cast<size_t>(n);
    unsigned long long* cnt = ws<unsigned long long>(c, S_FGSC_CNT, 2);
    const unsigned long long init[2] = {0ull, ~0ull};
    CK(cudaMemcpyAsync(cnt, init, sizeof init, cudaMemcpyHostToDevice, c->stream));
    uint16_t* body = location == GSCT_DEVICE ? reinterpret_cast<uint16_t*>(bytes + 16)
                                             : ws<uint16_t>(c, S_FGSC, 11 * static_cast<size_t>(n) + 1);
    launch_fgsc_encode(d, body, cnt, c->stream);
    CK(cudaGetLastError());
    if (location == GSCT_DEVICE) {
      CK(cudaMemcpyAsync(bytes, header, 16, cudaMemcpyHostToDevice, c->stream));
    } else {
      std::memcpy(bytes, header, 16);
      if (n) CK(cudaMemcpyAsync(bytes + 16, body, body_bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    unsigned long long* h = reinterpret_cast<unsigned long long*>(c->hscratch);
    CK(cudaMemcpyAsync(h, cnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (h[1] != ~0ull) {
      const int64_t i = static_cast<int64_t>(h[1] >> 2);
      contract(false, (h[1] & 3) == 2 ? "activate: zero quaternion in splat " + std::to_string(i)
                                      : "activate: non-finite parameter in splat " + std::to_string(i));
    }
    *saturated = static_cast<int64_t>(h[0]);
    if (h[0]) std::fprintf(stderr, "gsct: warning: values saturated to the binary16 range\n");
  });
}

int gsct_decompress_model(gsct_ctx c, const uint8_t* bytes, int64_t n_bytes, int location, gsct_cloud* out) {
  return run(c, [&] {
    contract(out != nullptr && n_bytes >= 0 && (bytes || n_bytes == 0), "decompress_model: null argument");
    const std::string src = "compressed model";
    uint8_t hdr[16] = {};
    const size_t have = static_cast<size_t>(std::min<int64_t>(n_bytes, 16));
    if (have) {
      if (location == GSCT_DEVICE)
        CK(cudaMemcpy(hdr, bytes, have, cudaMemcpyDeviceToHost));
      else
        std::memcpy(hdr, bytes, have);
    }
    // ByteReader (io.hpp:56-135) order: magic, version, count, then the size check
    const auto need = [&](size_t off, size_t k, const char* what) {
      if (static_cast<size_t>(n_bytes) < off + k)
        parse_fail(src + ": truncated while reading " + what + ", need " + std::to_string(k) + " bytes, have " +
                       std::to_string(static_cast<size_t>(n_bytes) - off),
                   off);
    };
    need(0, 4, "compressed model header");
    if (std::memcmp(hdr, "FGSC", 4) != 0)
      parse_fail(src + ": bad magic for compressed model header, expected 'FGSC' got '" +
                     std::string(reinterpret_cast<const char*>(hdr), 4) + "'",
                 0);
    need(4, 4, "format version");
    uint32_t version = 0;
    for (int k = 0; k < 4; ++k) version |= static_cast<uint32_t>(hdr[4 + k]) << (8 * k);
    if (version != 1) parse_fail(src + ": unsupported version " + std::to_string(version), 4);
    need(8, 8, "splat count");
    uint64_t count = 0;
    for (int k = 0; k < 8; ++k) count |= static_cast<uint64_t>(hdr[8 + k]) << (8 * k);
    const size_t expected = 16 + 22 * static_cast<size_t>(count);
    if (static_cast<size_t>(n_bytes) != expected)
      parse_fail(src + ": file is " + std::to_string(n_bytes) + " bytes, header requires " + std::to_string(expected),
                 static_cast<size_t>(n_bytes));
    contract(out->n == static_cast<int64_t>(count), "decompress_model: output holds " + std::to_string(out->n) +
                                                        " splats, the model " + std::to_string(count));
    const int64_t n = static_cast<int64_t>(count);
    if (n == 0) return;
    contract(out->pos && out->log_scale && out->quat && out->raw_density, "decompress_model: null output array");
    // std::log over the positive binary16 values (glibc, exact reference arithmetic), once
    double* table = ws<double>(c, S_FGSC_LOG, kFgscHalfs);
    if (!c->fgsc_table_ready) {
      std::vector<double> t(kFgscHalfs, 0.0);
      for (int hb = 1; hb < kFgscHalfs; ++hb) {
        const int e = (hb >> 10) & 0x1f, m = hb & 0x3ff;
        const double v = e == 0 ? std::ldexp(static_cast<double>(m), -24) : std::ldexp(static_cast<double>(1024 + m), e - 25);
        t[static_cast<size_t>(hb)] = std::log(v);
      }
      CK(cudaMemcpy(table, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice));
      c->fgsc_table_ready = true;
    }
    const uint16_t* body;
    if (location == GSCT_DEVICE) {
      contract((reinterpret_cast<uintptr_t>(bytes) & 1) == 0, "decompress_model: byte buffer must be 2-byte aligned");
      body = reinterpret_cast<const uint16_t*>(bytes + 16);
    } else {
      uint16_t* b = ws<uint16_t>(c, S_FGSC, 11 * static_cast<size_t>(n));
      CK(cudaMemcpyAsync(b, bytes + 16, 22 * static_cast<size_t>(n), cudaMemcpyHostToDevice, c->stream));
      body = b;
    }
    const size_t un = static_cast<size_t>(n);
    double *p, *l, *q, *r;
    if (out->location == GSCT_DEVICE) {
      p = const_cast<double*>(out->pos);
      l = const_cast<double*>(out->log_scale);
      q = const_cast<double*>(out->quat);
      r = const_cast<double*>(out->raw_density);
    } else {
      c->hio.invalidate_cloud();  // decoded into the host-cloud replica's buffers
      p = ws<double>(c, S_POS, 3 * un);
      l = ws<double>(c, S_LS, 3 * un);
      q = ws<double>(c, S_Q, 4 * un);
      r = ws<double>(c, S_RAW, un);
    }
    launch_fgsc_decode(body, n, table, p, l, q, r, c->stream);
    CK(cudaGetLastError());
    if (out->location == GSCT_HOST) {
      d2h(c, const_cast<double*>(out->pos), p, 3 * un * sizeof(double), c->stream);
      d2h(c, const_cast<double*>(out->log_scale), l, 3 * un * sizeof(double), c->stream);
      d2h(c, const_cast<double*>(out->quat), q, 4 * un * sizeof(double), c->stream);
      d2h(c, const_cast<double*>(out->raw_density), r, un * sizeof(double), c->stream);
    }
    CK(cudaStreamSynchronize(c->stream));
    CK(c->hio.finish());
  });
}

int gsct_debug_voxel_boxes(gsct_ctx c, const gsct_cloud* cloud, const gsct_grid* grid, const gsct_window* window,
                           const gsct_voxel_settings* vs, int32_t* lo, int32_t* hi, uint8_t* skip) {
  return run(c, [&] {
    const VoxGrid vg = make_grid(grid);
    const Window win = make_window(grid, window);
    contract(vs != nullptr, "VoxelSettings: null");
    reset_stats(c);
    const Cloud d = upload_cloud(c, cloud);
    const size_t un = static_cast<size_t>(d.n);
    if (un == 0) return;
    int32_t* dlo = ws<int32_t>(c, S_DBG0, 3 * un);
    int32_t* dhi = ws<int32_t>(c, S_DBG1, 3 * un);
    uint8_t* dskip = ws<uint8_t>(c, S_DBG2, un);
    launch_voxel_preprocess(d, vg, win, vs->tau_cut, vs->sigma_cap, nullptr, nullptr, dlo, dhi, dskip, c->dstats,
                            c->stream);
    CK(cudaMemcpyAsync(lo, dlo, 3 * un * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(hi, dhi, 3 * un * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(skip, dskip, un, cudaMemcpyDeviceToHost, c->stream));
    finish_sync(c, nullptr, false, nullptr);
  });
}

}  // extern "C"
