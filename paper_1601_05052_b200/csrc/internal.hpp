// internal.hpp -- shared between the C-ABI translation units (not installed).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace ddb {
// A few persistent host threads for the drop-in's pageable <-> pinned
// copies (abi.cu): run(n, f) calls f(0..n-1) spread over the threads and
// the caller, and returns when all are done.
class HostPool {
 public:
  explicit HostPool(unsigned n);
  ~HostPool();
  void run(unsigned n, const std::function<void(unsigned)>& f);
  unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }

 private:
  void loop();
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned next_ = 0, total_ = 0, finished_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};
}  // namespace ddb

#include "../../include/dedisp_b200.h"
#include "common.cuh"

struct dd_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 0;
  int smem_optin = 0;
  int l2_bytes = 0;
  int cc_major = 0, cc_minor = 0;
  uint32_t* d_scratch = nullptr;  // 4 x u32 reduction slots
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  void* d_flush = nullptr;  // cold-L2 timing buffer (2 x L2), lazily allocated
  uint64_t flush_bytes = 0;
  // dd_dedisperse's device buffers (grown, never shrunk) and its last plan,
  // reused while the table (host copy compared) and the config repeat
  void* d_in = nullptr;
  void* d_sh = nullptr;
  void* d_out = nullptr;
  uint64_t in_cap = 0, sh_cap = 0, out_cap = 0;
  std::vector<uint32_t> cached_table;
  dd_plan* cached_plan = nullptr;
  uint64_t cached_key[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  dd_config last_run{};
  uint32_t last_family = 0;
  // pageable host buffers (the reference API's std::vectors) go through two
  // pinned bounce buffers: host threads copy one while the DMA engine moves
  // the other
  void* h_bounce[2] = {nullptr, nullptr};
  uint64_t bounce_bytes = 0;
  cudaEvent_t ev_bounce[2] = {nullptr, nullptr};
  ddb::HostPool* pool = nullptr;
  uint32_t cached_max_delay = 0;  // of cached_table
};

#include <cuda.h>

struct dd_plan {
  dd_context* ctx = nullptr;
  // rectangle family (DD_STAGING_RECT): kernel, group lows, tensor map cache
  void (*rect_fn)(const CUtensorMap, const ddb::TiledArgs) = nullptr;
  uint32_t* d_glo = nullptr;
  CUtensorMap tmap{};
  const float* tmap_in = nullptr;
  uint64_t tmap_beam_stride = 0;
  uint32_t tmap_beams = 0;
  uint32_t family = DD_STAGING_DIRECT;
  bool reference_order = false;
  ddb::TiledArgs args{};
  const uint32_t* d_shifts = nullptr;
  uint8_t* d_rec = nullptr;
  uint2* d_ls = nullptr;
  uint32_t* d_chan_span = nullptr;  // [channels] widest span per channel (k_plan)
  uint32_t* d_stage_ch = nullptr;   // packed stages: [stages + 1] first channels
  uint32_t* d_chan_off = nullptr;   // packed stages: [channels] window offsets
  void (*smem_fn)(const ddb::TiledArgs) = nullptr;
  void (*smem_fn_fixed)(const ddb::TiledArgs) = nullptr;  // channel-range passes of a packed plan
  uint32_t blocks = 0, threads = 0, smem = 0;
  uint32_t grid_y = 1;
  uint32_t max_span = 0, max_delay = 0, group_span = 0, regwin_span = 0;
  uint64_t staged_bytes = 0;
};

namespace ddb {

// error state (abi.cu)
dd_status fail(dd_status st, const std::string& msg);
dd_status cuda_fail(cudaError_t e, const char* where);
void clear_error();

// launchers (table.cu, dedisp.cu)
cudaError_t launch_delay_table(uint32_t* d_shifts, uint32_t* d_max, uint32_t num_dms,
                               uint32_t channels, uint32_t dm_offset, double f_min, double width,
                               double dm_first, double dm_step, double rate, cudaStream_t st);
cudaError_t launch_plan(const uint32_t* d_shifts, uint8_t* d_rec, uint2* d_ls, uint32_t* d_max_span,
                        unsigned long long* d_span_sum, uint32_t channels, uint32_t tiles_dm,
                        uint32_t tile_dm, uint32_t group, uint32_t rec_bytes, uint32_t window_format,
                        uint32_t* d_chan_span, cudaStream_t st);
cudaError_t launch_max_u32(const uint32_t* d_v, uint64_t n, uint32_t* d_out, cudaStream_t st);
cudaError_t launch_flush_read(const void* buf, uint64_t bytes, uint32_t* sink, cudaStream_t st);

using KernelFn = void (*)(const TiledArgs);
// Staged-kernel variant for work_dm x work_time; nullptr when not
// instantiated.  *max_threads = the variant's block-size cap.
// items_time != 0 selects a compile-time-stride build when one exists
KernelFn find_smem_kernel(uint32_t k, uint32_t w, uint32_t* max_threads = nullptr,
                          uint32_t items_time = 0, KernelFn* packed = nullptr);
// Register-window variant for (work_dm, work_time) covering group_span
// (or the widest one); *span_out = its SPAN.  nullptr when not instantiated.
KernelFn find_regwin_kernel(uint32_t k, uint32_t w, uint32_t group_span, uint32_t* span_out);
bool regwin_shape_ok(uint32_t k, uint32_t w, uint32_t items_time, uint64_t block);
KernelFn find_tmem_kernel(uint32_t k, uint32_t w, uint32_t group_span, uint32_t* span_out,
                          bool occ = false);
bool tmem_shape_ok(uint32_t k, uint32_t w, uint32_t items_time, uint64_t block);
bool tmem_has_occupancy_build(uint32_t k, uint32_t w);
// True when the staged family can run cfg (block size within the variant's cap).
inline bool smem_variant_ok(uint32_t k, uint32_t w, uint64_t block, uint32_t items_time = 0) {
  uint32_t cap = 0;
  return find_smem_kernel(k, w, &cap, items_time) != nullptr && ((block + 31) & ~31ull) <= cap;
}
cudaError_t launch_reference(const float* in, uint64_t pitch, const uint32_t* shifts, float* out,
                             uint64_t out_pitch, uint32_t channels, uint32_t s, uint32_t num_dms,
                             cudaStream_t st);
cudaError_t launch_direct(const TiledArgs& a, uint32_t blocks, uint32_t threads,
                          cudaStream_t st);
cudaError_t launch_smem(KernelFn fn, const TiledArgs& a, uint32_t blocks, uint32_t threads,
                        uint32_t smem, cudaStream_t st, uint32_t beams = 1);
cudaError_t prepare_smem(KernelFn fn, uint32_t smem);
// K6 rectangles (dedisp.cu) and their pre-pass (table.cu)
using RectFn = void (*)(const CUtensorMap, const TiledArgs);
RectFn find_rect_kernel(uint32_t k, uint32_t w, uint32_t items_time);
cudaError_t launch_rect(RectFn fn, const CUtensorMap& tmap, const TiledArgs& a, uint32_t blocks,
                        uint32_t threads, uint32_t smem, cudaStream_t st, uint32_t beams);
cudaError_t prepare_rect(RectFn fn, uint32_t smem);
cudaError_t launch_plan_rect(const uint32_t* d_shifts, uint32_t* d_glo, uint32_t* d_rec,
                             uint32_t* d_max_width, uint32_t channels, uint32_t tiles_dm,
                             uint32_t tile_dm, uint32_t rect_ch, uint32_t groups,
                             uint32_t rec_words, cudaStream_t st);
// checked builds (DDB_CHECKED): device bounds violations so far (dedisp.cu)
cudaError_t debug_violations(unsigned long long* count, int* checked, int reset);

// host logic shared with the tuner (abi.cu)
dd_limits effective_limits(const dd_limits* l);
bool setup_ok(const dd_setup* s, std::string* why);
double channel_frequency(const dd_setup& s, uint32_t ch);
double trial_dm(const dd_setup& s, uint32_t i);

}  // namespace ddb
