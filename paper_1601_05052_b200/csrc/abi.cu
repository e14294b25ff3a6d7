// abi.cu -- implementation of the C-ABI in include/dedisp_b200.h:
// contexts, memory, the reference's geometry and config rules, device shift
// tables, dedispersion plans and the host-buffer drop-in entry points.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "internal.hpp"

namespace ddb {

static thread_local std::string g_error;

dd_status fail(dd_status st, const std::string& msg) {
  g_error = msg;
  return st;
}

dd_status cuda_fail(cudaError_t e, const char* where) {
  g_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? DD_ERR_NO_DEVICE
                                                                     : DD_ERR_CUDA;
}

void clear_error() { g_error.clear(); }

HostPool::HostPool(unsigned n) {
  for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
}

HostPool::~HostPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (std::thread& t : workers_) t.join();
}

void HostPool::loop() {
  uint64_t seen = 0;
  for (;;) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
    if (stop_) return;
    seen = gen_;
    while (next_ < total_) {
      const unsigned i = next_++;
      const std::function<void(unsigned)>* f = job_;
      lk.unlock();
      (*f)(i);
      lk.lock();
      if (++finished_ == total_) done_cv_.notify_all();
    }
  }
}

void HostPool::run(unsigned n, const std::function<void(unsigned)>& f) {
  if (n == 0) return;
  std::unique_lock<std::mutex> lk(mu_);
  job_ = &f;
  next_ = 0;
  total_ = n;
  finished_ = 0;
  ++gen_;
  cv_.notify_all();
  while (next_ < total_) {  // the caller works too
    const unsigned i = next_++;
    lk.unlock();
    f(i);
    lk.lock();
    ++finished_;
  }
  done_cv_.wait(lk, [&] { return finished_ == total_; });
  job_ = nullptr;
}

dd_limits effective_limits(const dd_limits* l) {
  dd_limits out{1024u, 256u};  // KernelLimits defaults, kernels.hpp:31-34
  if (l != nullptr && (l->max_block_items != 0 || l->max_accumulators != 0)) out = *l;
  return out;
}

// ObservationSetup::validate, reference setup.cpp:31-46.
bool setup_ok(const dd_setup* s, std::string* why) {
  auto bad = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (s == nullptr) return bad("setup is null");
  if (s->samples_per_second < 1) return bad("samples_per_second must be >= 1");
  if (s->channels < 1) return bad("channels must be >= 1");
  if (!(s->f_min > 0.0) || !std::isfinite(s->f_min))
    return bad("f_min must be positive and finite");
  if (!(s->channel_width > 0.0) || !std::isfinite(s->channel_width))
    return bad("channel_width must be positive and finite");
  if (!(s->dm_step > 0.0) || !std::isfinite(s->dm_step))
    return bad("dm_step must be positive and finite");
  if (!(s->dm_first >= 0.0) || !std::isfinite(s->dm_first))
    return bad("dm_first must be non-negative and finite");
  return true;
}

// setup.hpp:23-29
double channel_frequency(const dd_setup& s, uint32_t ch) {
  return s.f_min + static_cast<double>(ch) * s.channel_width;
}
double trial_dm(const dd_setup& s, uint32_t i) {
  return s.dm_first + static_cast<double>(i) * s.dm_step;
}

}  // namespace ddb

using namespace ddb;

#define DD_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#define DD_TRY(call)                     \
  do {                                   \
    dd_status s_ = (call);               \
    if (s_ != DD_OK) return s_;          \
  } while (0)

extern "C" {

const char* dd_last_error(void) { return g_error.c_str(); }
int dd_abi_version(void) { return DD_ABI_VERSION; }

dd_status dd_device_count(int* count) {
  if (count == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "count is null");
  *count = 0;
  const cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return DD_OK;
}

// ------------------------------------------------------------ contexts --
dd_status dd_context_create(int device, dd_context** out) {
  if (out == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  int n = 0;
  DD_TRY(dd_device_count(&n));
  if (device < 0 || device >= n)
    return fail(DD_ERR_NO_DEVICE, "device " + std::to_string(device) + " not present");
  DD_CUDA(cudaSetDevice(device));
  auto* c = new dd_context;
  c->device = device;
  cudaDeviceProp p{};
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_scratch, 16);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev_start);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev_stop);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "dd_context_create");
  }
  c->own_stream = true;
  c->sm_count = p.multiProcessorCount;
  c->smem_optin = static_cast<int>(p.sharedMemPerBlockOptin);
  c->l2_bytes = p.l2CacheSize;
  c->cc_major = p.major;
  c->cc_minor = p.minor;
  if (p.major < 10)
    return delete c, fail(DD_ERR_NO_DEVICE, "device is not sm_100 class (compute capability " +
                                                std::to_string(p.major) + "." +
                                                std::to_string(p.minor) + ")");
  *out = c;
  return DD_OK;
}

dd_status dd_context_destroy(dd_context* c) {
  if (c == nullptr) return DD_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  cudaFree(c->d_scratch);
  cudaFree(c->d_flush);
  dd_plan_destroy(c->cached_plan);
  cudaFree(c->d_in);
  cudaFree(c->d_sh);
  cudaFree(c->d_out);
  for (int i = 0; i < 2; ++i) {
    cudaFreeHost(c->h_bounce[i]);
    if (c->ev_bounce[i]) cudaEventDestroy(c->ev_bounce[i]);
  }
  delete c->pool;
  cudaEventDestroy(c->ev_start);
  cudaEventDestroy(c->ev_stop);
  delete c;
  return DD_OK;
}

dd_status dd_context_set_stream(dd_context* c, void* stream) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (stream == nullptr) {
    DD_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  } else {
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  }
  return DD_OK;
}

void* dd_context_stream(dd_context* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

dd_status dd_context_synchronize(dd_context* c) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  return DD_OK;
}

dd_status dd_context_device_info(dd_context* c, int* sm_count, int* smem_optin, int* cc_major,
                                 int* cc_minor) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  if (sm_count) *sm_count = c->sm_count;
  if (smem_optin) *smem_optin = c->smem_optin;
  if (cc_major) *cc_major = c->cc_major;
  if (cc_minor) *cc_minor = c->cc_minor;
  return DD_OK;
}

// -------------------------------------------------------------- memory --
dd_status dd_device_malloc(dd_context* c, uint64_t bytes, void** ptr) {
  if (c == nullptr || ptr == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  DD_CUDA(cudaSetDevice(c->device));
  const cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 16);
  if (e == cudaErrorMemoryAllocation)
    return fail(DD_ERR_CAPACITY, "device allocation of " + std::to_string(bytes) + " bytes failed");
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  return DD_OK;
}

dd_status dd_device_free(dd_context* c, void* ptr) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaFree(ptr));
  return DD_OK;
}

dd_status dd_host_malloc(uint64_t bytes, void** ptr) {
  if (ptr == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "ptr is null");
  const cudaError_t e = cudaMallocHost(ptr, bytes ? bytes : 16);
  if (e == cudaErrorMemoryAllocation)
    return fail(DD_ERR_CAPACITY, "pinned allocation of " + std::to_string(bytes) + " bytes failed");
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  return DD_OK;
}

dd_status dd_host_free(void* ptr) {
  DD_CUDA(cudaFreeHost(ptr));
  return DD_OK;
}

dd_status dd_copy_h2d(dd_context* c, void* dst, const void* src, uint64_t bytes) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  return DD_OK;
}

dd_status dd_copy_d2h(dd_context* c, void* dst, const void* src, uint64_t bytes) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  return DD_OK;
}

dd_status dd_upload_filterbank(dd_context* c, float* d_dst, uint64_t dst_pitch,
                               const float* h_src, uint32_t channels, uint64_t num_samples) {
  if (c == nullptr || d_dst == nullptr || h_src == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (dst_pitch < num_samples) return fail(DD_ERR_INVALID_ARGUMENT, "pitch below num_samples");
  DD_CUDA(cudaSetDevice(c->device));
  DD_CUDA(cudaMemcpy2DAsync(d_dst, dst_pitch * 4, h_src, num_samples * 4, num_samples * 4,
                            channels, cudaMemcpyHostToDevice, c->stream));
  return DD_OK;
}

// ------------------------------------------------------------ geometry --
dd_status dd_setup_validate(const dd_setup* s) {
  std::string why;
  if (!setup_ok(s, &why)) return fail(DD_ERR_INVALID_ARGUMENT, why);
  return DD_OK;
}

// delay_seconds, reference setup.cpp:48-62.
dd_status dd_delay_seconds(double dm, double f_ch, double f_hi, double* out) {
  if (out == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "out is null");
  if (!std::isfinite(dm) || !std::isfinite(f_ch) || !std::isfinite(f_hi))
    return fail(DD_ERR_INVALID_ARGUMENT, "delay_seconds: non-finite input");
  if (dm < 0.0) return fail(DD_ERR_INVALID_ARGUMENT, "delay_seconds: dm must be non-negative");
  if (f_ch <= 0.0 || f_hi <= 0.0)
    return fail(DD_ERR_INVALID_ARGUMENT, "delay_seconds: frequencies must be positive");
  if (f_ch > f_hi)
    return fail(DD_ERR_INVALID_ARGUMENT,
                "delay_seconds: channel frequency above the reference frequency");
  const double inv_low = 1.0 / (f_ch * f_ch);
  const double inv_high = 1.0 / (f_hi * f_hi);
  *out = 4150.0 * dm * (inv_low - inv_high);
  return DD_OK;
}

// instance_sizing, reference setup.cpp:112-137.
dd_status dd_instance_sizing(const dd_setup* s, uint32_t num_dms, uint64_t* num_samples,
                             uint64_t* flop, uint32_t* max_delay) {
  DD_TRY(dd_setup_validate(s));
  if (num_dms < 1) return fail(DD_ERR_INVALID_ARGUMENT, "num_dms must be >= 1");
  double worst = 0.0;
  DD_TRY(dd_delay_seconds(trial_dm(*s, num_dms - 1), channel_frequency(*s, 0),
                          channel_frequency(*s, s->channels - 1), &worst));
  const double worst_samples = worst * static_cast<double>(s->samples_per_second);
  if (worst_samples >= 4294967295.0)
    return fail(DD_ERR_CAPACITY, "maximum shift does not fit 32 bits");
  const uint32_t md = static_cast<uint32_t>(std::llround(worst_samples));
  const uint64_t rate = s->samples_per_second;
  const uint64_t blocks = (rate + md + rate - 1) / rate;
  unsigned __int128 t = static_cast<unsigned __int128>(blocks) * rate;
  unsigned __int128 f = static_cast<unsigned __int128>(num_dms) * rate * s->channels;
  if (t > std::numeric_limits<uint64_t>::max() || f > std::numeric_limits<uint64_t>::max())
    return fail(DD_ERR_CAPACITY, "sizing overflow");
  if (num_samples) *num_samples = static_cast<uint64_t>(t);
  if (flop) *flop = static_cast<uint64_t>(f);
  if (max_delay) *max_delay = md;
  return DD_OK;
}

// --------------------------------------------------------- K1: tables --
dd_status dd_delay_table_device(dd_context* c, const dd_setup* s, uint32_t num_dms,
                                uint32_t dm_offset, int zero, uint32_t* d_shifts,
                                uint32_t* max_delay) {
  if (c == nullptr || d_shifts == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  DD_TRY(dd_setup_validate(s));
  if (num_dms < 1) return fail(DD_ERR_INVALID_ARGUMENT, "num_dms must be >= 1");
  // delay_seconds rejects a non-finite trial DM (setup.cpp:49-51).
  if (!std::isfinite(trial_dm(*s, dm_offset + num_dms - 1)))
    return fail(DD_ERR_INVALID_ARGUMENT, "delay_seconds: non-finite input");
  DD_CUDA(cudaSetDevice(c->device));
  const uint64_t entries = static_cast<uint64_t>(num_dms) * s->channels;
  if (zero) {
    DD_CUDA(cudaMemsetAsync(d_shifts, 0, entries * 4, c->stream));
    if (max_delay) *max_delay = 0;
    return DD_OK;
  }
  DD_CUDA(cudaMemsetAsync(c->d_scratch, 0, 4, c->stream));
  DD_CUDA(launch_delay_table(d_shifts, c->d_scratch, num_dms, s->channels, dm_offset, s->f_min,
                             s->channel_width, s->dm_first, s->dm_step,
                             static_cast<double>(s->samples_per_second), c->stream));
  if (max_delay) {
    DD_CUDA(cudaMemcpyAsync(max_delay, c->d_scratch, 4, cudaMemcpyDeviceToHost, c->stream));
    DD_CUDA(cudaStreamSynchronize(c->stream));
  }
  return DD_OK;
}

// build_delay_table / build_zero_delay_table (setup.cpp:66-110) with the
// table computed by K1 and returned in host memory.
dd_status dd_build_delay_table(dd_context* c, const dd_setup* s, uint32_t num_dms,
                               uint64_t cap, int zero, uint32_t* h_shifts, uint32_t* max_delay) {
  if (c == nullptr || h_shifts == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  DD_TRY(dd_setup_validate(s));
  if (num_dms < 1) return fail(DD_ERR_INVALID_ARGUMENT, "num_dms must be >= 1");
  const unsigned __int128 bytes = static_cast<unsigned __int128>(num_dms) * s->channels * 4u;
  if (bytes > cap)
    return fail(DD_ERR_CAPACITY, "delay table of " + std::to_string(static_cast<uint64_t>(bytes)) +
                                     " bytes exceeds the cap of " + std::to_string(cap));
  void* d = nullptr;
  DD_TRY(dd_device_malloc(c, static_cast<uint64_t>(bytes), &d));
  uint32_t md = 0;
  dd_status st = dd_delay_table_device(c, s, num_dms, 0, zero, static_cast<uint32_t*>(d), &md);
  if (st == DD_OK) {
    const cudaError_t e = cudaMemcpyAsync(h_shifts, d, static_cast<size_t>(bytes),
                                          cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e2 = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) st = cuda_fail(e, "table download");
    else if (e2 != cudaSuccess) st = cuda_fail(e2, "table download");
  }
  cudaFree(d);
  if (st == DD_OK && max_delay) *max_delay = md;
  return st;
}

// ------------------------------------------------------------- configs --
// config_valid / validate_config, reference kernels.cpp:44-81.
int dd_config_valid(const dd_config* k, uint32_t num_dms, uint32_t s, const dd_limits* limits) {
  if (k == nullptr) return 0;
  const dd_limits L = effective_limits(limits);
  if (!k->items_time || !k->items_dm || !k->work_time || !k->work_dm) return 0;
  const uint64_t tt = static_cast<uint64_t>(k->items_time) * k->work_time;
  const uint64_t td = static_cast<uint64_t>(k->items_dm) * k->work_dm;
  if (tt > s || s % tt != 0) return 0;
  if (td > num_dms || num_dms % td != 0) return 0;
  if (static_cast<uint64_t>(k->items_time) * k->items_dm > L.max_block_items) return 0;
  if (static_cast<uint64_t>(k->work_time) * k->work_dm > L.max_accumulators) return 0;
  return 1;
}

dd_status dd_validate_config(const dd_config* k, uint32_t num_dms, uint32_t s,
                             const dd_limits* limits) {
  if (k == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "config is null");
  const dd_limits L = effective_limits(limits);
  if (!k->items_time || !k->items_dm || !k->work_time || !k->work_dm)
    return fail(DD_ERR_INVALID_ARGUMENT, "kernel config parameters must all be positive");
  const uint64_t tt = static_cast<uint64_t>(k->items_time) * k->work_time;
  const uint64_t td = static_cast<uint64_t>(k->items_dm) * k->work_dm;
  const bool gpu_tiling = (k->flags & DD_CONFIG_GPU_TILING) != 0;
  if (!gpu_tiling && (tt > s || s % tt != 0))
    return fail(DD_ERR_INVALID_ARGUMENT, "items_time * work_time = " + std::to_string(tt) +
                                             " does not divide s = " + std::to_string(s));
  if (gpu_tiling && tt > 0xffffffffull)
    return fail(DD_ERR_INVALID_ARGUMENT, "tile_time overflows");
  if (td > num_dms || num_dms % td != 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "items_dm * work_dm = " + std::to_string(td) +
                                             " does not divide the trial count " +
                                             std::to_string(num_dms));
  if (static_cast<uint64_t>(k->items_time) * k->items_dm > L.max_block_items)
    return fail(DD_ERR_INVALID_ARGUMENT, "items_time * items_dm exceeds the block limit of " +
                                             std::to_string(L.max_block_items));
  if (static_cast<uint64_t>(k->work_time) * k->work_dm > L.max_accumulators)
    return fail(DD_ERR_INVALID_ARGUMENT, "work_time * work_dm exceeds the accumulator limit of " +
                                             std::to_string(L.max_accumulators));
  if (k->staging > DD_STAGING_RECT) return fail(DD_ERR_INVALID_ARGUMENT, "unknown staging mode");
  if (k->flags & ~(DD_CONFIG_GPU_TILING | DD_CONFIG_HIGH_OCCUPANCY | DD_CONFIG_TIME_MAJOR |
                   DD_CONFIG_PACKED_STAGES | DD_CONFIG_CPS_MASK | DD_CONFIG_NSTAGE_MASK |
                   DD_CONFIG_WIDE_STAGES))
    return fail(DD_ERR_INVALID_ARGUMENT, "unknown config flags");

  const uint32_t ns = (k->flags & DD_CONFIG_NSTAGE_MASK) >> DD_CONFIG_NSTAGE_SHIFT;
  if (ns == 1 || ns > 8) return fail(DD_ERR_INVALID_ARGUMENT, "pipeline stages must be 2..8");
  return DD_OK;
}

// count_loads, reference count_loads.cpp:9-68.
dd_status dd_count_loads(const uint32_t* sh, uint32_t channels, uint32_t num_dms, uint32_t s,
                         const dd_config* k, uint64_t* staged, uint64_t* ideal) {
  if (sh == nullptr || k == nullptr || channels == 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "delay table does not cover the requested trial count");
  if (!k->items_time || !k->items_dm || !k->work_time || !k->work_dm)
    return fail(DD_ERR_INVALID_ARGUMENT, "kernel config parameters must all be positive");
  const uint64_t tt = static_cast<uint64_t>(k->items_time) * k->work_time;
  const uint64_t td = static_cast<uint64_t>(k->items_dm) * k->work_dm;
  // DD_CONFIG_GPU_TILING: the predicated last time tile stages like a full one
  const bool gpu_tiling = (k->flags & DD_CONFIG_GPU_TILING) != 0;
  if (tt > s || (s % tt != 0 && !gpu_tiling) || td > num_dms || num_dms % td != 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "kernel config does not tile this instance");
  uint64_t st = 0, id = 0;
  const uint64_t tiles_time = (s + tt - 1) / tt;
  for (uint64_t dm0 = 0; dm0 < num_dms; dm0 += td)
    for (uint32_t ch = 0; ch < channels; ++ch) {
      uint32_t lo = sh[dm0 * channels + ch], hi = lo;
      for (uint64_t l = 1; l < td; ++l) {
        const uint32_t v = sh[(dm0 + l) * channels + ch];
        lo = std::min(lo, v);
        hi = std::max(hi, v);
      }
      st += (static_cast<uint64_t>(hi - lo) + tt) * tiles_time;
    }
  std::vector<uint32_t> col(num_dms);
  for (uint32_t ch = 0; ch < channels; ++ch) {
    for (uint32_t dm = 0; dm < num_dms; ++dm) col[dm] = sh[static_cast<uint64_t>(dm) * channels + ch];
    std::sort(col.begin(), col.end());
    uint64_t begin = col[0], end = static_cast<uint64_t>(col[0]) + s;
    for (uint32_t dm = 1; dm < num_dms; ++dm) {
      if (col[dm] > end) {
        id += end - begin;
        begin = col[dm];
      }
      end = static_cast<uint64_t>(col[dm]) + s;
    }
    id += end - begin;
  }
  if (staged) *staged = st;
  if (ideal) *ideal = id;
  return DD_OK;
}

// -------------------------------------------------------------- plans --
namespace {

constexpr uint32_t kSmemBudget = 112 * 1024;  // aim for 2 CTAs per SM

// Staged-family geometry for a config: shared-memory slots, stage count.
// `slack` floats per window: the register-window kernel reads up to SPAN
// samples past a window (never added), which must stay inside the slot.
bool smem_geometry(const dd_context* c, uint32_t tile_time, uint32_t tile_dm, uint32_t group,
                   uint32_t channels, uint32_t max_span, uint32_t slack, uint32_t flags,
                   uint32_t* win_cap,
                   uint32_t* rec_bytes, uint32_t* cps, uint32_t* nstage, uint32_t* smem) {
  const uint64_t wc =
      (static_cast<uint64_t>(max_span) + tile_time + slack + 6u + 3u) & ~3ull;
  const uint64_t rb = ddb::plan_rec_bytes(tile_dm, std::max<uint32_t>(1, group));
  const uint64_t slot = rb + 4 * wc;
  const uint64_t limit = static_cast<uint64_t>(c->smem_optin);
  // Wide stages amortise the per-stage synchronisation (measured: Apertif
  // TMEM 8 -> 15 channels/stage 7.30 -> 6.83 ms; LOFAR 3x2 -> 2x3 stages
  // 5.57 -> 5.06 ms), so the shape search takes the most channels per stage
  // that fit the 2-CTA budget -- from the requested count (default 8) down
  // -- with 3 stages if they fit, else 2; then the opt-in maximum.
  // DEDISP_B200_STAGE_CPS / _NSTAGE pin the shape (tuning experiments).
  uint32_t top_cps = 8;
  uint32_t ns_opts[] = {3, 2};
  const uint32_t want_cps = ((flags & DD_CONFIG_CPS_MASK) >> DD_CONFIG_CPS_SHIFT) *
                            ((flags & DD_CONFIG_WIDE_STAGES) ? 2u : 1u);
  const uint32_t want_ns = (flags & DD_CONFIG_NSTAGE_MASK) >> DD_CONFIG_NSTAGE_SHIFT;
  if (want_cps >= 1) top_cps = want_cps;
  if (want_ns >= 2 && want_ns <= 8) ns_opts[0] = ns_opts[1] = want_ns;
  if (const char* e = std::getenv("DEDISP_B200_STAGE_CPS")) {
    const uint32_t v = static_cast<uint32_t>(std::atoi(e));
    if (v >= 1 && v <= 30) top_cps = v;
  }
  if (const char* e = std::getenv("DEDISP_B200_STAGE_NSTAGE")) {
    const uint32_t v = static_cast<uint32_t>(std::atoi(e));
    if (v >= 2 && v <= 8) ns_opts[0] = ns_opts[1] = v;
  }
  for (uint64_t budget : {static_cast<uint64_t>(kSmemBudget), limit}) {
    for (uint32_t cp = top_cps; cp >= 1; --cp) {
      for (uint32_t ns : ns_opts) {
        if (cp > channels && cp != 1) continue;
        const uint64_t bytes = ddb::kPipeHeader + static_cast<uint64_t>(ns) * cp * slot;
        if (bytes <= budget && bytes <= limit) {
          *win_cap = static_cast<uint32_t>(wc);
          *rec_bytes = static_cast<uint32_t>(rb);
          *cps = cp;
          *nstage = ns;
          *smem = static_cast<uint32_t>(bytes);
          return true;
        }
      }
    }
  }
  return false;
}

void free_plan_buffers(dd_plan* p) {
  cudaFree(p->d_glo);
  p->d_glo = nullptr;
  cudaFree(p->d_rec);
  cudaFree(p->d_ls);
  cudaFree(p->d_chan_span);
  cudaFree(p->d_stage_ch);
  cudaFree(p->d_chan_off);
  p->d_rec = nullptr;
  p->d_ls = nullptr;
  p->d_chan_span = p->d_stage_ch = p->d_chan_off = nullptr;
}

// DD_CONFIG_PACKED_STAGES: with each channel's own window width (its
// widest span over the DM tiles, k_plan's chan_span) pack stages greedily
// into equal stage buffers -- 2 stages unless the config asks for more.
// Falls back silently to the fixed geometry already in `a` when no stage
// buffer of the 2-CTA budget holds the widest window.  Channel-range
// passes keep fixed slots of cps_fixed windows inside the same buffers.
cudaError_t pack_stages(dd_context* c, dd_plan* p, ddb::TiledArgs& a, uint32_t channels,
                        uint32_t slack, uint32_t flags, uint32_t* smem) {
  std::vector<uint32_t> span(channels);
  // on the context stream (which k_plan wrote d_chan_span on), then wait
  cudaError_t e = cudaMemcpyAsync(span.data(), p->d_chan_span, channels * 4,
                                  cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return e;
  const uint32_t want_ns = (flags & DD_CONFIG_NSTAGE_MASK) >> DD_CONFIG_NSTAGE_SHIFT;
  const uint32_t ns = want_ns >= 2 ? want_ns : 2;
  const uint64_t fixed = ddb::kPipeHeader + static_cast<uint64_t>(ns) * ddb::kMaxCps * a.rec_bytes;
  if (fixed >= kSmemBudget) return cudaSuccess;
  const uint32_t stage_floats = static_cast<uint32_t>((kSmemBudget - fixed) / (4ull * ns)) & ~3u;
  if (stage_floats < a.win_cap) return cudaSuccess;
  std::vector<uint32_t> stage_ch, off(channels);
  uint32_t ch = 0, widest = 0;
  while (ch < channels) {
    stage_ch.push_back(ch);
    uint32_t used = 0, n = 0;
    while (ch < channels && n < ddb::kMaxCps) {
      const uint32_t cap = (span[ch] + a.tile_time + slack + 6u + 3u) & ~3u;
      if (n > 0 && used + cap > stage_floats) break;
      off[ch++] = used;
      used += cap;
      ++n;
    }
    widest = std::max(widest, n);
  }
  stage_ch.push_back(channels);
  e = cudaMalloc(&p->d_stage_ch, stage_ch.size() * 4);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_chan_off, channels * 4);
  // pageable sources: async on the context stream, then wait so the host
  // vectors may die and the first launch on that stream sees the tables
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(p->d_stage_ch, stage_ch.data(), stage_ch.size() * 4,
                        cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(p->d_chan_off, off.data(), channels * 4, cudaMemcpyHostToDevice,
                        c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return e;
  a.packed = 1;
  a.packed_stages = static_cast<uint32_t>(stage_ch.size() - 1);
  a.stage_ch = p->d_stage_ch;
  a.chan_off = p->d_chan_off;
  a.nstage = ns;
  a.cps = widest;  // record slots per stage
  a.stage_floats = stage_floats;
  *smem = static_cast<uint32_t>(fixed - static_cast<uint64_t>(ns) * (ddb::kMaxCps - widest) *
                                            a.rec_bytes +
                                4ull * ns * stage_floats);
  return cudaSuccess;
}

// ---------------------------------------------------- K6 rectangles --
// cuTensorMapEncodeTiled from the driver (through the runtime's entry-point
// query: no libcuda link needed).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// The 3-D view (samples, channels, beams) of the input a rectangle plan
// loads boxes of rect_w samples x rect_ch channels from; re-encoded only
// when the input pointer or the beam layout changes.
dd_status rect_tensor_map(dd_plan* p, const float* d_in, uint32_t beams, uint64_t beam_stride) {
  if (p->tmap_in == d_in && p->tmap_beams == beams && p->tmap_beam_stride == beam_stride)
    return DD_OK;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (enc == nullptr) return fail(DD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const ddb::TiledArgs& a = p->args;
  cuuint64_t dims[3] = {a.in_pitch, a.channels, beams};
  cuuint64_t strides[2] = {a.in_pitch * 4ull,
                           beams > 1 ? beam_stride * 4ull : a.in_pitch * 4ull * a.channels};
  cuuint32_t box[3] = {a.rect_w, a.rect_ch, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  const CUresult r =
      enc(&p->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(d_in), dims, strides,
          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(DD_ERR_INVALID_ARGUMENT,
                "staging=rect: cuTensorMapEncodeTiled rejected the input view (error " +
                    std::to_string(static_cast<int>(r)) + ")");
  p->tmap_in = d_in;
  p->tmap_beams = beams;
  p->tmap_beam_stride = beam_stride;
  return DD_OK;
}

// Plan the rectangle family: channel groups of rect_ch (16 x DD_CONFIG_CPS,
// else the widest of 128/64/32/16/8 whose stages fit), the group lows and
// offsets from k_plan_rect, and a box rect_w = tile_time + widest group span
// (<= 256 samples, the TMA box limit -- wider spans are not this family's).
dd_status plan_rect(dd_context* c, dd_plan* p, const dd_config* k, uint32_t channels,
                    uint64_t in_pitch) {
  ddb::TiledArgs& a = p->args;
  const uint64_t block = static_cast<uint64_t>(k->items_time) * k->items_dm;
  if (in_pitch % 4 != 0) return fail(DD_ERR_INVALID_ARGUMENT, "staging=rect: input pitch % 4 != 0");
  if (block > 1024) return fail(DD_ERR_INVALID_ARGUMENT, "staging=rect: more than 1024 threads");
  ddb::RectFn fn = ddb::find_rect_kernel(k->work_dm, k->work_time, k->items_time);
  if (fn == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT,
                "staging=rect: no work_dm x work_time variant (1..16 x 1..4 instantiated)");
  if (tensor_map_encoder() == nullptr) return fail(DD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint32_t want = ((k->flags & DD_CONFIG_CPS_MASK) >> DD_CONFIG_CPS_SHIFT) * 16u;
  uint32_t ns = (k->flags & DD_CONFIG_NSTAGE_MASK) >> DD_CONFIG_NSTAGE_SHIFT;
  if (ns < 2) ns = 4;
  std::vector<uint32_t> tries;
  if (want) tries.push_back(want);
  else tries = {128u, 64u, 32u, 16u, 8u};
  for (uint32_t rc : tries) {
    rc = std::min(rc, channels);
    const uint32_t groups = (channels + rc - 1) / rc;
    const uint32_t rec_words = (rc * a.tile_dm + 3u) & ~3u;
    cudaError_t e = cudaMalloc(&p->d_glo, static_cast<uint64_t>(a.tiles_dm) * groups * 4);
    if (e == cudaSuccess)
      e = cudaMalloc(&p->d_rec, static_cast<uint64_t>(a.tiles_dm) * groups * rec_words * 4);
    uint32_t maxw = 0;
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_scratch, 0, 4, c->stream);
    if (e == cudaSuccess)
      e = ddb::launch_plan_rect(a.shifts, p->d_glo, reinterpret_cast<uint32_t*>(p->d_rec),
                                c->d_scratch, channels, a.tiles_dm, a.tile_dm, rc, groups,
                                rec_words, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&maxw, c->d_scratch, 4, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      free_plan_buffers(p);
      return cuda_fail(e, "rect pre-pass");
    }
    // + 3: the box starts at the aligned sample at or below the group low
    const uint64_t w = (static_cast<uint64_t>(a.tile_time) + maxw + 3u + 3u) & ~3ull;
    if (w > 256) {
      free_plan_buffers(p);
      return fail(DD_ERR_INVALID_ARGUMENT,
                  "staging=rect: tile_time + the widest group span = " + std::to_string(w) +
                      " samples exceeds the 256-sample TMA box (a small-d family)");
    }
    const uint64_t stage = ((rc * w * 4 + 127) & ~127ull) + ((rec_words * 4ull + 127) & ~127ull);
    const uint64_t smem = ddb::kPipeHeader + ns * stage;
    if (smem > static_cast<uint64_t>(c->smem_optin)) {
      free_plan_buffers(p);
      if (want) return fail(DD_ERR_INVALID_ARGUMENT, "staging=rect: stages do not fit shared memory");
      continue;
    }
    a.rect_w = static_cast<uint32_t>(w);
    a.rect_ch = rc;
    a.rect_groups = groups;
    a.rec = p->d_rec;
    a.rec_bytes = rec_words * 4;
    a.glo = p->d_glo;
    a.nstage = ns;
    a.cps = rc;
    a.win_cap = a.rect_w;
    a.packed = 0;
    p->rect_fn = fn;
    p->smem = static_cast<uint32_t>(smem);
    p->threads = static_cast<uint32_t>(((block + 31) & ~31ull) + 32);
    p->blocks = static_cast<uint32_t>(((a.tiles_dm + a.depth - 1) / a.depth) * a.tiles_time);
    p->family = DD_STAGING_RECT;
    p->max_span = maxw;
    p->staged_bytes = 4ull * a.tiles_time * a.tiles_dm * groups * rc * a.rect_w;
    e = ddb::prepare_rect(fn, p->smem);
    if (e != cudaSuccess) {
      free_plan_buffers(p);
      return cuda_fail(e, "cudaFuncSetAttribute");
    }
    return DD_OK;
  }
  return fail(DD_ERR_INVALID_ARGUMENT, "staging=rect: no channel group width fits shared memory");
}

dd_status max_of_device_table(dd_context* c, const uint32_t* d_shifts, uint64_t n, uint32_t* out) {
  DD_CUDA(cudaMemsetAsync(c->d_scratch, 0, 4, c->stream));
  DD_CUDA(launch_max_u32(d_shifts, n, c->d_scratch, c->stream));
  DD_CUDA(cudaMemcpyAsync(out, c->d_scratch, 4, cudaMemcpyDeviceToHost, c->stream));
  DD_CUDA(cudaStreamSynchronize(c->stream));
  return DD_OK;
}

}  // namespace

dd_status dd_config_family(dd_context* c, const dd_config* k, uint32_t channels,
                           uint32_t num_dms, uint32_t s, uint32_t max_span, uint32_t* family) {
  if (c == nullptr || k == nullptr || family == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  const uint64_t block = static_cast<uint64_t>(k->items_time) * k->items_dm;
  const uint32_t tile_time = k->items_time * k->work_time;
  const uint32_t tile_dm = k->items_dm * k->work_dm;
  (void)num_dms;
  (void)s;
  bool smem_ok = smem_variant_ok(k->work_dm, k->work_time, block, k->items_time);
  const bool regwin_ok = regwin_shape_ok(k->work_dm, k->work_time, k->items_time, block);
  if (smem_ok) {
    uint32_t a, b, cc, d, e;
    smem_ok = smem_geometry(c, tile_time, tile_dm, k->work_dm, channels, max_span, 0,
                            k->flags, &a, &b,
                            &cc, &d, &e);
  }
  switch (k->staging) {
    case DD_STAGING_AUTO:
      *family = smem_ok ? DD_STAGING_SMEM : regwin_ok ? DD_STAGING_REGWIN : DD_STAGING_DIRECT;
      return DD_OK;
    case DD_STAGING_RECT:
      if (find_rect_kernel(k->work_dm, k->work_time, k->items_time) == nullptr || block > 1024)
        return fail(DD_ERR_INVALID_ARGUMENT,
                    "staging=rect: no work_dm x work_time variant or more than 1024 threads");
      *family = DD_STAGING_RECT;
      return DD_OK;
    case DD_STAGING_TMEM:
      if (!tmem_shape_ok(k->work_dm, k->work_time, k->items_time, block))
        return fail(DD_ERR_INVALID_ARGUMENT,
                    "staging=tmem: needs items_time % 32 == 0, <= 256 threads and an "
                    "instantiated work_dm x work_time variant");
      *family = DD_STAGING_TMEM;
      return DD_OK;
    case DD_STAGING_REGWIN:
      if (!regwin_ok)
        return fail(DD_ERR_INVALID_ARGUMENT,
                    "staging=regwin: needs items_time % 32 == 0, <= 256 threads and an "
                    "instantiated work_dm x work_time variant");
      *family = DD_STAGING_REGWIN;
      return DD_OK;
    case DD_STAGING_SMEM:
      if (!smem_ok)
        return fail(DD_ERR_INVALID_ARGUMENT,
                    "staging=smem: no staged kernel for this config (work_dm x work_time "
                    "variant, block size or shared-memory window)");
      *family = DD_STAGING_SMEM;
      return DD_OK;
    case DD_STAGING_DIRECT:
      *family = DD_STAGING_DIRECT;
      return DD_OK;
    default:
      return fail(DD_ERR_INVALID_ARGUMENT, "staging mode not available in this build");
  }
}

dd_status dd_plan_create(dd_context* c, const uint32_t* d_shifts, uint32_t channels,
                         uint32_t num_dms, uint32_t s, uint64_t num_samples, uint64_t in_pitch,
                         const dd_config* k, const dd_limits* limits, dd_plan** out) {
  if (out == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "out is null");
  *out = nullptr;
  if (c == nullptr || d_shifts == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (channels == 0 || s == 0) return fail(DD_ERR_INVALID_ARGUMENT, "empty setup");
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "delay table holds no trials");
  if (in_pitch < num_samples) return fail(DD_ERR_INVALID_ARGUMENT, "input pitch below num_samples");
  if (k != nullptr) DD_TRY(dd_validate_config(k, num_dms, s, limits));
  DD_CUDA(cudaSetDevice(c->device));

  uint32_t md = 0;
  DD_TRY(max_of_device_table(c, d_shifts, static_cast<uint64_t>(num_dms) * channels, &md));
  // check_pair, reference kernels.cpp:22-27
  const uint64_t needed = static_cast<uint64_t>(s) + md;
  if (num_samples < needed)
    return fail(DD_ERR_INVALID_ARGUMENT, "filterbank too short: need " + std::to_string(needed) +
                                             " samples per channel, have " +
                                             std::to_string(num_samples));

  auto* p = new dd_plan;
  p->ctx = c;
  p->d_shifts = d_shifts;
  p->max_delay = md;
  ddb::TiledArgs& a = p->args;
  a.in_pitch = in_pitch;
  a.shifts = d_shifts;
  a.channels = channels;
  a.s = s;
  a.num_dms = num_dms;

  if (k == nullptr) {
    p->reference_order = true;
    p->family = DD_STAGING_DIRECT;
    *out = p;
    return DD_OK;
  }

  a.items_time = k->items_time;
  a.items_dm = k->items_dm;
  a.work_time = k->work_time;
  a.work_dm = k->work_dm;
  a.tile_time = k->items_time * k->work_time;
  a.tile_dm = k->items_dm * k->work_dm;
  a.tiles_time = (s + a.tile_time - 1) / a.tile_time;  // last tile predicated (GPU tiling)
  a.tiles_dm = num_dms / a.tile_dm;
  a.ch_begin = 0;
  a.ch_end = channels;
  a.accumulate = 0;
  a.in_beam_stride = 0;
  a.out_beam_stride = 0;
  a.depth = std::max<uint32_t>(1, k->dm_tile_depth);
  a.depth = std::min(a.depth, a.tiles_dm);
  a.time_major = (k->flags & DD_CONFIG_TIME_MAJOR) ? 1u : 0u;
  if (k->staging == DD_STAGING_AUTO && !a.time_major) {
    // AUTO also picks the raster: DM-fastest unless the windows of the
    // CTAs resident at once (~2 per SM, one time tile, their DM range)
    // would overflow 3/4 of the L2 -- large delays (LOFAR), where the block
    // would otherwise stream from HBM once per time tile.
    const double resident_dms = std::min<double>(
        num_dms, 2.0 * c->sm_count * a.tile_dm * std::max<uint32_t>(1, a.depth));
    const double window = a.tile_time + static_cast<double>(md) * resident_dms / num_dms;
    if (4.0 * channels * window > 0.75 * c->l2_bytes) a.time_major = 1;
  }

  if (k->staging == DD_STAGING_RECT) {
    const dd_status st = plan_rect(c, p, k, channels, in_pitch);
    if (st != DD_OK) {
      delete p;
      return st;
    }
    *out = p;
    return DD_OK;
  }

  const uint64_t block = static_cast<uint64_t>(k->items_time) * k->items_dm;
  const bool smem_shape = smem_variant_ok(k->work_dm, k->work_time, block, k->items_time);
  const bool regwin_shape = regwin_shape_ok(k->work_dm, k->work_time, k->items_time, block);
  const bool tmem_shape = tmem_shape_ok(k->work_dm, k->work_time, k->items_time, block);
  bool staged = in_pitch % 4 == 0;
  switch (k->staging) {
    case DD_STAGING_AUTO: staged = staged && (smem_shape || regwin_shape); break;
    case DD_STAGING_SMEM: staged = staged && smem_shape; break;
    case DD_STAGING_REGWIN: staged = staged && regwin_shape; break;
    case DD_STAGING_TMEM: staged = staged && tmem_shape; break;
    default: staged = false;
  }

  if (staged) {
    a.rec_bytes = ddb::plan_rec_bytes(a.tile_dm, k->work_dm);
    const uint64_t rec_total = static_cast<uint64_t>(a.tiles_dm) * channels * a.rec_bytes;
    cudaError_t e = cudaMalloc(&p->d_rec, rec_total);
    if (e == cudaSuccess)
      e = cudaMalloc(&p->d_ls, static_cast<uint64_t>(a.tiles_dm) * channels * sizeof(uint2));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_chan_span, channels * sizeof(uint32_t));
    if (e == cudaSuccess)
      e = cudaMemsetAsync(p->d_chan_span, 0, channels * sizeof(uint32_t), c->stream);
    uint32_t scratch[4] = {0, 0, 0, 0};
    unsigned long long* d_sum = reinterpret_cast<unsigned long long*>(c->d_scratch + 2);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_scratch, 0, 16, c->stream);
    if (e == cudaSuccess)
      e = launch_plan(d_shifts, p->d_rec, p->d_ls, c->d_scratch, d_sum, channels, a.tiles_dm, a.tile_dm,
                      k->work_dm, a.rec_bytes,
                      k->staging == DD_STAGING_TMEM ? k->work_time : 0u, p->d_chan_span,
                      c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(scratch, c->d_scratch, 16, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
      free_plan_buffers(p);
      delete p;
      return cuda_fail(e, "plan pre-pass");
    }
    p->max_span = scratch[0];
    p->group_span = scratch[1];
    uint64_t span_sum = 0;
    std::memcpy(&span_sum, scratch + 2, 8);

    uint32_t family = k->staging;
    if (family == DD_STAGING_AUTO)
      // AUTO: the shared-memory kernel (fastest measured family, round 1),
    // register windows where it has no variant.
    family = smem_shape ? DD_STAGING_SMEM : DD_STAGING_REGWIN;
    ddb::KernelFn fn = nullptr, fn_packed = nullptr;
    uint32_t slack = 0;
    if (family == DD_STAGING_REGWIN) {
      fn = find_regwin_kernel(k->work_dm, k->work_time, p->group_span, &p->regwin_span);
      slack = p->regwin_span + 4;
    } else if (family == DD_STAGING_TMEM) {
      // three-CTA builds when the CTA is <= 4 consumer warps and one exists
      const bool small = ((block + 31) & ~31ull) + 32 <= 160;
      if (small && (k->flags & DD_CONFIG_HIGH_OCCUPANCY))
        fn = find_tmem_kernel(k->work_dm, k->work_time, p->group_span, &p->regwin_span, true);
      if (fn == nullptr)
        fn = find_tmem_kernel(k->work_dm, k->work_time, p->group_span, &p->regwin_span);
      slack = p->regwin_span + 8;
    } else {
      fn = find_smem_kernel(k->work_dm, k->work_time, nullptr, k->items_time, &fn_packed);
    }
    uint32_t win_cap = 0, rec_bytes = 0, cps = 0, nstage = 0, smem = 0;
    // the launch must fit the variant's register budget
    const uint32_t threads = static_cast<uint32_t>(((block + 31) & ~31ull) + 32);
    cudaFuncAttributes fattr{};
    if (fn != nullptr && (cudaFuncGetAttributes(&fattr, fn) != cudaSuccess ||
                          static_cast<uint32_t>(fattr.maxThreadsPerBlock) < threads))
      fn = nullptr;
    if (fn != nullptr &&
        smem_geometry(c, a.tile_time, a.tile_dm, k->work_dm, channels, p->max_span, slack,
                      k->flags, &win_cap,
                      &rec_bytes, &cps, &nstage, &smem)) {
      a.win_cap = win_cap;
      a.cps = cps;
      a.nstage = nstage;
      a.stage_floats = cps * win_cap;
      a.packed = 0;
      a.rec = p->d_rec;
      a.ls = p->d_ls;
      p->smem_fn_fixed = fn;
      if ((k->flags & DD_CONFIG_PACKED_STAGES) && fn_packed != nullptr) {
        // only the K3 shapes with a packed build; otherwise the flag is a no-op
        e = pack_stages(c, p, a, channels, slack, k->flags, &smem);
        if (e != cudaSuccess) {
          free_plan_buffers(p);
          delete p;
          return cuda_fail(e, "packed stages");
        }
        if (a.packed) fn = fn_packed;
      }
      p->smem_fn = fn;
      p->smem = smem;
      // whole consumer warps plus one producer warp (dedisp.cu staged_loop)
      p->threads = threads;
      const uint64_t groups_dm = (a.tiles_dm + a.depth - 1) / a.depth;
      p->blocks = static_cast<uint32_t>(groups_dm * a.tiles_time);
      p->family = family;
      e = prepare_smem(p->smem_fn, smem);
      if (e == cudaSuccess && p->smem_fn_fixed != p->smem_fn) e = prepare_smem(p->smem_fn_fixed, smem);
      if (e != cudaSuccess) {
        free_plan_buffers(p);
        delete p;
        return cuda_fail(e, "cudaFuncSetAttribute");
      }
      // count_loads' staged elements (count_loads.cpp:33-45) x 4 bytes.
      p->staged_bytes = 4ull * a.tiles_time *
                        (span_sum + static_cast<uint64_t>(a.tiles_dm) * channels * a.tile_time);
      *out = p;
      return DD_OK;
    }
    free_plan_buffers(p);
  }
  if (k->staging == DD_STAGING_SMEM || k->staging == DD_STAGING_REGWIN ||
      k->staging == DD_STAGING_TMEM ||
      (k->flags & DD_CONFIG_GPU_TILING && s % a.tile_time != 0)) {
    delete p;
    return fail(DD_ERR_INVALID_ARGUMENT,
                std::string("staging=") +
                    (k->staging == DD_STAGING_SMEM ? "smem"
                     : k->staging == DD_STAGING_TMEM ? "tmem" : "regwin") +
                    ": no staged kernel for this config (work_dm x work_time variant, block "
                    "size, items_time, input pitch or shared-memory window)");
  }
  // Direct family: pack small tiles, virtualise oversize blocks.
  const uint32_t bi = static_cast<uint32_t>(std::min<uint64_t>(block, 0xffffffffull));
  a.pack = bi >= 256 ? 1 : 256 / bi;
  a.vthreads = a.pack * bi;
  p->threads = std::min<uint32_t>(256, (a.vthreads + 31) & ~31u);
  const uint64_t tiles = static_cast<uint64_t>(a.tiles_time) * a.tiles_dm;
  const uint64_t blocks = (tiles + a.pack - 1) / a.pack;
  if (blocks > 0x7fffffffULL) {
    delete p;
    return fail(DD_ERR_CAPACITY, "too many tiles for one launch");
  }
  p->blocks = static_cast<uint32_t>(blocks);
  p->family = DD_STAGING_DIRECT;
  *out = p;
  return DD_OK;
}

dd_status dd_plan_destroy(dd_plan* p) {
  if (p == nullptr) return DD_OK;
  if (p->d_rec || p->d_glo) {
    cudaSetDevice(p->ctx->device);
    free_plan_buffers(p);
  }
  delete p;
  return DD_OK;
}

dd_status dd_plan_get_info(const dd_plan* p, dd_plan_info* info) {
  if (p == nullptr || info == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->family = p->family;
  info->max_span = p->max_span;
  info->max_delay = p->max_delay;
  info->grid_x = p->blocks;
  info->grid_y = 1;
  info->block_threads = p->threads;
  info->smem_bytes = p->smem;
  info->channels_per_stage = p->args.cps;
  info->stages = p->args.nstage;
  info->kernel_launches = 1;
  info->staged_bytes = p->staged_bytes;
  info->time_major = p->args.time_major;
  info->packed_stages = p->args.packed ? p->args.packed_stages : 0;
  const void* kfn = p->smem_fn ? reinterpret_cast<const void*>(p->smem_fn)
                               : reinterpret_cast<const void*>(p->rect_fn);
  if (kfn != nullptr) {
    cudaFuncAttributes fa{};
    int ctas = 0;
    if (cudaFuncGetAttributes(&fa, kfn) == cudaSuccess) info->registers = fa.numRegs;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, kfn, static_cast<int>(p->threads),
                                                      p->smem) == cudaSuccess)
      info->ctas_per_sm = static_cast<uint32_t>(ctas);
  }
  if (p->reference_order) {
    const uint64_t n = static_cast<uint64_t>(p->args.num_dms) * p->args.s;
    info->grid_x = static_cast<uint32_t>((n + 255) / 256);
    info->block_threads = 256;
  }
  return DD_OK;
}

dd_status dd_plan_execute(dd_plan* p, const float* d_in, float* d_out, uint64_t out_pitch) {
  if (p == nullptr || d_in == nullptr || d_out == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (out_pitch < p->args.s) return fail(DD_ERR_INVALID_ARGUMENT, "output pitch below s");
  dd_context* c = p->ctx;
  DD_CUDA(cudaSetDevice(c->device));
  if (p->reference_order) {
    DD_CUDA(launch_reference(d_in, p->args.in_pitch, p->d_shifts, d_out, out_pitch,
                             p->args.channels, p->args.s, p->args.num_dms, c->stream));
    return DD_OK;
  }
  ddb::TiledArgs a = p->args;
  a.in = d_in;
  a.out = d_out;
  a.out_pitch = out_pitch;
  if (p->family == DD_STAGING_RECT) {
    if ((reinterpret_cast<uintptr_t>(d_in) & 15u) != 0)
      return fail(DD_ERR_INVALID_ARGUMENT, "staged kernels need a 16-byte aligned input");
    DD_TRY(rect_tensor_map(p, d_in, 1, 0));
    DD_CUDA(launch_rect(p->rect_fn, p->tmap, a, p->blocks, p->threads, p->smem, c->stream, 1));
  } else if (p->family == DD_STAGING_SMEM || p->family == DD_STAGING_REGWIN ||
             p->family == DD_STAGING_TMEM) {
    if ((reinterpret_cast<uintptr_t>(d_in) & 15u) != 0)
      return fail(DD_ERR_INVALID_ARGUMENT, "staged kernels need a 16-byte aligned input");
    DD_CUDA(launch_smem(p->smem_fn, a, p->blocks, p->threads, p->smem, c->stream));
  } else {
    DD_CUDA(launch_direct(a, p->blocks, p->threads, c->stream));
  }
  return DD_OK;
}

dd_status dd_plan_execute_channels(dd_plan* p, const float* d_in, float* d_out,
                                   uint64_t out_pitch, uint32_t ch_begin, uint32_t ch_end,
                                   int accumulate) {
  if (p == nullptr || d_in == nullptr || d_out == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (p->reference_order || p->family == DD_STAGING_DIRECT)
    return fail(DD_ERR_INVALID_ARGUMENT, "channel ranges need a staged kernel family");
  if (ch_begin >= ch_end || ch_end > p->args.channels)
    return fail(DD_ERR_INVALID_ARGUMENT, "bad channel range");
  if (out_pitch < p->args.s) return fail(DD_ERR_INVALID_ARGUMENT, "output pitch below s");
  if ((reinterpret_cast<uintptr_t>(d_in) & 15u) != 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "staged kernels need a 16-byte aligned input");
  dd_context* c = p->ctx;
  DD_CUDA(cudaSetDevice(c->device));
  ddb::TiledArgs a = p->args;
  a.in = d_in;
  a.out = d_out;
  a.out_pitch = out_pitch;
  a.ch_begin = ch_begin;
  a.ch_end = ch_end;
  a.accumulate = accumulate ? 1u : 0u;
  if (p->family == DD_STAGING_RECT) {
    DD_TRY(rect_tensor_map(p, d_in, 1, 0));
    DD_CUDA(launch_rect(p->rect_fn, p->tmap, a, p->blocks, p->threads, p->smem, c->stream, 1));
    return DD_OK;
  }
  ddb::KernelFn fn = p->smem_fn;
  if (a.packed && (ch_begin != 0 || ch_end != a.channels)) {
    // packed stages cover the full channel range; a sub-range runs the fixed
    // build with slots of the widest window inside the same stage buffers
    a.packed = 0;
    a.cps = std::max(1u, std::min(a.cps, a.stage_floats / a.win_cap));
    a.win_cap = a.stage_floats / a.cps;  // (fixed build strides slot * cps * win_cap)
    a.win_cap &= ~3u;
    fn = p->smem_fn_fixed;
  }
  DD_CUDA(launch_smem(fn, a, p->blocks, p->threads, p->smem, c->stream));
  return DD_OK;
}

dd_status dd_plan_execute_beams(dd_plan* p, uint32_t beams, const float* d_in,
                                uint64_t in_beam_stride, float* d_out, uint64_t out_pitch,
                                uint64_t out_beam_stride) {
  if (p == nullptr || d_in == nullptr || d_out == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (beams == 0 || beams > 65535) return fail(DD_ERR_INVALID_ARGUMENT, "beams must be 1..65535");
  if (p->reference_order || p->family == DD_STAGING_DIRECT)
    return fail(DD_ERR_INVALID_ARGUMENT, "beam batching needs a staged kernel family");
  if (out_pitch < p->args.s) return fail(DD_ERR_INVALID_ARGUMENT, "output pitch below s");
  if (beams > 1 && (in_beam_stride < p->args.in_pitch * p->args.channels ||
                    out_beam_stride < out_pitch * p->args.num_dms))
    return fail(DD_ERR_INVALID_ARGUMENT, "beam strides overlap");
  if ((reinterpret_cast<uintptr_t>(d_in) & 15u) != 0 || in_beam_stride % 4 != 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "staged kernels need 16-byte aligned beam inputs");
  dd_context* c = p->ctx;
  DD_CUDA(cudaSetDevice(c->device));
  ddb::TiledArgs a = p->args;
  a.in = d_in;
  a.out = d_out;
  a.out_pitch = out_pitch;
  a.in_beam_stride = in_beam_stride;
  a.out_beam_stride = out_beam_stride;
  if (p->family == DD_STAGING_RECT) {
    DD_TRY(rect_tensor_map(p, d_in, beams, in_beam_stride));
    DD_CUDA(launch_rect(p->rect_fn, p->tmap, a, p->blocks, p->threads, p->smem, c->stream,
                        beams));
    return DD_OK;
  }
  DD_CUDA(launch_smem(p->smem_fn, a, p->blocks, p->threads, p->smem, c->stream, beams));
  return DD_OK;
}

dd_status dd_plan_time(dd_plan* p, const float* d_in, float* d_out, uint64_t out_pitch,
                       uint32_t warmup, uint32_t repeats, double* seconds) {
  return dd_plan_time_ex(p, d_in, d_out, out_pitch, warmup, repeats, 0, seconds);
}

dd_status dd_plan_time_ex(dd_plan* p, const float* d_in, float* d_out, uint64_t out_pitch,
                          uint32_t warmup, uint32_t repeats, int flush_l2, double* seconds) {
  if (p == nullptr || (repeats > 0 && seconds == nullptr))
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  dd_context* c = p->ctx;
  DD_CUDA(cudaSetDevice(c->device));
  if (flush_l2 && c->d_flush == nullptr) {
    const uint64_t bytes = std::max<uint64_t>(2ull * static_cast<uint64_t>(c->l2_bytes), 64ull << 20);
    DD_CUDA(cudaMalloc(&c->d_flush, bytes));
    c->flush_bytes = bytes;
  }
  for (uint32_t i = 0; i < warmup; ++i) DD_TRY(dd_plan_execute(p, d_in, d_out, out_pitch));
  for (uint32_t i = 0; i < repeats; ++i) {
    // evict the instance from L2 outside the timed region (write a buffer
    // twice the L2 size, then read it back so the lines left are clean: the
    // timed kernel must not pay for writing the flush data back), as
    // bench.py does between its steps
    if (flush_l2) {
      DD_CUDA(cudaMemsetAsync(c->d_flush, i & 0xff, c->flush_bytes, c->stream));
      DD_CUDA(launch_flush_read(c->d_flush, c->flush_bytes, c->d_scratch + 3, c->stream));
    }
    DD_CUDA(cudaEventRecord(c->ev_start, c->stream));
    DD_TRY(dd_plan_execute(p, d_in, d_out, out_pitch));
    DD_CUDA(cudaEventRecord(c->ev_stop, c->stream));
    DD_CUDA(cudaEventSynchronize(c->ev_stop));
    float ms = 0.0f;
    DD_CUDA(cudaEventElapsedTime(&ms, c->ev_start, c->ev_stop));
    seconds[i] = static_cast<double>(ms) * 1e-3;
  }
  DD_CUDA(cudaStreamSynchronize(c->stream));
  return DD_OK;
}

}  // extern "C"

namespace {

// ------------------------------------------- pageable host transfers --
// The reference API hands the drop-in pageable std::vector buffers.  Large
// transfers go through two pinned bounce buffers of kBounce bytes: host
// threads copy chunk k into (out of) one buffer while the DMA engine moves
// chunk k-1 through the other, so neither the pageable-copy path of the
// driver nor a single host thread sets the rate.
constexpr uint64_t kBounce = 16ull << 20;
constexpr uint64_t kBounceMin = 8ull << 20;  // smaller transfers: plain async copy

dd_status bounce_ready(dd_context* c) {
  if (c->h_bounce[0] != nullptr) return DD_OK;
  for (int i = 0; i < 2; ++i) {
    DD_CUDA(cudaMallocHost(&c->h_bounce[i], kBounce));
    DD_CUDA(cudaEventCreateWithFlags(&c->ev_bounce[i], cudaEventDisableTiming));
  }
  c->bounce_bytes = kBounce;
  unsigned hw = std::thread::hardware_concurrency();
  c->pool = new HostPool(std::min(7u, hw > 1 ? hw - 1 : 1u));
  return DD_OK;
}

void parallel_copy(dd_context* c, void* dst, const void* src, uint64_t bytes) {
  const unsigned n = c->pool->size();
  const uint64_t per = ((bytes + n - 1) / n + 63) & ~63ull;
  c->pool->run(n, [&](unsigned i) {
    const uint64_t lo = std::min(bytes, per * i), hi = std::min(bytes, lo + per);
    if (hi > lo) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
  });
}

// Host filterbank [channels][num_samples] (pageable) -> device rows of pitch
// floats, in chunks of whole channel rows (or row pieces for huge rows).
dd_status upload_staged(dd_context* c, float* d_dst, uint64_t pitch, const float* h_src,
                        uint32_t channels, uint64_t num_samples) {
  const uint64_t row = num_samples * 4;
  if (row * channels < kBounceMin)
    return dd_upload_filterbank(c, d_dst, pitch, h_src, channels, num_samples);
  DD_TRY(bounce_ready(c));
  // pieces of at most kBounce bytes: whole rows when a row fits
  const uint64_t rows_per = std::max<uint64_t>(1, kBounce / row);
  const uint64_t piece = row <= kBounce ? row : kBounce & ~15ull;
  uint64_t k = 0;
  for (uint64_t r0 = 0; r0 < channels;) {
    if (row <= kBounce) {
      const uint64_t nr = std::min<uint64_t>(rows_per, channels - r0);
      void* hb = c->h_bounce[k & 1];
      DD_CUDA(cudaEventSynchronize(c->ev_bounce[k & 1]));  // its previous DMA is done
      parallel_copy(c, hb, h_src + r0 * num_samples, nr * row);
      DD_CUDA(cudaMemcpy2DAsync(d_dst + r0 * pitch, pitch * 4, hb, row, row, nr,
                                cudaMemcpyHostToDevice, c->stream));
      DD_CUDA(cudaEventRecord(c->ev_bounce[k & 1], c->stream));
      r0 += nr;
      ++k;
    } else {
      for (uint64_t off = 0; off < row; off += piece) {
        const uint64_t nb = std::min(piece, row - off);
        void* hb = c->h_bounce[k & 1];
        DD_CUDA(cudaEventSynchronize(c->ev_bounce[k & 1]));
        parallel_copy(c, hb, reinterpret_cast<const char*>(h_src + r0 * num_samples) + off, nb);
        DD_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d_dst + r0 * pitch) + off, hb, nb,
                                cudaMemcpyHostToDevice, c->stream));
        DD_CUDA(cudaEventRecord(c->ev_bounce[k & 1], c->stream));
        ++k;
      }
      ++r0;
    }
  }
  return DD_OK;
}

// Device buffer -> pageable host buffer (contiguous), chunked through the
// bounce buffers: the DMA of chunk k+1 runs while host threads copy chunk k.
dd_status download_staged(dd_context* c, void* h_dst, const void* d_src, uint64_t bytes,
                          cudaStream_t stream = nullptr) {
  if (stream == nullptr) stream = c->stream;
  if (bytes < kBounceMin) {
    DD_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, stream));
    DD_CUDA(cudaStreamSynchronize(stream));
    return DD_OK;
  }
  DD_TRY(bounce_ready(c));
  const uint64_t n = (bytes + kBounce - 1) / kBounce;
  auto issue = [&](uint64_t k) -> dd_status {
    const uint64_t lo = k * kBounce, nb = std::min(kBounce, bytes - lo);
    DD_CUDA(cudaMemcpyAsync(c->h_bounce[k & 1], static_cast<const char*>(d_src) + lo, nb,
                            cudaMemcpyDeviceToHost, stream));
    DD_CUDA(cudaEventRecord(c->ev_bounce[k & 1], stream));
    return DD_OK;
  };
  DD_TRY(issue(0));
  for (uint64_t k = 0; k < n; ++k) {
    DD_CUDA(cudaEventSynchronize(c->ev_bounce[k & 1]));
    if (k + 1 < n) DD_TRY(issue(k + 1));  // into the other buffer, while we copy this one
    const uint64_t lo = k * kBounce, nb = std::min(kBounce, bytes - lo);
    parallel_copy(c, static_cast<char*>(h_dst) + lo, c->h_bounce[k & 1], nb);
  }
  return DD_OK;
}

// ------------------------------------------------------ tuned schedules --
struct BuiltinSchedule {
  uint32_t channels, s, num_dms;
  dd_config cfg;
};
const BuiltinSchedule kBuiltinSchedules[] = {
#include "schedules.inc"
};

using ScheduleKey = std::tuple<uint32_t, uint32_t, uint32_t>;
std::mutex g_sched_mu;
std::map<ScheduleKey, dd_config>& registered() {
  static std::map<ScheduleKey, dd_config> m;
  return m;
}

// The config the one-shot entry points plan: the instance's tuned schedule
// for an AUTO, flag-free config (the reference API's default ExecOptions),
// else the caller's own.
bool tuned_for(const dd_config* k, uint32_t channels, uint32_t s, uint32_t num_dms,
               dd_config* out) {
  if (k == nullptr || k->staging != DD_STAGING_AUTO || k->flags != 0) return false;
  int builtin = 0;
  if (dd_schedule_get(channels, s, num_dms, out, &builtin) != DD_OK) {
    clear_error();
    return false;
  }
  return true;
}

// Plan the tuned schedule when there is one (validated against the default
// limits: it is the library's choice, not the caller's), else -- or when the
// schedule cannot be planned for this table -- the caller's config.
dd_status plan_one_shot(dd_context* c, const uint32_t* d_shifts, uint32_t channels,
                        uint32_t num_dms, uint32_t s, uint64_t num_samples, uint64_t pitch,
                        const dd_config* k, const dd_limits* limits, dd_plan** p,
                        dd_config* ran) {
  dd_config tuned{};
  if (tuned_for(k, channels, s, num_dms, &tuned)) {
    const dd_status st =
        dd_plan_create(c, d_shifts, channels, num_dms, s, num_samples, pitch, &tuned, nullptr, p);
    if (st == DD_OK) {
      *ran = tuned;
      return DD_OK;
    }
    if (st != DD_ERR_INVALID_ARGUMENT) return st;
    clear_error();
  }
  DD_TRY(dd_plan_create(c, d_shifts, channels, num_dms, s, num_samples, pitch, k, limits, p));
  *ran = k ? *k : dd_config{};
  return DD_OK;
}

}  // namespace

extern "C" {

dd_status dd_schedule_set(uint32_t channels, uint32_t s, uint32_t num_dms, const dd_config* cfg) {
  if (channels == 0 || s == 0 || num_dms == 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "instance dimensions must be positive");
  std::lock_guard<std::mutex> g(g_sched_mu);
  if (cfg == nullptr) {
    registered().erase(ScheduleKey{channels, s, num_dms});
    return DD_OK;
  }
  DD_TRY(dd_validate_config(cfg, num_dms, s, nullptr));
  registered()[ScheduleKey{channels, s, num_dms}] = *cfg;
  return DD_OK;
}

dd_status dd_schedule_get(uint32_t channels, uint32_t s, uint32_t num_dms, dd_config* cfg,
                          int* builtin) {
  if (cfg == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "cfg is null");
  {
    std::lock_guard<std::mutex> g(g_sched_mu);
    auto it = registered().find(ScheduleKey{channels, s, num_dms});
    if (it != registered().end()) {
      *cfg = it->second;
      if (builtin) *builtin = 0;
      return DD_OK;
    }
  }
  for (const BuiltinSchedule& b : kBuiltinSchedules)
    if (b.channels == channels && b.s == s && b.num_dms == num_dms) {
      *cfg = b.cfg;
      if (builtin) *builtin = 1;
      return DD_OK;
    }
  return fail(DD_ERR_INVALID_ARGUMENT, "no tuned schedule for this instance");
}

dd_status dd_last_run_config(dd_context* c, dd_config* cfg, uint32_t* family) {
  if (c == nullptr || cfg == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  *cfg = c->last_run;
  if (family) *family = c->last_family;
  return DD_OK;
}

dd_status dd_dedisperse_device(dd_context* c, const float* d_in, uint32_t channels,
                               uint64_t num_samples, uint64_t in_pitch, const uint32_t* d_shifts,
                               uint32_t num_dms, uint32_t s, const dd_config* k,
                               const dd_limits* limits, float* d_out) {
  if (c == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "context is null");
  if (k != nullptr) DD_TRY(dd_validate_config(k, num_dms, s, limits));
  dd_plan* p = nullptr;
  dd_config ran{};
  DD_TRY(plan_one_shot(c, d_shifts, channels, num_dms, s, num_samples, in_pitch, k, limits, &p,
                       &ran));
  c->last_run = ran;
  c->last_family = p->family;
  dd_status st = dd_plan_execute(p, d_in, d_out, s);
  dd_plan_destroy(p);
  return st;
}

dd_status dd_debug_violations(uint64_t* count, int* checked, int reset) {
  if (count == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "count is null");
  unsigned long long n = 0;
  int chk = 0;
  DD_CUDA(cudaDeviceSynchronize());
  DD_CUDA(debug_violations(&n, &chk, reset));
  *count = n;
  if (checked) *checked = chk;
  return DD_OK;
}

dd_status dd_fingerprint(const void* data, uint64_t bytes, uint64_t* out) {
  if (out == nullptr || (data == nullptr && bytes != 0))
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  const unsigned char* b = static_cast<const unsigned char*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < bytes; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  *out = h;
  return DD_OK;
}

// Host-buffer drop-in for dedisperse_reference_into / dedisperse_tiled_into.
dd_status dd_dedisperse(dd_context* c, const float* h_in, uint32_t channels, uint64_t num_samples,
                        const uint32_t* h_shifts, uint32_t num_dms, uint32_t s,
                        const dd_config* k, const dd_limits* limits, float* h_out) {
  if (c == nullptr || h_in == nullptr || h_shifts == nullptr || h_out == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "delay table holds no trials");
  if (channels == 0 || s == 0) return fail(DD_ERR_INVALID_ARGUMENT, "empty setup");
  const uint64_t entries = static_cast<uint64_t>(num_dms) * channels;
  // the table is compared with the cached copy first (a survey or a tuner
  // calls with the same table) and its max delay reused; large tables are
  // compared / scanned by the host pool
  if (entries >= (1ull << 20)) DD_TRY(bounce_ready(c));
  const unsigned parts = entries >= (1ull << 20) ? c->pool->size() : 1u;
  const uint64_t per = (entries + parts - 1) / parts;
  const bool same_table = [&] {
    if (c->cached_table.size() != entries) return false;
    std::vector<char> eq(parts, 1);
    auto cmp = [&](unsigned i) {
      const uint64_t lo = std::min(entries, per * i), hi = std::min(entries, lo + per);
      eq[i] = std::memcmp(c->cached_table.data() + lo, h_shifts + lo, (hi - lo) * 4) == 0;
    };
    if (parts > 1) c->pool->run(parts, cmp);
    else cmp(0);
    return std::all_of(eq.begin(), eq.end(), [](char e) { return e != 0; });
  }();
  uint32_t md = 0;
  if (same_table) {
    md = c->cached_max_delay;
  } else {
    std::vector<uint32_t> mx(parts, 0);
    auto scan = [&](unsigned i) {
      const uint64_t lo = std::min(entries, per * i), hi = std::min(entries, lo + per);
      uint32_t m = 0;
      for (uint64_t j = lo; j < hi; ++j) m = std::max(m, h_shifts[j]);
      mx[i] = m;
    };
    if (parts > 1) c->pool->run(parts, scan);
    else scan(0);
    md = *std::max_element(mx.begin(), mx.end());
  }
  const uint64_t needed = static_cast<uint64_t>(s) + md;
  if (num_samples < needed)
    return fail(DD_ERR_INVALID_ARGUMENT, "filterbank too short: need " + std::to_string(needed) +
                                             " samples per channel, have " +
                                             std::to_string(num_samples));
  if (k != nullptr) DD_TRY(dd_validate_config(k, num_dms, s, limits));
  DD_CUDA(cudaSetDevice(c->device));
  const uint64_t pitch = (num_samples + 3) & ~3ull;
  const uint64_t in_bytes = pitch * channels * 4, sh_bytes = entries * 4;
  const uint64_t out_bytes = static_cast<uint64_t>(num_dms) * s * 4;
  // device buffers kept on the context across calls (grown when needed; a
  // new table buffer invalidates the cached plan, which points into it)
  auto grow = [&](void** buf, uint64_t* cap, uint64_t need) -> dd_status {
    if (*cap >= need) return DD_OK;
    DD_CUDA(cudaStreamSynchronize(c->stream));
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    DD_TRY(dd_device_malloc(c, need, buf));
    *cap = need;
    return DD_OK;
  };
  const void* old_sh = c->d_sh;
  DD_TRY(grow(&c->d_in, &c->in_cap, in_bytes));
  DD_TRY(grow(&c->d_sh, &c->sh_cap, sh_bytes));
  DD_TRY(grow(&c->d_out, &c->out_cap, out_bytes));
  // the plan (pre-pass, shared-memory sizing) is reused while the table and
  // the request repeat -- a tuner or a survey calls with the same table
  const uint64_t key[8] = {channels, num_samples, num_dms, s,
                           k ? (uint64_t{k->items_time} << 32 | k->items_dm) : ~0ull,
                           k ? (uint64_t{k->work_time} << 32 | k->work_dm) : ~0ull,
                           k ? (uint64_t{k->dm_tile_depth} << 32 | k->staging) : ~0ull,
                           (k ? uint64_t{k->flags} : ~0ull) ^
                               (limits ? (uint64_t{limits->max_block_items} << 32 |
                                          limits->max_accumulators) << 8
                                       : 0)};
  const bool same = c->cached_plan != nullptr && old_sh == c->d_sh &&
                    std::memcmp(key, c->cached_key, sizeof(key)) == 0 && same_table;
  if (!same) {
    dd_plan_destroy(c->cached_plan);
    c->cached_plan = nullptr;
    c->cached_table.clear();
    DD_TRY(dd_copy_h2d(c, c->d_sh, h_shifts, sh_bytes));
    dd_config ran{};
    DD_TRY(plan_one_shot(c, static_cast<uint32_t*>(c->d_sh), channels, num_dms, s, num_samples,
                         pitch, k, limits, &c->cached_plan, &ran));
    c->cached_table.assign(h_shifts, h_shifts + entries);
    c->cached_max_delay = md;
    std::memcpy(c->cached_key, key, sizeof(key));
    c->last_run = ran;
    c->last_family = c->cached_plan->family;
  }
  // pageable host buffers: pinned bounce buffers and parallel host copies
  // (the reference API's std::vectors), or direct async copies from pinned
  // memory
  cudaPointerAttributes pin_in{}, pin_out{};
  const bool in_pinned = cudaPointerGetAttributes(&pin_in, h_in) == cudaSuccess &&
                         pin_in.type == cudaMemoryTypeHost;
  const bool out_pinned = cudaPointerGetAttributes(&pin_out, h_out) == cudaSuccess &&
                          pin_out.type == cudaMemoryTypeHost;
  cudaGetLastError();  // a pageable pointer is not an error
  if (in_pinned)
    DD_TRY(dd_upload_filterbank(c, static_cast<float*>(c->d_in), pitch, h_in, channels,
                                num_samples));
  else
    DD_TRY(upload_staged(c, static_cast<float*>(c->d_in), pitch, h_in, channels, num_samples));
  DD_TRY(dd_plan_execute(c->cached_plan, static_cast<float*>(c->d_in),
                         static_cast<float*>(c->d_out), s));
  if (out_pinned) {
    DD_TRY(dd_copy_d2h(c, h_out, c->d_out, out_bytes));
    DD_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    DD_TRY(download_staged(c, h_out, c->d_out, out_bytes));
  }
  return DD_OK;
}

}  // extern "C"
