// stream.cu -- streaming block ingest through the C-ABI (
// the Python mirror is paper_1601_05052_b200/stream.py).
//
// The reference dedisperses one padded block (setup.cpp:130-133): output
// second n needs input samples [n*s, (n+1)*s + max_delay).  A block stream
// keeps, per channel, a ring row of t + R*s samples on the device (t =
// instance_sizing's num_samples, R = ceil(t/s)); each push appends one
// second behind the window, the window start advances by s and the plan
// runs on the window through an offset pointer; only when the row is used
// up is the window's tail moved to the front, once every R pushes, between
// non-overlapping ranges.  Every output equals a one-shot pass over the same
// samples bit for bit (same plan, same data, same order).
#include <algorithm>
#include <string>

#include "internal.hpp"

using namespace ddb;

struct dd_block_stream {
  dd_context* ctx = nullptr;
  dd_plan* plan = nullptr;
  uint32_t channels = 0, s = 0, num_dms = 0;
  uint64_t t = 0, pitch = 0;
  uint64_t start = 0, filled = 0;
  uint64_t pushes = 0, outputs = 0, compactions = 0;
  bool ring = true;  // s % 4 == 0: the window start stays 16-byte aligned
  float* d_ring = nullptr;
  float* d_tmp = nullptr;  // compaction through a temporary when !ring
  uint32_t* d_shifts = nullptr;
  float* d_out = nullptr;
};

namespace {
void release(dd_block_stream* b) {
  if (b == nullptr) return;
  if (b->ctx) cudaSetDevice(b->ctx->device);
  dd_plan_destroy(b->plan);
  cudaFree(b->d_ring);
  cudaFree(b->d_tmp);
  cudaFree(b->d_shifts);
  cudaFree(b->d_out);
  delete b;
}
}  // namespace

extern "C" {

dd_status dd_block_stream_create(dd_context* c, const dd_setup* setup, uint32_t num_dms,
                                 const dd_config* cfg, dd_block_stream** out) {
  if (c == nullptr || out == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  std::string why;
  if (!setup_ok(setup, &why)) return fail(DD_ERR_INVALID_ARGUMENT, why);
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "need at least one trial DM");
  uint64_t t = 0;
  uint32_t md = 0;
  {
    const dd_status st = dd_instance_sizing(setup, num_dms, &t, nullptr, &md);
    if (st != DD_OK) return st;
  }
  auto* b = new dd_block_stream;
  b->ctx = c;
  b->channels = setup->channels;
  b->s = setup->samples_per_second;
  b->num_dms = num_dms;
  b->t = t;
  b->ring = b->s % 4 == 0;
  const uint64_t rounds = b->ring ? (t + b->s - 1) / b->s : 0;
  b->pitch = (t + rounds * b->s + 3) & ~3ull;
  cudaError_t e = cudaSetDevice(c->device);
  if (e == cudaSuccess)
    e = cudaMalloc(&b->d_ring, b->pitch * b->channels * sizeof(float));
  if (e == cudaSuccess && !b->ring)
    e = cudaMalloc(&b->d_tmp, b->pitch * b->channels * sizeof(float));
  if (e == cudaSuccess)
    e = cudaMalloc(&b->d_shifts, static_cast<uint64_t>(num_dms) * b->channels * sizeof(uint32_t));
  if (e == cudaSuccess)
    e = cudaMalloc(&b->d_out, static_cast<uint64_t>(num_dms) * b->s * sizeof(float));
  if (e == cudaSuccess)
    e = cudaMemsetAsync(b->d_ring, 0, b->pitch * b->channels * sizeof(float), c->stream);
  if (e != cudaSuccess) {
    release(b);
    return cuda_fail(e, "dd_block_stream_create");
  }
  dd_status st = dd_delay_table_device(c, setup, num_dms, 0, 0, b->d_shifts, nullptr);
  // cfg == NULL or an AUTO flag-free config: the instance's tuned schedule
  // (the same choice as the one-shot entry points), else the config itself
  dd_config run{};
  bool have = false;
  if (cfg == nullptr || (cfg->staging == DD_STAGING_AUTO && cfg->flags == 0)) {
    int builtin = 0;
    have = dd_schedule_get(b->channels, b->s, num_dms, &run, &builtin) == DD_OK;
    clear_error();
  }
  if (st == DD_OK && have) {
    st = dd_plan_create(c, b->d_shifts, b->channels, num_dms, b->s, t, b->pitch, &run, nullptr,
                        &b->plan);
    if (st == DD_ERR_INVALID_ARGUMENT) {
      clear_error();
      st = DD_OK;
      b->plan = nullptr;
    }
  }
  if (st == DD_OK && b->plan == nullptr) {
    // no schedule for this instance: a shared-memory staged shape whose DM
    // tile divides the trial count (predicated last time tile)
    uint32_t k = 8;
    while (num_dms % k != 0) k >>= 1;
    dd_config fallback{32, 1, 1, k, 1, DD_STAGING_SMEM, DD_CONFIG_GPU_TILING};
    st = dd_plan_create(c, b->d_shifts, b->channels, num_dms, b->s, t, b->pitch,
                        cfg ? cfg : &fallback, nullptr, &b->plan);
  }
  if (st != DD_OK) {
    release(b);
    return st;
  }
  *out = b;
  return DD_OK;
}

dd_status dd_block_stream_push(dd_block_stream* b, const float* h_second, float* h_out,
                               int* produced) {
  if (b == nullptr || h_second == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (produced) *produced = 0;
  dd_context* c = b->ctx;
  cudaStream_t st = c->stream;
  if (cudaSetDevice(c->device) != cudaSuccess) return fail(DD_ERR_CUDA, "cudaSetDevice");
  const uint64_t row = b->pitch * sizeof(float);
  if (b->filled == b->t) {  // slide: drop the oldest second
    b->start += b->s;
    b->filled -= b->s;
    if (!b->ring) {
      cudaError_t e = cudaMemcpy2DAsync(b->d_tmp, row, b->d_ring + b->start, row,
                                        b->filled * sizeof(float), b->channels,
                                        cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(b->d_ring, row, b->d_tmp, row, b->filled * sizeof(float),
                              b->channels, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return cuda_fail(e, "block stream compaction");
      b->start = 0;
      ++b->compactions;
    }
  }
  if (b->start + b->filled + b->s > b->pitch) {
    // the row is used up: move the window's tail to the front (no overlap:
    // start >= R*s >= t - s = filled)
    const cudaError_t e = cudaMemcpy2DAsync(b->d_ring, row, b->d_ring + b->start, row,
                                            b->filled * sizeof(float), b->channels,
                                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "block stream compaction");
    b->start = 0;
    ++b->compactions;
  }
  const uint64_t end = b->start + b->filled;
  cudaError_t e = cudaMemcpy2DAsync(b->d_ring + end, row, h_second, b->s * sizeof(float),
                                    b->s * sizeof(float), b->channels, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "block stream upload");
  b->filled += b->s;
  ++b->pushes;
  if (b->filled < b->t) return DD_OK;
  const dd_status ds = dd_plan_execute(b->plan, b->d_ring + b->start, b->d_out, b->s);
  if (ds != DD_OK) return ds;
  ++b->outputs;
  if (h_out != nullptr) {
    e = cudaMemcpyAsync(h_out, b->d_out, static_cast<uint64_t>(b->num_dms) * b->s * sizeof(float),
                        cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "block stream download");
  }
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "dd_block_stream_push");
  if (produced) *produced = 1;
  return DD_OK;
}

dd_status dd_block_stream_info(const dd_block_stream* b, uint64_t* num_samples,
                               uint64_t* pushes, uint64_t* outputs, uint64_t* compactions,
                               const float** d_out) {
  if (b == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (num_samples) *num_samples = b->t;
  if (pushes) *pushes = b->pushes;
  if (outputs) *outputs = b->outputs;
  if (compactions) *compactions = b->compactions;
  if (d_out) *d_out = b->d_out;
  return DD_OK;
}

dd_status dd_block_stream_destroy(dd_block_stream* b) {
  if (b == nullptr) return DD_OK;
  cudaSetDevice(b->ctx->device);
  cudaStreamSynchronize(b->ctx->stream);
  release(b);
  return DD_OK;
}

}  // extern "C"
