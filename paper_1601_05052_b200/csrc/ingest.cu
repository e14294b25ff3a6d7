// ingest.cu -- on-device SIGPROC payload ingest.
//
// A SIGPROC filterbank payload is time-major with channel 0 at the HIGHEST
// frequency; the dedispersion layout is channel-major with channel 0 at the
// LOWEST (reference sigproc.cpp:177-189 does this transpose + reversal on
// the host, sample by sample, rejecting non-finite samples with a
// format_error carrying the byte offset).  Here the payload is copied to the
// device as-is and transposed by 32x32 shared-memory tiles (coalesced reads
// along channels, coalesced writes along time); the first non-finite
// sample's payload index is reported through an atomicMin.
#include <cstdint>

#include "internal.hpp"

namespace ddb {

__global__ void __launch_bounds__(256) k_sigproc_transpose(const float* __restrict__ src,
                                                           uint32_t channels, uint64_t samples,
                                                           float* __restrict__ dst,
                                                           uint64_t dst_pitch,
                                                           unsigned long long* first_bad) {
  __shared__ float tile[32][33];
  const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * 32;  // time
  const uint32_t k0 = blockIdx.y * 32;                         // payload channel
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  unsigned long long bad = ~0ull;
  for (uint32_t r = ty; r < 32; r += 8) {
    const uint64_t j = j0 + r;
    const uint32_t k = k0 + tx;
    float v = 0.0f;
    if (j < samples && k < channels) {
      const uint64_t idx = j * channels + k;
      v = src[idx];
      if (!isfinite(v)) bad = min(bad, static_cast<unsigned long long>(idx));
    }
    tile[r][tx] = v;
  }
  if (bad != ~0ull) atomicMin(first_bad, bad);
  __syncthreads();
  for (uint32_t r = ty; r < 32; r += 8) {
    const uint32_t k = k0 + r;
    const uint64_t j = j0 + tx;
    if (k < channels && j < samples) dst[static_cast<uint64_t>(channels - 1 - k) * dst_pitch + j] = tile[tx][r];
  }
}

}  // namespace ddb

using namespace ddb;

extern "C" dd_status dd_sigproc_to_filterbank(dd_context* c, const float* d_payload,
                                              uint32_t channels, uint64_t num_samples,
                                              float* d_dst, uint64_t dst_pitch,
                                              int64_t* first_bad) {
  if (c == nullptr || d_payload == nullptr || d_dst == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (channels == 0 || num_samples == 0 || dst_pitch < num_samples)
    return fail(DD_ERR_INVALID_ARGUMENT, "bad payload shape");
  cudaError_t e = cudaSetDevice(c->device);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_scratch, 0xff, 8, c->stream);
  if (e != cudaSuccess) return cuda_fail(e, "dd_sigproc_to_filterbank");
  const uint64_t bx = (num_samples + 31) / 32;
  const uint32_t by = (channels + 31) / 32;
  if (bx > 0x7fffffffULL || by > 65535) return fail(DD_ERR_CAPACITY, "payload too large");
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(c->d_scratch);
  k_sigproc_transpose<<<dim3(static_cast<uint32_t>(bx), by), 256, 0, c->stream>>>(
      d_payload, channels, num_samples, d_dst, dst_pitch, bad);
  e = cudaGetLastError();
  unsigned long long h = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(e, "dd_sigproc_to_filterbank");
  if (first_bad) *first_bad = h == ~0ull ? -1 : static_cast<int64_t>(h);
  return DD_OK;
}

extern "C" dd_status dd_upload_block_range(dd_context* c, const float* h_block, uint64_t h_pitch,
                                           float* d_block, uint64_t d_pitch, uint32_t channels,
                                           uint64_t t0, uint64_t t1, void* stream) {
  if (c == nullptr || h_block == nullptr || d_block == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  if (t1 < t0 || t1 > h_pitch || t1 > d_pitch)
    return fail(DD_ERR_INVALID_ARGUMENT, "sample range outside the block");
  if (t1 == t0 || channels == 0) return DD_OK;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  const cudaError_t e = cudaMemcpy2DAsync(d_block + t0, d_pitch * 4, h_block + t0, h_pitch * 4,
                                          (t1 - t0) * 4, channels, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "dd_upload_block_range");
  return DD_OK;
}
