// Microbenchmark: TMEM -> register bandwidth of tcgen05.ld.32x32b at
// warp-uniform DYNAMIC column offsets (the register-window access pattern),
// vs shared-memory LDS.32 at lane-contiguous addresses.  One CTA per SM,
// 4..16 warps; prints bytes/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define X16 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}"

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(512, 1) k_tmem(float* out, int iters, long long* cyc) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
  // fill: each warp writes 16 columns x its 32 lanes at col (warp/4)*16.. (disjoint per warp)
  {
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint((float)(threadIdx.x + i));
    for (int c = 0; c < 480; c += 16)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], " X16 ";" ::"r"(base + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)((it * 7 + warp * 3) & 255);
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 " X16 ", [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(base + col));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) acc[i] += __uint_as_float(r[i]);
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

__global__ void __launch_bounds__(512, 1) k_lds(float* out, int iters, long long* cyc) {
  __shared__ float buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int off = ((it * 7 + warp * 3) & 255) + lane;
    const float* p = buf + off;
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] += p[i * 32];
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int which = 0; which < 2; ++which) {
      if (which == 0) k_tmem<<<sms, warps * 32>>>(out, iters, cyc);
      else k_lds<<<sms, warps * 32>>>(out, iters, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * iters * 32 * 16 * 4;
      printf("%-5s warps=%2d: %8.1f bytes/clk/SM (%lld cycles, %.2f clk per 16-col warp load)\n",
             which == 0 ? "tmem" : "lds", warps, bytes / c, c, (double)c / iters);
    }
  }
  return 0;
}
