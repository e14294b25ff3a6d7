// Microbenchmark: tcgen05.ld.32x32b.xN throughput vs N (4, 8, 16, 32) and
// loads in flight per warp (1, 2, 4), at warp-uniform dynamic columns.
// One CTA per SM, 4..16 warps; prints bytes/clk/SM and clk per load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_ld2 tools/ubench/tmem_ld2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int N>
__device__ __forceinline__ void ld(uint32_t a, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void ld<4>(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
template <>
__device__ __forceinline__ void ld<8>(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(a));
}
template <>
__device__ __forceinline__ void ld<16>(uint32_t a, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(a));
}

template <int N, int F>
__global__ void __launch_bounds__(512, 1) k_tmem(float* out, int iters, long long* cyc) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
  float acc[F][N];
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int i = 0; i < N; ++i) acc[f][i] = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it += F) {
    uint32_t r[F][N];
#pragma unroll
    for (int f = 0; f < F; ++f) ld<N>(base + (uint32_t)(((it + f) * 7 + warp * 3) & 255), r[f]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int i = 0; i < N; ++i) acc[f][i] += __uint_as_float(r[f][i]);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int i = 0; i < N; ++i) s += acc[f][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int N, int F>
void run(int sms, float* out, long long* cyc) {
  const int iters = 4096;
  for (int warps : {4, 8, 12, 16}) {
    k_tmem<N, F><<<sms, warps * 32>>>(out, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * iters * 32 * N * 4;
    printf("x%-2d inflight=%d warps=%2d: %7.1f B/clk/SM  %6.2f clk/load/SMSP\n", N, F, warps,
           bytes / c, (double)c / (iters * warps / 4.0));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<4, 1>(sms, out, cyc);
  run<4, 2>(sms, out, cyc);
  run<4, 4>(sms, out, cyc);
  run<8, 1>(sms, out, cyc);
  run<8, 2>(sms, out, cyc);
  run<8, 4>(sms, out, cyc);
  run<16, 1>(sms, out, cyc);
  run<16, 2>(sms, out, cyc);
  return 0;
}
