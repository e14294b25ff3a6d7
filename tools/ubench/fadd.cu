// Microbenchmark: FP32 add throughput per SM on this B200 -- the binding
// on-chip ceiling of the dedispersion kernels (one IEEE RN add per
// (output, channel)).  Measures scalar FADD (add.rn.f32) and paired FADD2
// (add.rn.f32x2) with many independent accumulator chains per thread and
// 8..32 warps per SM, one CTA per SM, timed with clock64 inside the kernel
// (per-SM cycles: clock-rate independent) and with CUDA events (wall, for
// the adds/s figure at the clock the GPU actually ran).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fadd tools/ubench/fadd.cu
// Prints one JSON line per variant plus a summary line with the peak.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(1024, 1) k_fadd(float* out, int iters, long long* cyc,
                                                  float step) {
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(step));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH>
__global__ void __launch_bounds__(1024, 1) k_fadd2(float* out, int iters, long long* cyc,
                                                   float step) {
  // CH independent float2 chains: 2*CH adds per iteration per thread
  unsigned long long acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const float x = threadIdx.x * 1e-3f + c, y = x + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc[c]) : "f"(x), "f"(y));
  }
  unsigned long long st;
  asm("mov.b64 %0, {%1, %1};" : "=l"(st) : "f"(step));
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc[c]) : "l"(st));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[c]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

struct Result {
  double adds_per_clk_sm, adds_per_s, ms, mhz_eff;
};

template <class F>
Result run(F kern, int adds_per_iter_thread, int sms, int threads, int iters) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  kern<<<sms, threads>>>(out, 64, cyc, 1e-7f);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<sms, threads>>>(out, iters, cyc, 1e-7f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  long long* h = new long long[sms];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mean_cyc = 0.0;
  for (int i = 0; i < sms; ++i) mean_cyc += static_cast<double>(h[i]);
  mean_cyc /= sms;
  delete[] h;
  const double adds_per_sm = static_cast<double>(adds_per_iter_thread) * iters * threads;
  Result r;
  r.adds_per_clk_sm = adds_per_sm / mean_cyc;
  r.adds_per_s = adds_per_sm * sms / (ms * 1e-3);
  r.ms = ms;
  r.mhz_eff = mean_cyc / (ms * 1e-3) / 1e6;
  cudaFree(out);
  cudaFree(cyc);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return r;
}

int main() {
  cudaDeviceProp p{};
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int iters = 1 << 16;
  double best1 = 0, best2 = 0, best1_s = 0, best2_s = 0;
  for (int threads : {256, 512, 1024}) {
    {
      Result r = run(k_fadd<8>, 8, sms, threads, iters);
      printf("{\"op\": \"FADD\", \"chains\": 8, \"warps_per_sm\": %d, \"adds_per_clk_sm\": %.2f, "
             "\"tadds_per_s\": %.3f, \"ms\": %.3f, \"clk_mhz_effective\": %.0f}\n",
             threads / 32, r.adds_per_clk_sm, r.adds_per_s / 1e12, r.ms, r.mhz_eff);
      if (r.adds_per_clk_sm > best1) best1 = r.adds_per_clk_sm, best1_s = r.adds_per_s;
    }
    {
      Result r = run(k_fadd2<8>, 16, sms, threads, iters);
      printf("{\"op\": \"FADD2\", \"chains\": 8, \"warps_per_sm\": %d, \"adds_per_clk_sm\": %.2f, "
             "\"tadds_per_s\": %.3f, \"ms\": %.3f, \"clk_mhz_effective\": %.0f}\n",
             threads / 32, r.adds_per_clk_sm, r.adds_per_s / 1e12, r.ms, r.mhz_eff);
      if (r.adds_per_clk_sm > best2) best2 = r.adds_per_clk_sm, best2_s = r.adds_per_s;
    }
  }
  printf("{\"summary\": true, \"gpu\": \"%s\", \"sm_count\": %d, \"max_clock_mhz\": %d, "
         "\"fadd_adds_per_clk_sm\": %.2f, \"fadd2_adds_per_clk_sm\": %.2f, "
         "\"fadd_tadds_per_s\": %.3f, \"fadd2_tadds_per_s\": %.3f}\n",
         p.name, sms, clk_khz / 1000, best1, best2, best1_s / 1e12, best2_s / 1e12);
  return 0;
}
