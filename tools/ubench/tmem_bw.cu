// Microbenchmark: tcgen05.ld.32x32b.xN (TMEM -> registers) throughput with
// the loaded values barely consumed (one add per load: the TMEM datapath
// alone) and fully consumed by FADD2 (N/2 paired adds per load: the
// dedispersion inner loop's mix), N = 4..64, 1..4 loads in flight per wait,
// 4..16 warps per SM, one CTA per SM, warp-uniform dynamic columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/tmem_bw.bin tools/ubench/tmem_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int N>
struct Ld;
#define LD_ASM(N, LIST, ...)                                                                    \
  template <>                                                                                   \
  struct Ld<N> {                                                                                \
    static __device__ __forceinline__ void go(uint32_t a, uint32_t (&r)[N]) {                  \
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x" #N ".b32 {" LIST "}, [%" #N "];"       \
                   : __VA_ARGS__                                                                \
                   : "r"(a));                                                                   \
    }                                                                                           \
  };
LD_ASM(4, "%0,%1,%2,%3", "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]))
LD_ASM(8, "%0,%1,%2,%3,%4,%5,%6,%7", "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
       "=r"(r[5]), "=r"(r[6]), "=r"(r[7]))
LD_ASM(16, "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15", "=r"(r[0]), "=r"(r[1]),
       "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
       "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]))
LD_ASM(32,
       "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"
       "%24,%25,%26,%27,%28,%29,%30,%31",
       "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
       "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
       "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
       "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
       "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]))

__device__ __forceinline__ void fadd2(float& a, float& b, uint32_t x, uint32_t y) {
  asm volatile(
      "{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
      "add.rn.f32x2 ra, ra, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a), "+f"(b)
      : "r"(x), "r"(y));
}

// FULL = false: one add per load (TMEM path alone); true: every value added.
template <int N, int F, bool FULL>
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
  float acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; it += F) {
    uint32_t r[F][N];
#pragma unroll
    for (int f = 0; f < F; ++f)
      Ld<N>::go(base + (uint32_t)(((it + f) * 7 + warp * 3) & 255), r[f]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int f = 0; f < F; ++f) {
      if constexpr (FULL) {
#pragma unroll
        for (int i = 0; i < N; i += 2) fadd2(acc[i], acc[i + 1], r[f][i], r[f][i + 1]);
      } else {
        acc[f % N] += __uint_as_float(r[f][0] ^ r[f][N - 1]);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int N, int F, bool FULL>
void run(int sms, float* out, long long* cyc) {
  const int iters = 2048;
  for (int warps : {4, 8, 16}) {
    k_tmem<N, F, FULL><<<sms, warps * 32>>>(out, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * iters * 32 * N * 4;
    printf("{\"n\": %d, \"inflight\": %d, \"consume\": \"%s\", \"warps\": %d, \"bytes_per_clk_sm\": %.1f, "
           "\"clk_per_ld_sm\": %.2f}\n",
           N, F, FULL ? "fadd2-all" : "one-add", warps, bytes / c, (double)c / (iters * (double)warps));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  run<4, 4, false>(sms, out, cyc);
  run<8, 4, false>(sms, out, cyc);
  run<16, 4, false>(sms, out, cyc);
  run<32, 2, false>(sms, out, cyc);
  run<8, 4, true>(sms, out, cyc);
  run<16, 2, true>(sms, out, cyc);
  run<32, 2, true>(sms, out, cyc);
  return 0;
}
