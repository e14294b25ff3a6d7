// Microbenchmark: L2 -> shared-memory throughput of 1-D bulk copies
// (cp.async.bulk, the staging path of the dedispersion kernels).  Every CTA
// streams `chunk`-byte copies from a global buffer small enough to stay in
// L2 (or large enough to come from HBM) into a ring of shared-memory slots
// guarded by mbarriers; prints GB/s for the whole GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/bulk_l2.bin tools/ubench/bulk_l2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32) k_bulk(const uint8_t* src, uint64_t src_bytes, uint32_t chunk,
                                           uint32_t slots, uint32_t iters, uint64_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  uint8_t* buf = smem + 128;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < slots; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint64_t off = (static_cast<uint64_t>(blockIdx.x) * 7919u * chunk) % src_bytes;
  for (uint32_t i = 0; i < iters; ++i) {
    const uint32_t s = i % slots;
    if (i >= slots) {  // wait for the copy that last used this slot
      const uint32_t parity = ((i / slots) - 1) & 1u;
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar[s])), "r"(parity));
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(chunk));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(buf + static_cast<uint64_t>(s) * chunk)),
        "l"(src + off), "r"(chunk), "r"(smem_u32(&bar[s])));
    off += chunk;
    if (off + chunk > src_bytes) off = 0;
  }
  for (uint32_t i = iters; i < iters + slots; ++i) {  // drain
    const uint32_t s = i % slots;
    const uint32_t parity = ((i / slots) - 1) & 1u;
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar[s])), "r"(parity));
  }
  sink[blockIdx.x] = buf[threadIdx.x];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t big = 2ull << 30;
  uint8_t* src;
  uint64_t* sink;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  cudaMalloc(&sink, 8 * 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t footprints[] = {32ull << 20, 96ull << 20, big};
  for (uint64_t footprint : footprints) {
    for (uint32_t chunk : {4096u, 8192u, 16384u}) {
      for (uint32_t ctas_per_sm : {2u, 4u}) {
        const uint32_t slots = 4;
        const uint32_t smem = 128 + slots * chunk;
        cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const uint32_t iters = 2000;
        const uint32_t grid = sms * ctas_per_sm;
        k_bulk<<<grid, 32, smem>>>(src, footprint, chunk, slots, 50, sink);
        cudaEventRecord(a);
        k_bulk<<<grid, 32, smem>>>(src, footprint, chunk, slots, iters, sink);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(grid) * iters * chunk;
        printf("footprint %5llu MB chunk %5u B  %u CTAs/SM: %8.1f GB/s\n",
               static_cast<unsigned long long>(footprint >> 20), chunk, ctas_per_sm,
               bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
