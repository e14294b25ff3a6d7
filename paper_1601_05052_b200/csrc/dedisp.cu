// dedisp.cu -- the dedispersion kernels (K2 reference-order, K2' direct
// tiled, K3 TMA-staged tiled) for sm_100a.
//
// Arithmetic contract (reference kernels.cpp:83-108): each
// output element owns ONE fp32 accumulator, starts at 0.0f and adds the
// channels in ascending order with IEEE round-to-nearest adds.  Tiling and
// thread mapping change only the schedule, never that sequence, so every
// kernel here is bit-identical to dedisperse_reference.  Build flags must
// not enable fast-math / FTZ (see build.py).
#include "common.cuh"

namespace ddb {

// ---------------------------------------------------------------------
// K2: reference order, one thread per output (dedisperse_reference_into,
// kernels.cpp:91-101).  The first parity target and the cfg == NULL path.
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_reference(const float* __restrict__ in, uint64_t pitch,
                                                   const uint32_t* __restrict__ shifts,
                                                   float* __restrict__ out, uint64_t out_pitch,
                                                   uint32_t channels, uint32_t s,
                                                   uint32_t num_dms) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<uint64_t>(num_dms) * s) return;
  const uint32_t dm = static_cast<uint32_t>(i / s);
  const uint32_t j = static_cast<uint32_t>(i - static_cast<uint64_t>(dm) * s);
  const uint32_t* row = shifts + static_cast<uint64_t>(dm) * channels;
  float acc = 0.0f;
  for (uint32_t ch = 0; ch < channels; ++ch) acc += in[ch * pitch + j + row[ch]];
  out[static_cast<uint64_t>(dm) * out_pitch + j] = acc;
}

// ---------------------------------------------------------------------
// K2': direct tiled kernel for ANY reference-valid config (SURVEY.md §7
// hard part 10).  Honours the reference's tile decomposition and thread
// mapping (kernels.cpp:127-178: item (it, id) owns times t0+it+wt*items_time
// and DMs dm0+id+wd*items_dm), with loads straight from global through
// L1/L2.  Small tiles are packed `pack` to a CTA and oversize blocks
// (items > 1024 under raised limits) run as virtual threads; accumulators
// beyond 16 per item are processed in 16-wide passes over the channels.
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_direct(const TiledArgs a) {
  const uint32_t block_items = a.items_time * a.items_dm;
  const uint32_t nout = a.work_time * a.work_dm;
  const uint64_t tiles = static_cast<uint64_t>(a.tiles_time) * a.tiles_dm;
  for (uint32_t v = threadIdx.x; v < a.vthreads; v += blockDim.x) {
    const uint64_t tile = static_cast<uint64_t>(blockIdx.x) * a.pack + v / block_items;
    if (tile >= tiles) break;
    const uint32_t item = v % block_items;
    const uint32_t it = item % a.items_time, id = item / a.items_time;
    const uint32_t dm0 = static_cast<uint32_t>(tile / a.tiles_time) * a.tile_dm;
    const uint32_t t0 = static_cast<uint32_t>(tile % a.tiles_time) * a.tile_time;
    for (uint32_t o0 = 0; o0 < nout; o0 += 16) {
      float acc[16];
      uint32_t t[16];
      const uint32_t* row[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        acc[u] = 0.0f;
        const uint32_t o = min(o0 + u, nout - 1);
        const uint32_t wd = o / a.work_time, wt = o % a.work_time;
        t[u] = t0 + wt * a.items_time + it;
        row[u] = a.shifts + static_cast<uint64_t>(dm0 + wd * a.items_dm + id) * a.channels;
      }
      for (uint32_t ch = 0; ch < a.channels; ++ch) {
        const float* src = a.in + ch * a.in_pitch;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (o0 + u < nout) acc[u] += src[t[u] + row[u][ch]];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (o0 + u < nout) {
          const uint32_t o = o0 + u;
          const uint32_t wd = o / a.work_time;
          a.out[static_cast<uint64_t>(dm0 + wd * a.items_dm + id) * a.out_pitch + t[u]] = acc[u];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------
// K3: TMA-staged tiled kernel (the paper's data-reuse lever, §3.2).
//
// CTA = tile_dm x tile_time outputs (x depth DM tiles walked in sequence).
// Per channel the contiguous window [t0+lo, t0+hi+tile_time) that the
// tile's shifts span is copied once into shared memory by a 1-D bulk copy
// (cp.async.bulk -> UBLKCP) and then read by every DM of the tile.  Channels
// are grouped `cps` per pipeline stage; `nstage` stages are in flight, each
// guarded by an mbarrier whose transaction count is the stage's bytes.
// Thread (it, id) keeps its work_dm x work_time accumulators in registers
// with the reference mapping (times it + j*items_time, DMs id + k*items_dm),
// so a warp's 32 lanes read 32 consecutive floats: one conflict-free
// shared-memory wavefront per warp-load.  Outputs are written coalesced.
// ---------------------------------------------------------------------
// Register budget: K*W accumulators + ~24 bookkeeping registers, so the
// thread cap per variant is what keeps the accumulators out of local memory.
template <int K, int W>
constexpr int smem_max_threads() {
  return K * W > 32 ? 256 : (K * W > 16 ? 512 : 1024);
}

template <int K, int W>
__global__ void __launch_bounds__(smem_max_threads<K, W>()) k_smem(const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint8_t* recs = smem + 128;
  float* wins = reinterpret_cast<float*>(recs + a.nstage * a.cps * a.rec_bytes);

  const uint32_t tid = threadIdx.x;
  const uint32_t it = tid % a.items_time, id = tid / a.items_time;
  const uint32_t groups_dm = (a.tiles_dm + a.depth - 1) / a.depth;
  const uint32_t gy = blockIdx.x % groups_dm;  // DM-fastest raster: neighbours share input
  const uint32_t t0 = (blockIdx.x / groups_dm) * a.tile_time;
  const uint32_t b_first = gy * a.depth;
  const uint32_t ntiles = min(a.depth, a.tiles_dm - b_first);
  const uint32_t nchunk = (a.channels + a.cps - 1) / a.cps;
  const uint32_t total = ntiles * nchunk;

  if (tid == 0) {
    for (uint32_t s = 0; s < a.nstage; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();

  // Producer (one thread): stage chunk g = (tile, channel group) into slot.
  auto issue = [&](uint32_t g) {
    const uint32_t b = b_first + g / nchunk;
    const uint32_t ch0 = (g % nchunk) * a.cps;
    const uint32_t ncs = min(a.cps, a.channels - ch0);
    const uint32_t slot = g % a.nstage;
    const uint8_t* rsrc = a.rec + (static_cast<uint64_t>(b) * a.channels + ch0) * a.rec_bytes;
    uint32_t bytes = ncs * a.rec_bytes;
    for (uint32_t cc = 0; cc < ncs; ++cc) {
      const uint32_t* r = reinterpret_cast<const uint32_t*>(rsrc + cc * a.rec_bytes);
      const uint32_t lo = __ldg(r), span = __ldg(r + 1);
      const uint32_t start = (t0 + lo) & ~3u;
      const uint32_t end = (t0 + lo + span + a.tile_time + 3u) & ~3u;
      bytes += (end - start) * 4u;
    }
    mbar_arrive_expect_tx(&full[slot], bytes);
    bulk_g2s(recs + slot * a.cps * a.rec_bytes, rsrc, ncs * a.rec_bytes, &full[slot]);
    for (uint32_t cc = 0; cc < ncs; ++cc) {
      const uint32_t* r = reinterpret_cast<const uint32_t*>(rsrc + cc * a.rec_bytes);
      const uint32_t lo = __ldg(r), span = __ldg(r + 1);
      const uint32_t start = (t0 + lo) & ~3u;
      const uint32_t end = (t0 + lo + span + a.tile_time + 3u) & ~3u;
      bulk_g2s(wins + static_cast<uint64_t>(slot * a.cps + cc) * a.win_cap,
               a.in + static_cast<uint64_t>(ch0 + cc) * a.in_pitch + start, (end - start) * 4u,
               &full[slot]);
    }
  };
  if (tid == 0) {
    const uint32_t pre = min(a.nstage, total);
    for (uint32_t g = 0; g < pre; ++g) issue(g);
  }

  float acc[K][W];
  for (uint32_t g = 0; g < total; ++g) {
    const uint32_t q = g % nchunk;
    if (q == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
    }
    const uint32_t slot = g % a.nstage;
    mbar_wait(&full[slot], (g / a.nstage) & 1u);
    const uint32_t ncs = min(a.cps, a.channels - q * a.cps);
    const uint8_t* rbase = recs + slot * a.cps * a.rec_bytes;
    const float* wbase = wins + static_cast<uint64_t>(slot) * a.cps * a.win_cap;
    for (uint32_t cc = 0; cc < ncs; ++cc) {
      const uint32_t* r = reinterpret_cast<const uint32_t*>(rbase + cc * a.rec_bytes);
      const float* w = wbase + cc * a.win_cap + ((t0 + r[0]) & 3u) + it;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float* p = w + r[4 + id + k * a.items_dm];
#pragma unroll
        for (int j = 0; j < W; ++j) acc[k][j] += p[j * a.items_time];
      }
    }
    if (q == nchunk - 1) {
      const uint32_t dm0 = (b_first + g / nchunk) * a.tile_dm;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        float* o = a.out + static_cast<uint64_t>(dm0 + id + k * a.items_dm) * a.out_pitch + t0 + it;
#pragma unroll
        for (int j = 0; j < W; ++j) o[j * a.items_time] = acc[k][j];
      }
    }
    __syncthreads();  // every warp is done with `slot` before it is refilled
    if (tid == 0 && g + a.nstage < total) issue(g + a.nstage);
  }
}

// ------------------------------------------------------------ dispatch --
using KernelFn = void (*)(const TiledArgs);

struct SmemVariant {
  int k, w;
  KernelFn fn;
  int max_threads;
};

#define DDB_V(K, W) {K, W, k_smem<K, W>, smem_max_threads<K, W>()}
static const SmemVariant kSmemVariants[] = {
    DDB_V(1, 1),  DDB_V(1, 2),  DDB_V(1, 4),  DDB_V(1, 5),  DDB_V(1, 8),  DDB_V(1, 10),
    DDB_V(1, 16), DDB_V(1, 25), DDB_V(2, 1),  DDB_V(2, 2),  DDB_V(2, 4),  DDB_V(2, 5),
    DDB_V(2, 8),  DDB_V(2, 10), DDB_V(2, 16), DDB_V(2, 25), DDB_V(4, 1),  DDB_V(4, 2),
    DDB_V(4, 4),  DDB_V(4, 5),  DDB_V(4, 8),  DDB_V(4, 10), DDB_V(4, 16), DDB_V(8, 1),
    DDB_V(8, 2),  DDB_V(8, 4),  DDB_V(8, 5),  DDB_V(8, 8),  DDB_V(16, 1), DDB_V(16, 2),
    DDB_V(16, 4),
};
#undef DDB_V

KernelFn find_smem_kernel(uint32_t k, uint32_t w, uint32_t* max_threads) {
  for (const SmemVariant& v : kSmemVariants)
    if (static_cast<uint32_t>(v.k) == k && static_cast<uint32_t>(v.w) == w) {
      if (max_threads) *max_threads = static_cast<uint32_t>(v.max_threads);
      return v.fn;
    }
  return nullptr;
}

cudaError_t launch_reference(const float* in, uint64_t pitch, const uint32_t* shifts, float* out,
                             uint64_t out_pitch, uint32_t channels, uint32_t s, uint32_t num_dms,
                             cudaStream_t st) {
  const uint64_t n = static_cast<uint64_t>(num_dms) * s;
  const uint64_t blocks = (n + 255) / 256;
  if (blocks > 0x7fffffffULL) return cudaErrorInvalidValue;
  k_reference<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(in, pitch, shifts, out, out_pitch,
                                                             channels, s, num_dms);
  return cudaGetLastError();
}

cudaError_t launch_direct(const TiledArgs& a, uint32_t blocks, uint32_t threads,
                          cudaStream_t st) {
  k_direct<<<blocks, threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_smem(KernelFn fn, const TiledArgs& a, uint32_t blocks, uint32_t threads,
                        uint32_t smem, cudaStream_t st) {
  fn<<<blocks, threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t prepare_smem(KernelFn fn, uint32_t smem) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

}  // namespace ddb
