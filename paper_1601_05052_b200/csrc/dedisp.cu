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
// The staging pipeline shared by K3 and K4 (the paper's data-reuse lever,
// §3.2).  CTA = tile_dm x tile_time outputs (x depth DM tiles walked in
// sequence).  Per channel the contiguous window [t0+lo, t0+hi+tile_time)
// that the tile's shifts span is copied ONCE into shared memory by a 1-D
// bulk copy (cp.async.bulk -> UBLKCP) and then read by every DM of the
// tile.  Channels are grouped `cps` per stage; `nstage` stages are in
// flight, each guarded by an mbarrier whose transaction count is the
// stage's bytes.  The plan record of each (DM tile, channel) -- lo, span and
// every DM's offset -- rides in the same stage.  CTAs are rastered
// DM-fastest so concurrently resident CTAs share one time range and the
// input is read from HBM about once (the L2 holds the sliding window).
// ---------------------------------------------------------------------
struct Pipe {
  uint64_t* full;   // [nstage] data landed (TMA transaction count)
  uint64_t* empty;  // [nstage] every consumer warp is done with the slot
  uint8_t* recs;
  float* wins;
  uint32_t t0, b_first, nchunk, total;
};

__device__ __forceinline__ Pipe pipe_setup(const TiledArgs& a, uint8_t* smem) {
  Pipe p;
  p.full = reinterpret_cast<uint64_t*>(smem);
  p.empty = reinterpret_cast<uint64_t*>(smem + 64);
  p.recs = smem + 128;
  p.wins = reinterpret_cast<float*>(p.recs + a.nstage * a.cps * a.rec_bytes);
  const uint32_t groups_dm = (a.tiles_dm + a.depth - 1) / a.depth;
  p.t0 = (blockIdx.x / groups_dm) * a.tile_time;
  p.b_first = (blockIdx.x % groups_dm) * a.depth;
  const uint32_t ntiles = min(a.depth, a.tiles_dm - p.b_first);
  p.nchunk = (a.channels + a.cps - 1) / a.cps;
  p.total = ntiles * p.nchunk;
  return p;
}

// Stage chunk g = (tile, channel group) into its slot: one bulk copy for the
// chunk's plan records, one per channel window, all counted on full[slot].
__device__ __forceinline__ void pipe_issue(const TiledArgs& a, const Pipe& p, uint32_t g) {
  const uint32_t b = p.b_first + g / p.nchunk;
  const uint32_t ch0 = (g % p.nchunk) * a.cps;
  const uint32_t ncs = min(a.cps, a.channels - ch0);
  const uint32_t slot = g % a.nstage;
  const uint8_t* rsrc = a.rec + (static_cast<uint64_t>(b) * a.channels + ch0) * a.rec_bytes;
  uint32_t start[8], bytes[8];
  uint32_t total = ncs * a.rec_bytes;
#pragma unroll
  for (uint32_t cc = 0; cc < 8; ++cc) {
    if (cc < ncs) {
      const uint32_t* r = reinterpret_cast<const uint32_t*>(rsrc + cc * a.rec_bytes);
      const uint32_t lo = __ldg(r), span = __ldg(r + 1);
      start[cc] = (p.t0 + lo) & ~3u;
      bytes[cc] = (((p.t0 + lo + span + a.tile_time + 3u) & ~3u) - start[cc]) * 4u;
      total += bytes[cc];
    }
  }
  mbar_arrive_expect_tx(&p.full[slot], total);
  bulk_g2s(p.recs + slot * a.cps * a.rec_bytes, rsrc, ncs * a.rec_bytes, &p.full[slot]);
#pragma unroll
  for (uint32_t cc = 0; cc < 8; ++cc) {
    if (cc < ncs)
      bulk_g2s(p.wins + static_cast<uint64_t>(slot * a.cps + cc) * a.win_cap,
               a.in + static_cast<uint64_t>(ch0 + cc) * a.in_pitch + start[cc], bytes[cc],
               &p.full[slot]);
  }
}

// Warp-specialised pipeline.  The LAST warp of the CTA is the producer: one
// lane runs ahead issuing bulk copies as soon as a slot is handed back
// (empty[slot]), so the plan-record reads and copy latency stay off the
// consumers' path.  The other warps run Body: zero(), channel(rec, window)
// per staged channel, store(dm0, t0) per finished tile; each consumer warp
// releases a slot with one mbarrier arrival -- there is no CTA-wide barrier
// in the loop, so warps drift up to nstage stages apart.
template <class Body>
__device__ __forceinline__ void staged_loop(const TiledArgs& a, uint8_t* smem) {
  const Pipe p = pipe_setup(a, smem);
  const uint32_t tid = threadIdx.x;
  const uint32_t consumers = blockDim.x / 32 - 1;
  if (tid == 0) {
    for (uint32_t s = 0; s < a.nstage; ++s) {
      mbar_init(&p.full[s], 1);
      mbar_init(&p.empty[s], consumers);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (tid >= consumers * 32) {  // producer warp
    if (tid == consumers * 32) {
      for (uint32_t g = 0; g < p.total; ++g) {
        const uint32_t use = g / a.nstage;
        if (use > 0) mbar_wait(&p.empty[g % a.nstage], (use - 1) & 1u);
        pipe_issue(a, p, g);
      }
    }
    return;
  }
  // Consumer threads beyond the config's items (the block is rounded up to
  // whole warps) only take part in the slot hand-back.
  const bool active = tid < a.items_time * a.items_dm;
  Body body(a);
  for (uint32_t g = 0; g < p.total; ++g) {
    const uint32_t q = g % p.nchunk;
    if (q == 0) body.zero();
    const uint32_t slot = g % a.nstage;
    mbar_wait(&p.full[slot], (g / a.nstage) & 1u);
    const uint32_t ncs = min(a.cps, a.channels - q * a.cps);
    const uint8_t* rbase = p.recs + slot * a.cps * a.rec_bytes;
    const float* wbase = p.wins + static_cast<uint64_t>(slot) * a.cps * a.win_cap;
    if (active) {
      for (uint32_t cc = 0; cc < ncs; ++cc) {
        const uint32_t* r = reinterpret_cast<const uint32_t*>(rbase + cc * a.rec_bytes);
        body.channel(r, wbase + cc * a.win_cap + ((p.t0 + r[0]) & 3u));
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&p.empty[slot]);
    if (active && q == p.nchunk - 1)
      body.store((p.b_first + g / p.nchunk) * a.tile_dm, p.t0);
  }
}

// ---------------------------------------------------------------------
// K3 body: the reference's item mapping.  Thread (it, id) keeps its
// work_dm x work_time accumulators in registers (times it + j*items_time,
// DMs id + k*items_dm), so a warp's lanes read consecutive floats: one
// conflict-free shared-memory wavefront per warp-load, one load per add.
// Bound: shared-memory operand bandwidth (32 adds/clk/SM).
// ---------------------------------------------------------------------
template <int K, int W>
struct SmemBody {
  const TiledArgs& a;
  uint32_t it, id;
  float acc[K][W];

  __device__ SmemBody(const TiledArgs& args) : a(args) {
    it = threadIdx.x % a.items_time;
    id = threadIdx.x / a.items_time;
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w) {
    w += it;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* p = w + r[4 + id + k * a.items_dm];
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] += p[j * a.items_time];
    }
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float* o = a.out + static_cast<uint64_t>(dm0 + id + k * a.items_dm) * a.out_pitch + t0 + it;
#pragma unroll
      for (int j = 0; j < W; ++j) o[j * a.items_time] = acc[k][j];
    }
  }
};

// Register budget: K*W accumulators + ~24 bookkeeping registers, so the
// thread cap per variant is what keeps the accumulators out of local memory.
template <int K, int W>
constexpr int smem_max_threads() {
  return K * W > 32 ? 256 : (K * W > 16 ? 512 : 992);
}

template <int K, int W>
__global__ void __launch_bounds__(smem_max_threads<K, W>() + 32) k_smem(const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  staged_loop<SmemBody<K, W>>(a, smem);
}

// ---------------------------------------------------------------------
// K4 body: register windows.  A warp owns K consecutive DMs and 32*W
// consecutive samples (lane l: W contiguous samples; items_time = 32 * warps
// along time).  Per channel each lane loads ONE window of W+SPAN samples
// from shared memory (stride W between lanes, W odd: conflict-free) and
// serves all K DMs from registers: DM k reads window[rel_k .. rel_k+W) with
// rel_k = off_k - min(off).  rel_k is warp-uniform but data-dependent, so a
// jump table over the SPAN+1 static register offsets selects the adds.
// That turns K*W shared loads per channel into W+SPAN (Apertif K=4, W=25:
// 100 adds from 37 loads instead of 100), lifting the shared-memory operand
// bound.  A warp whose K DMs spread further than SPAN in some channel takes
// the direct per-element path for that channel (any table stays exact).
// ---------------------------------------------------------------------
// Five IEEE fp32 adds acc[k][j..j+4] += win[r+j..r+j+4] as one asm block.
// The case number is baked into the asm text: otherwise the compiler
// "sinks" the identical add sequences of all cases into one shared block
// fed by register MOVs (25 MOVs + a compare chain per DM), which is exactly
// the overhead the jump table exists to avoid.
#define DDB_ADD5(R, J)                                                              \
  asm volatile(                                                                     \
      "add.rn.f32 %0, %0, %5;\n\tadd.rn.f32 %1, %1, %6;\n\tadd.rn.f32 %2, %2, %7;\n\t" \
      "add.rn.f32 %3, %3, %8;\n\tadd.rn.f32 %4, %4, %9; // rw" #R                   \
      : "+f"(acc[k][J]), "+f"(acc[k][J + 1]), "+f"(acc[k][J + 2]), "+f"(acc[k][J + 3]), \
        "+f"(acc[k][J + 4])                                                         \
      : "f"(win[R + J]), "f"(win[R + J + 1]), "f"(win[R + J + 2]), "f"(win[R + J + 3]), \
        "f"(win[R + J + 4]))

#define DDB_CASE(R)                                        \
  case R:                                                  \
    if constexpr (R <= SPAN) {                             \
      _Pragma("unroll") for (int j = 0; j < W; j += 5)     \
          DDB_ADD5(R, j);                                  \
    }                                                      \
    break;

template <int K, int W, int SPAN>
struct RegWinBody {
  static_assert(SPAN <= 31, "jump table covers 0..31");
  static_assert(W % 5 == 0, "cases add in groups of five");
  const TiledArgs& a;
  uint32_t col;  // first sample of this lane relative to t0
  uint32_t dml;  // first DM of this warp relative to dm0
  float acc[K][W];

  __device__ RegWinBody(const TiledArgs& args) : a(args) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t warps_time = a.items_time >> 5;
    col = ((warp % warps_time) * 32 + lane) * W;
    dml = (warp / warps_time) * K;
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w) {
    uint32_t off[K];
#pragma unroll
    for (int k = 0; k < K; ++k) off[k] = r[4 + dml + k];
    // The window starts at the warp's FIRST DM, so for non-decreasing rows
    // (every table build_delay_table makes) DM 0 reads window[0..W) with no
    // dispatch; any row below it or further than SPAN takes the direct path.
    bool fast = true;
#pragma unroll
    for (int k = 1; k < K; ++k) fast = fast && (off[k] - off[0] <= static_cast<uint32_t>(SPAN));
    const float* p = w + col;
    if (fast) {
      float win[W + SPAN];
      p += off[0];
#pragma unroll
      for (int i = 0; i < W + SPAN; ++i) win[i] = p[i];
#pragma unroll
      for (int j = 0; j < W; ++j) acc[0][j] += win[j];
#pragma unroll
      for (int k = 1; k < K; ++k) {
        switch (off[k] - off[0]) {
          DDB_CASE(0) DDB_CASE(1) DDB_CASE(2) DDB_CASE(3) DDB_CASE(4) DDB_CASE(5) DDB_CASE(6)
          DDB_CASE(7) DDB_CASE(8) DDB_CASE(9) DDB_CASE(10) DDB_CASE(11) DDB_CASE(12)
          DDB_CASE(13) DDB_CASE(14) DDB_CASE(15) DDB_CASE(16) DDB_CASE(17) DDB_CASE(18)
          DDB_CASE(19) DDB_CASE(20) DDB_CASE(21) DDB_CASE(22) DDB_CASE(23) DDB_CASE(24)
          DDB_CASE(25) DDB_CASE(26) DDB_CASE(27) DDB_CASE(28) DDB_CASE(29) DDB_CASE(30)
          DDB_CASE(31)
          default:
            break;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float* q = p + off[k];
#pragma unroll
        for (int j = 0; j < W; ++j) acc[k][j] += q[j];
      }
    }
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float* o = a.out + static_cast<uint64_t>(dm0 + dml + k) * a.out_pitch + t0 + col;
#pragma unroll
      for (int j = 0; j < W; ++j) o[j] = acc[k][j];
    }
  }
};
#undef DDB_CASE
#undef DDB_ADD5

template <int K, int W, int SPAN>
__global__ void __launch_bounds__(288) k_regwin(const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  staged_loop<RegWinBody<K, W, SPAN>>(a, smem);
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

struct RegWinVariant {
  int k, w, span;
  KernelFn fn;
};

#define DDB_R(K, W, S) {K, W, S, k_regwin<K, W, S>}
static const RegWinVariant kRegWinVariants[] = {
    DDB_R(2, 25, 8),  DDB_R(2, 25, 16), DDB_R(4, 25, 8),  DDB_R(4, 25, 16), DDB_R(4, 25, 31),
    DDB_R(4, 5, 8),   DDB_R(4, 5, 16),  DDB_R(8, 5, 16),  DDB_R(8, 5, 31),  DDB_R(16, 5, 31),
};
#undef DDB_R

// Smallest-SPAN variant that covers `group_span` (the widest spread of any
// work_dm-DM group in any channel); the widest one when none does (its
// direct path keeps outliers exact).  *span_out = the chosen SPAN.
KernelFn find_regwin_kernel(uint32_t k, uint32_t w, uint32_t group_span, uint32_t* span_out) {
  const RegWinVariant* cover = nullptr;  // smallest span >= group_span
  const RegWinVariant* widest = nullptr;
  for (const RegWinVariant& v : kRegWinVariants) {
    if (static_cast<uint32_t>(v.k) != k || static_cast<uint32_t>(v.w) != w) continue;
    if (widest == nullptr || v.span > widest->span) widest = &v;
    if (static_cast<uint32_t>(v.span) >= group_span && (cover == nullptr || v.span < cover->span))
      cover = &v;
  }
  const RegWinVariant* pick = cover ? cover : widest;
  if (pick == nullptr) return nullptr;
  if (span_out) *span_out = static_cast<uint32_t>(pick->span);
  return pick->fn;
}

bool regwin_shape_ok(uint32_t k, uint32_t w, uint32_t items_time, uint64_t block) {
  if (items_time % 32 != 0 || block > 256) return false;
  for (const RegWinVariant& v : kRegWinVariants)
    if (static_cast<uint32_t>(v.k) == k && static_cast<uint32_t>(v.w) == w) return true;
  return false;
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
