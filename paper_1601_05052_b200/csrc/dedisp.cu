// dedisp.cu -- the dedispersion kernels (K2 reference-order, K2' direct
// tiled, K3 TMA-staged tiled) for sm_100a.
//
// Arithmetic contract (reference kernels.cpp:83-108): each
// output element owns ONE fp32 accumulator, starts at 0.0f and adds the
// channels in ascending order with IEEE round-to-nearest adds.  Tiling and
// thread mapping change only the schedule, never that sequence, so every
// kernel here is bit-identical to dedisperse_reference.  Build flags must
// not enable fast-math / FTZ (see build.py).
#include <map>
#include <mutex>
#include <utility>

#include <cuda.h>

#include "common.cuh"
#include "regwin_dispatch.cuh"

namespace ddb {

// Bounds of the shared-memory stage a consumer is reading (checked builds).
struct ChkRange {
#ifdef DDB_CHECKED
  const float* lo = nullptr;
  const float* hi = nullptr;
  __device__ __forceinline__ void check(const float* p, int n) const {
    DDB_CHECK(p >= lo && p + n <= hi);
  }
#else
  __device__ __forceinline__ void check(const float*, int) const {}
#endif
};

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
// This CTA's beam: output rows of beam blockIdx.y (staged families).
__device__ __forceinline__ float* beam_out(const TiledArgs& a) {
  return a.out + blockIdx.y * a.out_beam_stride;
}

// Consumers waiting for a stage: spin on try_wait, or (DDB_CONSUMER_SLEEP,
// an A/B switch) let the hardware park the warp until the phase completes so
// the spin does not take issue slots from the warps that have work.
#ifndef DDB_CONSUMER_SLEEP
#define DDB_CONSUMER_SLEEP 0
#endif
__device__ __forceinline__ void consumer_wait(uint64_t* bar, uint32_t parity) {
  if constexpr (DDB_CONSUMER_SLEEP)
    mbar_wait_sleep(bar, parity);
  else
    mbar_wait(bar, parity);
}

struct Pipe {
  uint64_t* full;   // [nstage] data landed (TMA transaction count)
  uint64_t* empty;  // [nstage] every consumer warp is done with the slot
  uint8_t* recs;
  float* wins;
  uint32_t t0, b_first, nchunk, total;
};

template <bool PK>
__device__ __forceinline__ Pipe pipe_setup(const TiledArgs& a, uint8_t* smem) {
  Pipe p;
  p.full = reinterpret_cast<uint64_t*>(smem);
  p.empty = reinterpret_cast<uint64_t*>(smem + 64);
  p.recs = smem + kPipeHeader;
  p.wins = reinterpret_cast<float*>(p.recs + a.nstage * a.cps * a.rec_bytes);  // 16-B aligned
  const uint32_t groups_dm = (a.tiles_dm + a.depth - 1) / a.depth;
  if (a.time_major) {
    // time-fastest: the resident CTAs cover few DM groups over many time
    // tiles, so their windows share one input region per DM group (for
    // large delays, where DM-fastest CTAs touch the whole block at once)
    p.t0 = (blockIdx.x % a.tiles_time) * a.tile_time;
    p.b_first = (blockIdx.x / a.tiles_time) * a.depth;
  } else {
    p.t0 = (blockIdx.x / groups_dm) * a.tile_time;
    p.b_first = (blockIdx.x % groups_dm) * a.depth;
  }
  const uint32_t ntiles = min(a.depth, a.tiles_dm - p.b_first);
  if constexpr (PK)
    p.nchunk = a.packed_stages;
  else
    p.nchunk = (a.ch_end - a.ch_begin + a.cps - 1) / a.cps;
  p.total = ntiles * p.nchunk;
  return p;
}

// Channels of stage q (of a tile): first channel and count.  PK (packed
// stages, compile time: a runtime switch here cost every build ~15%) reads
// the plan's stage table.
template <bool PK>
__device__ __forceinline__ void stage_channels(const TiledArgs& a, uint32_t q, uint32_t& ch0,
                                               uint32_t& ncs) {
  if constexpr (PK) {
    ch0 = __ldg(a.stage_ch + q);
    ncs = __ldg(a.stage_ch + q + 1) - ch0;
  } else {
    ch0 = a.ch_begin + q * a.cps;
    ncs = min(a.cps, a.ch_end - ch0);
  }
}

// Offset (floats) of window cc of a stage whose first channel is ch0, and
// of a stage buffer.
template <bool PK>
__device__ __forceinline__ uint32_t window_offset(const TiledArgs& a, uint32_t ch0, uint32_t cc) {
  if constexpr (PK)
    return __ldg(a.chan_off + ch0 + cc);
  else
    return cc * a.win_cap;
}
template <bool PK>
__device__ __forceinline__ uint64_t stage_offset(const TiledArgs& a, uint32_t slot) {
  if constexpr (PK)
    return static_cast<uint64_t>(slot) * a.stage_floats;
  else
    return static_cast<uint64_t>(slot * a.cps) * a.win_cap;
}

// The producer warp.  Lane cc stages channel cc of each chunk (one bulk
// copy per lane, in parallel); lane 0 also copies the chunk's plan records
// and closes the phase.  Each lane keeps the (lo, span) of its channel for
// the next kSpanAhead chunks in registers, loaded from global memory that
// many chunks ahead: with short per-chunk work (few DMs, small d) the
// producer otherwise waits one L2 round trip per chunk.
constexpr int kSpanAhead = 4;

template <bool PK>
__device__ __forceinline__ uint2 lane_span(const TiledArgs& a, const Pipe& p, uint32_t g,
                                           uint32_t lane) {
  if (g >= p.total) return make_uint2(0u, 0u);
  const uint32_t b = p.b_first + g / p.nchunk;
  uint32_t ch0, ncs;
  stage_channels<PK>(a, g % p.nchunk, ch0, ncs);
  if (lane >= ncs) return make_uint2(0u, 0u);
  return __ldg(a.ls + static_cast<uint64_t>(b) * a.channels + ch0 + lane);
}

// Stage chunk g = (tile, channel group) into its slot: one bulk copy for the
// chunk's plan records (lane 0), one per channel window (lane cc), all
// counted on full[slot].
template <bool PK>
__device__ __forceinline__ void pipe_issue(const TiledArgs& a, const Pipe& p, uint32_t g,
                                           uint2 ls, uint32_t lane) {
  const uint32_t b = p.b_first + g / p.nchunk;
  uint32_t ch0, ncs;
  stage_channels<PK>(a, g % p.nchunk, ch0, ncs);
  const uint32_t slot = g % a.nstage;
  uint64_t* bar = &p.full[slot];
  // Each copy first raises the phase's expected bytes; the closing arrival
  // (the phase's only one, after the warp has issued every copy) cannot
  // complete it before every copy is counted.
  if (lane == 0) {
    const uint8_t* rsrc = a.rec + (static_cast<uint64_t>(b) * a.channels + ch0) * a.rec_bytes;
    mbar_expect_tx(bar, ncs * a.rec_bytes);
    bulk_g2s(p.recs + slot * a.cps * a.rec_bytes, rsrc, ncs * a.rec_bytes, bar);
  }
  if (lane < ncs) {
    const uint32_t cc = lane;
    const float* src =
        a.in + blockIdx.y * a.in_beam_stride + static_cast<uint64_t>(ch0 + cc) * a.in_pitch;
    float* dst = p.wins + stage_offset<PK>(a, slot);
    const uint32_t lo = ls.x, span = ls.y;
    const uint32_t start = (p.t0 + lo) & ~3u;
    // a predicated last time tile must not read past the (pitched) row
    const uint32_t end = min((p.t0 + lo + span + a.tile_time + 3u) & ~3u,
                             static_cast<uint32_t>(a.in_pitch));
    const uint32_t bytes = (end - start) * 4u;
    // the copy stays inside its channel's row and its stage slot
    DDB_CHECK(start < end && ch0 + cc < a.channels);
    DDB_CHECK(window_offset<PK>(a, ch0, cc) + (end - start) <=
              (PK ? a.stage_floats : a.cps * a.win_cap));
    mbar_expect_tx(bar, bytes);
    bulk_g2s(dst + window_offset<PK>(a, ch0, cc), src + start, bytes, bar);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}

// The producer warp: issue every chunk as soon as its slot is handed back.
template <bool PK>
__device__ __forceinline__ void pipe_produce(const TiledArgs& a, const Pipe& p) {
  const uint32_t lane = threadIdx.x & 31;
  uint2 ahead[kSpanAhead];
#pragma unroll
  for (int i = 0; i < kSpanAhead; ++i) ahead[i] = lane_span<PK>(a, p, i, lane);
  for (uint32_t g = 0; g < p.total; ++g) {
    const uint2 cur = ahead[0];
#pragma unroll
    for (int i = 0; i + 1 < kSpanAhead; ++i) ahead[i] = ahead[i + 1];
    ahead[kSpanAhead - 1] = lane_span<PK>(a, p, g + kSpanAhead, lane);
    const uint32_t use = g / a.nstage;
    if (use > 0) mbar_wait_sleep(&p.empty[g % a.nstage], (use - 1) & 1u);
    pipe_issue<PK>(a, p, g, cur, lane);
  }
}

// Channels per unrolled step of the consumer loop (Body::kUnroll, default 1).
template <class B, class = void>
struct ChannelUnroll {
  static constexpr uint32_t value = 1;
};
template <class B>
struct ChannelUnroll<B, decltype(void(B::kUnroll))> {
  static constexpr uint32_t value = B::kUnroll;
};

// Bodies that prefetch the next channel's record entry (kGroupPrefetch).
template <class B, class = void>
struct GroupPrefetch {
  static constexpr bool value = false;
};
template <class B>
struct GroupPrefetch<B, decltype(void(B::kGroupPrefetch))> {
  static constexpr bool value = B::kGroupPrefetch;
};

// Bodies that run a whole stage themselves (kStagePipe = true).
template <class B, class = void>
struct HasStagePipe {
  static constexpr bool value = false;
};
template <class B>
struct HasStagePipe<B, decltype(void(B::kStagePipe))> {
  static constexpr bool value = B::kStagePipe;
};

// Warp-specialised pipeline.  The LAST warp of the CTA is the producer: one
// lane runs ahead issuing bulk copies as soon as a slot is handed back
// (empty[slot]), so the plan-record reads and copy latency stay off the
// consumers' path.  The other warps run Body: zero(), channel(rec, window)
// per staged channel, store(dm0, t0) per finished tile; each consumer warp
// releases a slot with one mbarrier arrival -- there is no CTA-wide barrier
// in the loop, so warps drift up to nstage stages apart.
template <class Body, class... Extra>
__device__ __forceinline__ void staged_loop_with(const TiledArgs& a, uint8_t* smem,
                                                 Extra... extra) {
  constexpr bool PK = Body::kPacked;
  const Pipe p = pipe_setup<PK>(a, smem);
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
    pipe_produce<PK>(a, p);
    return;
  }
  // Consumer threads beyond the config's items (the block is rounded up to
  // whole warps) only take part in the slot hand-back.
  const bool active = tid < a.items_time * a.items_dm;
  Body body(a, extra...);
  for (uint32_t g = 0; g < p.total; ++g) {
    const uint32_t q = g % p.nchunk;
    if (q == 0) {
      if (a.accumulate && active)
        body.load((p.b_first + g / p.nchunk) * a.tile_dm, p.t0);
      else
        body.zero();
    }
    const uint32_t slot = g % a.nstage;
    consumer_wait(&p.full[slot], (g / a.nstage) & 1u);
    uint32_t ch0, ncs;
    stage_channels<PK>(a, q, ch0, ncs);
    const uint8_t* rbase = p.recs + slot * a.cps * a.rec_bytes;
    const float* wbase = p.wins + stage_offset<PK>(a, slot);
#ifdef DDB_CHECKED
    body.chk.lo = wbase;
    body.chk.hi = wbase + (PK ? a.stage_floats : a.cps * a.win_cap);
#endif
    if (active) {
      if constexpr (HasStagePipe<Body>::value) {
        body.stage(rbase, wbase, ncs);
      } else {
        const auto one = [&](uint32_t cc) {
          const uint32_t* r = reinterpret_cast<const uint32_t*>(rbase + cc * a.rec_bytes);
          const float* w = wbase + window_offset<PK>(a, ch0, cc);
          if constexpr (GroupPrefetch<Body>::value)
            body.channel(r, w, cc + 1 < ncs);
          else if constexpr (Body::kRowBase)
            body.channel(r, w);
          else
            body.channel(r, w + ((p.t0 + r[0]) & 3u));
        };
        uint32_t cc = 0;
        if constexpr (ChannelUnroll<Body>::value > 1) {
          // light bodies (few accumulators: small d): U channels per step so
          // their record and operand loads overlap instead of forming one
          // latency chain per channel
          constexpr uint32_t U = ChannelUnroll<Body>::value;
          for (; cc + U <= ncs; cc += U) {
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) one(cc + u);
          }
        }
        for (; cc < ncs; ++cc) one(cc);
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&p.empty[slot]);
    if (active && q == p.nchunk - 1)
      body.store((p.b_first + g / p.nchunk) * a.tile_dm, p.t0);
  }
}

template <class Body>
__device__ __forceinline__ void staged_loop(const TiledArgs& a, uint8_t* smem) {
  staged_loop_with<Body>(a, smem);
}

// ---------------------------------------------------------------------
// K3 body: the reference's item mapping.  Thread (it, id) keeps its
// work_dm x work_time accumulators in registers (times it + j*items_time,
// DMs id + k*items_dm), so a warp's lanes read consecutive floats: one
// conflict-free shared-memory wavefront per warp-load, one load per add.
// Bound: shared-memory operand bandwidth (32 adds/clk/SM).
// ---------------------------------------------------------------------
template <int K, int W, int IT = 0, bool PK = false>
struct SmemBody {
  static constexpr bool kRowBase = false;  // channel() gets the row at lo's sample
  static constexpr bool kPacked = PK;      // packed stages (compile time)
#ifndef DDB_SMEM_UNROLL
#define DDB_SMEM_UNROLL 4
#endif
  // few accumulators per thread (small d): unroll the channel loop
  static constexpr uint32_t kUnroll = K * W <= 8 ? DDB_SMEM_UNROLL : 1;
  const TiledArgs& a;
  uint32_t it, id;
  float acc[K][W];
  ChkRange chk;

  // IT > 0: items_time fixed at compile time, so a thread's W samples sit
  // at immediate offsets from one address (no per-load address arithmetic)
  __device__ __forceinline__ uint32_t stride() const { return IT > 0 ? IT : a.items_time; }
  __device__ SmemBody(const TiledArgs& args) : a(args) {
    it = threadIdx.x % stride();
    id = threadIdx.x / stride();
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }
  // The K*W adds issue in pairs as FADD2 (flattened (k, j) order, two
  // independent RN adds each: bit-exact), halving the FP32 instructions of
  // the loop; an odd K*W leaves one scalar add.
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w) {
    w += it;
    const float* p[K];
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = w + r[4 + id + k * a.items_dm];
#ifdef DDB_CHECKED
    for (int k = 0; k < K; ++k) chk.check(p[k], (W - 1) * stride() + 1);
#endif
#pragma unroll
    for (int n = 0; n + 1 < K * W; n += 2) {
      const int k0 = n / W, j0 = n % W, k1 = (n + 1) / W, j1 = (n + 1) % W;
      const float2 s = fadd2(make_float2(acc[k0][j0], acc[k1][j1]),
                             make_float2(p[k0][j0 * stride()], p[k1][j1 * stride()]));
      acc[k0][j0] = s.x;
      acc[k1][j1] = s.y;
    }
    if ((K * W) & 1) acc[K - 1][W - 1] += p[K - 1][(W - 1) * stride()];
  }
  __device__ __forceinline__ void load(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* o =
          beam_out(a) + static_cast<uint64_t>(dm0 + id + k * a.items_dm) * a.out_pitch + t0 + it;
#pragma unroll
      for (int j = 0; j < W; ++j)
        acc[k][j] = t0 + it + j * a.items_time < a.s ? o[j * a.items_time] : 0.0f;
    }
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      DDB_CHECK(dm0 + id + k * a.items_dm < a.num_dms);
      float* o =
          beam_out(a) + static_cast<uint64_t>(dm0 + id + k * a.items_dm) * a.out_pitch + t0 + it;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (t0 + it + j * a.items_time < a.s) o[j * a.items_time] = acc[k][j];
    }
  }
};

// Register budget: K*W accumulators + ~24 bookkeeping registers, so the
// thread cap per variant is what keeps the accumulators out of local memory.
template <int K, int W>
constexpr int smem_max_threads() {
  return K * W > 32 ? 256 : (K * W > 16 ? 512 : 992);
}

// MT > 0: a build for up to MT consumer threads (instead of the
// accumulator-count default) -- e.g. two DM rows of 160 threads
template <int K, int W, int IT = 0, bool PK = false, int MT = 0>
__global__ void __launch_bounds__((MT > 0 ? MT : smem_max_threads<K, W>()) + 32)
    k_smem(const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  staged_loop<SmemBody<K, W, IT, PK>>(a, smem);
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
// The register-window dispatch (acc[j] += win[rel + j], rel warp-uniform
// but data-dependent) is generated PTX: one brx.idx.uni jump table per DM
// (regwin_dispatch.cuh, from gen_dispatch.py).  Written as a C++ switch,
// nvcc sinks the identical add blocks of all cases into one block fed by
// register MOVs, or lowers the switch to a compare tree with reconvergence
// barriers -- both several times the cost of the adds themselves.
__device__ __forceinline__ float4 lds128(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

// Window geometry of a register-window variant.  W % 4 == 0 ("vector"):
// lanes own W contiguous samples at a stride of W floats with W/4 odd, so
// 16-byte loads of 32 lanes hit 8 distinct bank groups (conflict-free); the
// window is read from the 16-byte-aligned address at or below its start and
// the misalignment (0..3) is folded into every DM's dispatch offset.
// Otherwise ("scalar", W odd): 4-byte loads at an odd stride, also
// conflict-free, and DM 0 needs no dispatch.
template <int W, int SPAN>
struct RwGeom {
  static constexpr bool kVec = W % 4 == 0;
  static constexpr int kMaxRel = kVec ? SPAN + 3 : SPAN;
  static constexpr int kWin = kVec ? ((W + SPAN + 3 + 3) / 4) * 4 : W + SPAN;
};

// One staged channel as seen by a register-window warp: its offsets, the
// fast/slow decision, and (fast) the lane's window in registers.
template <int K, int W, int SPAN>
struct RwChan {
  const float* base;  // lane's column at window position 0 (input time t0+lo)
  uint32_t off[K];
  uint32_t al;        // vector mode: misalignment of the window start
  bool fast;
  float win[RwGeom<W, SPAN>::kWin];
};

template <int K, int W, int SPAN>
struct RegWin {
  static constexpr int kMaxRel = RwGeom<W, SPAN>::kMaxRel;
  static constexpr int kWin = RwGeom<W, SPAN>::kWin;
  static_assert(kMaxRel <= 31, "jump table covers 0..31");
  static_assert(W % 5 == 0 || W % 4 == 0, "cases add in groups of four or five");
  float acc[K][W];

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }

  // Issue the shared-memory reads of one channel (results land while the
  // previous channel's adds run).  The window starts at the warp's FIRST
  // DM; for non-decreasing rows (every table build_delay_table makes) the
  // other DMs sit 0..SPAN samples later.  Rows below the first or further
  // than SPAN take the direct path, so any table stays exact.
  __device__ __forceinline__ static void load(RwChan<K, W, SPAN>& c, const uint32_t* r,
                                              const float* w, uint32_t col, uint32_t dml) {
#pragma unroll
    for (int k = 0; k < K; ++k) c.off[k] = r[4 + dml + k];
    bool fast = true;
#pragma unroll
    for (int k = 1; k < K; ++k) fast = fast && (c.off[k] - c.off[0] <= static_cast<uint32_t>(SPAN));
    c.fast = fast;
    c.base = w + col;
    if (fast) {
      const float* p = c.base + c.off[0];
      if constexpr (RwGeom<W, SPAN>::kVec) {
        c.al = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(p) >> 2) & 3u;
        const float* pa = p - c.al;
#pragma unroll
        for (int i = 0; i < kWin / 4; ++i) {
          const float4 v = lds128(pa + 4 * i);
          c.win[4 * i] = v.x;
          c.win[4 * i + 1] = v.y;
          c.win[4 * i + 2] = v.z;
          c.win[4 * i + 3] = v.w;
        }
      } else {
        c.al = 0;
#pragma unroll
        for (int i = 0; i < kWin; ++i) c.win[i] = p[i];
      }
    }
  }

  __device__ __forceinline__ void compute(const RwChan<K, W, SPAN>& c) {
    if (c.fast) {
      if constexpr (RwGeom<W, SPAN>::kVec) {
#pragma unroll
        for (int k = 0; k < K; ++k)
          rw_dispatch<W, kWin, kMaxRel>(acc[k], c.win, c.al + c.off[k] - c.off[0]);
      } else {
#pragma unroll
        for (int j = 0; j < W; ++j) acc[0][j] += c.win[j];
#pragma unroll
        for (int k = 1; k < K; ++k) rw_dispatch<W, kWin, kMaxRel>(acc[k], c.win, c.off[k] - c.off[0]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float* q = c.base + c.off[k];
#pragma unroll
        for (int j = 0; j < W; ++j) acc[k][j] += q[j];
      }
    }
  }
};

// K4 body: one register-window channel at a time (load then compute).  A
// software-pipelined variant that prefetched the next channel's window was
// measured 2x slower: the doubled register footprint halved the resident
// warps, and warp-level parallelism hides the shared-memory latency better.
template <int K, int W, int SPAN>
struct RegWinBody {
  static constexpr bool kRowBase = false;
  static constexpr bool kPacked = false;
  const TiledArgs& a;
  uint32_t col;  // first sample of this lane relative to t0
  uint32_t dml;  // first DM of this warp relative to dm0
  RegWin<K, W, SPAN> rw;
  ChkRange chk;

  __device__ RegWinBody(const TiledArgs& args) : a(args) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t warps_time = a.items_time >> 5;
    col = ((warp % warps_time) * 32 + lane) * W;
    dml = (warp / warps_time) * K;
  }
  __device__ __forceinline__ void zero() { rw.zero(); }
  __device__ __forceinline__ void load(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* o = beam_out(a) + static_cast<uint64_t>(dm0 + dml + k) * a.out_pitch + t0 + col;
#pragma unroll
      for (int j = 0; j < W; ++j) rw.acc[k][j] = t0 + col + j < a.s ? o[j] : 0.0f;
    }
  }
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w) {
    RwChan<K, W, SPAN> c;
    RegWin<K, W, SPAN>::load(c, r, w, col, dml);
#ifdef DDB_CHECKED
    if (c.fast) {
      chk.check(c.base + c.off[0] - c.al, RwGeom<W, SPAN>::kWin);
    } else {
      for (int k = 0; k < K; ++k) chk.check(c.base + c.off[k], W);
    }
#endif
    rw.compute(c);
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      DDB_CHECK(dm0 + dml + k < a.num_dms);
      float* o = beam_out(a) + static_cast<uint64_t>(dm0 + dml + k) * a.out_pitch + t0 + col;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (t0 + col + j < a.s) o[j] = rw.acc[k][j];
    }
  }
};

// Register cap per variant: the accumulators, one window and ~40 registers
// of addressing.  A tight cap is what lets several CTAs share an SM; ptxas
// left to itself spends the whole file on one CTA.
template <int K, int W, int SPAN>
constexpr int regwin_maxreg() {
  return ((K * W + RwGeom<W, SPAN>::kWin + 40 + 7) / 8) * 8;
}

template <int K, int W, int SPAN>
__global__ void __maxnreg__((regwin_maxreg<K, W, SPAN>())) k_regwin(const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  staged_loop<RegWinBody<K, W, SPAN>>(a, smem);
}

// ---------------------------------------------------------------------
// K5: TMEM windows.  Same ownership as K4 (a warp owns K consecutive DMs
// and 32*W consecutive samples; W % 4 == 0 with W/4 odd so 16-byte window
// loads are conflict-free), but the data-dependent selection is done by
// the tensor-memory datapath instead of a jump table: each lane writes its
// window into its own TMEM row (tcgen05.st, 32x32b), and every DM reads W
// columns back at the warp-uniform dynamic column offset rel_k
// (tcgen05.ld at taddr + rel_k) -- TMEM used as a dynamically indexed
// register file.  The loaded vectors are adjacent registers, so the adds
// issue as FADD2 (add.rn.f32x2: two independent IEEE RN adds).  Bit-exact:
// every output still gets one add per channel, channels ascending.
// ---------------------------------------------------------------------
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]),
      "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]),
      "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                   taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
               "f"(v[7])
               : "memory");
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
               : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                 "=f"(r[6]), "=f"(r[7])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7]), "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]),
        "=f"(r[14]), "=f"(r[15])
      : "r"(taddr)
      : "memory");
}

// W = 12 as x8 + x4 in ONE asm statement: both loads address the same
// register ([taddr], [taddr+8]), so ptxas moves the column to a uniform
// register once (one R2UR per DM instead of two)
__device__ __forceinline__ void tmem_ld12(uint32_t taddr, float* r) {
  asm volatile(
      "{\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%12];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8, %9, %10, %11}, [%12+8];\n\t}"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7]), "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11])
      : "r"(taddr)
      : "memory");
}

// W = 20 as x16 + x4 in one asm statement (two LDTMs instead of three)
__device__ __forceinline__ void tmem_ld20(uint32_t taddr, float* r) {
  asm volatile(
      "{\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%20];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16, %17, %18, %19}, [%20+16];\n\t}"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
        "=f"(r[7]), "=f"(r[8]), "=f"(r[9]), "=f"(r[10]), "=f"(r[11]), "=f"(r[12]), "=f"(r[13]),
        "=f"(r[14]), "=f"(r[15]), "=f"(r[16]), "=f"(r[17]), "=f"(r[18]), "=f"(r[19])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#ifndef DDB_TMEM_GROUP
#define DDB_TMEM_GROUP 4
#endif
#ifndef DDB_TMEM_READ16
#define DDB_TMEM_READ16 0
#endif
#ifndef DDB_TMEM_LD12
#define DDB_TMEM_LD12 1
#endif
#ifndef DDB_TMEM_LD20
#define DDB_TMEM_LD20 0
#endif
#ifndef DDB_TMEM_ST_SPLIT
#define DDB_TMEM_ST_SPLIT 1
#endif
#ifndef DDB_TMEM_TAIL_EARLY
#define DDB_TMEM_TAIL_EARLY 1
#endif
#ifndef DDB_TMEM_GPREFETCH
#define DDB_TMEM_GPREFETCH 0
#endif
// the warp's TMEM address broadcast from lane 0 (__shfl_sync), so ptxas
// keeps it in a uniform register: the window stores address tmem[UR + imm]
// with no R2UR per store and the DM reads add it as a uniform operand.
// Measured (profiles/r02_ab_tmem_uniform.txt, --cold): W = 12 K = 8 at
// Apertif d=4096 5.994 -> 5.805 ms, d=1024 1.575 -> 1.524 ms; the W = 20
// build (d=128) 0.262 -> 0.270 ms, so it is applied to W = 12 only
#ifndef DDB_TMEM_UNIFORM
#define DDB_TMEM_UNIFORM 1
#endif
// the x8 window tail stored unconditionally (columns no DM reads when the
// window fits 32): no branch + WARPSYNC around the tail store
// the channel's window geometry (vectors, start) broadcast from lane 0 too:
// its tests become uniform branches
#ifndef DDB_TMEM_UNIFORM_G
#define DDB_TMEM_UNIFORM_G 0
#endif
#ifndef DDB_TMEM_TAIL_ALWAYS
#define DDB_TMEM_TAIL_ALWAYS 0
#endif
// launch bound of k_tmemwin: 288 threads (up to 8 consumer warps), or an A/B
// build bounded to 160 threads x 2 CTAs (<= 204 registers)
#ifndef DDB_TMEM_LB2
#define DDB_TMEM_LB2 0
#endif
// software-pipelined stages: channel c+1's window loads (LDS) are issued
// before channel c's TMEM reads and adds, and land in a second TMEM column
// block, so the window stores no longer wait on the shared-memory loads
#ifndef DDB_TMEM_PIPE
#define DDB_TMEM_PIPE 0
#endif

template <int K, int W, int SPAN, int COLS, bool FULL_HEAD = true>
struct TmemBody {
  static constexpr bool kRowBase = true;  // channel() gets the 16-byte aligned row start
  static constexpr bool kPacked = false;
  static constexpr bool kStagePipe = DDB_TMEM_PIPE != 0;
  static constexpr int kBufs = kStagePipe ? 2 : 1;  // TMEM window blocks per warp
  static_assert(W % 4 == 0, "16-byte window loads (W/4 odd is conflict-free, even is 2-way)");
  static_assert(COLS == 32 || COLS == 64, "32 or 64 TMEM columns per warp window");
  static_assert(W + SPAN + 3 <= COLS, "window must fit the warp's TMEM columns");
  static_assert(K % 2 == 0, "DMs are read back in pairs");
  static constexpr bool kFullHead = FULL_HEAD;
  // head vectors loaded unconditionally; the last one only when the window
  // reaches it (measured: 8 always 6.68 ms, 7 + 1 predicated 6.53, 6 + 2
  // 6.56 at Apertif d=4096 -- the predicated vector saves shared-memory
  // bandwidth, but each predicated register stays live across the channel)
#ifndef DDB_TMEM_HEAD_ALWAYS
#define DDB_TMEM_HEAD_ALWAYS 7
#endif
  static constexpr int kHeadAlways = DDB_TMEM_HEAD_ALWAYS;
  // window columns beyond the first 32: 0, 8, 16 or 32
  static constexpr int kNeed = W + SPAN + 3 - 32;
  static constexpr int kTail = kNeed <= 0 ? 0 : kNeed <= 8 ? 8 : kNeed <= 16 ? 16 : 32;
  // an x8 tail loaded right after the head (DDB_TMEM_TAIL_EARLY), so its
  // shared-memory latency overlaps the head's stores
  static constexpr bool kTailEarly = DDB_TMEM_TAIL_EARLY && kTail == 8;
  static_assert(kTail == 0 || COLS == 64, "windows past 32 columns need 64 per warp");
  const TiledArgs& a;
  uint32_t col, dml, taddr;
  float acc[K][W];
  ChkRange chk;

  __device__ TmemBody(const TiledArgs& args, uint32_t tmem_base) : a(args) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t warps_time = a.items_time >> 5;
    col = ((warp % warps_time) * 32 + lane) * W;
    dml = (warp / warps_time) * K;
    // lanes (warp % 4) * 32.. are this warp's TMEM rows; COLS columns per warp
    taddr = tmem_base + (((warp & 3) * 32) << 16) + (warp >> 2) * COLS * kBufs;
    if constexpr (DDB_TMEM_UNIFORM && W == 12) taddr = __shfl_sync(0xffffffffu, taddr, 0);
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }
  // Per-channel state fetched from shared memory.
  struct Pre {
    uint32_t off[K];  // window columns of the warp's DMs (k_plan window format)
    uint32_t nv;      // 16-byte window vectors to stage; 0 = slow path
    const float* base;  // this lane's 16-byte aligned window start
    float win[32];  // first 32 window columns (fast path)
    float tail[kTailEarly ? 8 : 1];  // columns 32..39, loaded with the head
  };

  // Offsets + (fast) the first half of the window: only the 16-byte vectors
  // the warp's DMs actually span this channel (nv, warp-uniform) are read.
  // k_plan's window format (table.cu) precomputes the columns relative to
  // the aligned window start, the alignment and the start itself.
  __device__ __forceinline__ void fetch(Pre& n, const uint32_t* r, const float* w) const {
    if constexpr (K % 4 == 0) {
      const uint4* o = reinterpret_cast<const uint4*>(r + 4 + dml);
#pragma unroll
      for (int k = 0; k < K; k += 4) {
        const uint4 v = o[k / 4];
        n.off[k] = v.x;
        n.off[k + 1] = v.y;
        n.off[k + 2] = v.z;
        n.off[k + 3] = v.w;
      }
    } else {
      const uint2* o = reinterpret_cast<const uint2*>(r + 4 + dml);
#pragma unroll
      for (int k = 0; k < K; k += 2) {
        const uint2 v = o[k / 2];
        n.off[k] = v.x;
        n.off[k + 1] = v.y;
      }
    }
    const uint2 g0 = (DDB_TMEM_GPREFETCH && gvalid_)
                        ? gnext_
                        : *reinterpret_cast<const uint2*>(r + 4 + a.tile_dm + 2 * (dml / K));
    uint2 g = g0;
    if constexpr (DDB_TMEM_UNIFORM_G) {
      g.x = __shfl_sync(0xffffffffu, g.x, 0);
      g.y = __shfl_sync(0xffffffffu, g.y, 0);
    }
    // fast iff the window fits the columns this variant stages
    n.nv = g.x <= static_cast<uint32_t>((32 + kTail) / 4) ? g.x : 0u;
    n.base = w + col + g.y;  // w: the channel's 16-byte aligned row (kRowBase)
    const float* pa = n.base;
#ifdef DDB_CHECKED
    // the unconditional head reads (32 floats, or the predicated ones)
    chk.check(pa, kFullHead ? 4 * kHeadAlways : 4 * static_cast<int>(min(n.nv, 8u)));
    if (kFullHead && n.nv > static_cast<uint32_t>(kHeadAlways)) chk.check(pa, 32);
#endif
    if constexpr (kFullHead) {
      // head vectors unpredicated: columns past the window are never read
      // back, the slot's slack keeps the reads inside shared memory, and
      // unconditional definitions let the allocator retire the staging
      // registers between channels (predicated ones keep them live)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i >= kHeadAlways) {
          lds128_maybe(static_cast<uint32_t>(i) < n.nv, pa + 4 * i, n.win[4 * i],
                       n.win[4 * i + 1], n.win[4 * i + 2], n.win[4 * i + 3]);
          continue;
        }
        const float4 v = *reinterpret_cast<const float4*>(pa + 4 * i);
        n.win[4 * i] = v.x;
        n.win[4 * i + 1] = v.y;
        n.win[4 * i + 2] = v.z;
        n.win[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        lds128_maybe(static_cast<uint32_t>(i) < n.nv, pa + 4 * i, n.win[4 * i],
                     n.win[4 * i + 1], n.win[4 * i + 2], n.win[4 * i + 3]);
    }
    if constexpr (kTailEarly) {
#ifdef DDB_CHECKED
      if (n.nv > 8) chk.check(pa + 32, 4 * static_cast<int>(min(n.nv - 8u, 2u)));
#endif
#pragma unroll
      for (int i = 0; i < 2; ++i)
        lds128_maybe(n.nv > 8u + i, pa + 32 + 4 * i, n.tail[4 * i], n.tail[4 * i + 1],
                     n.tail[4 * i + 2], n.tail[4 * i + 3]);
    }
  }

  // Window -> this lane's TMEM row; afterwards n.win may be refilled.
  __device__ __forceinline__ void commit(Pre& n, uint32_t buf = 0) const {
    if (n.nv == 0) return;
    const uint32_t taddr = this->taddr + buf;
    if constexpr (DDB_TMEM_ST_SPLIT == 1) {
      // four x8 stores: each can issue as soon as its two 16-byte loads
      // have landed instead of one x32 store waiting for all eight
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_st8(taddr + 8 * q, n.win + 8 * q);
    } else if constexpr (DDB_TMEM_ST_SPLIT == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) tmem_st4(taddr + 4 * q, n.win + 4 * q);
    } else if constexpr (DDB_TMEM_ST_SPLIT == 3) {
#pragma unroll
      for (int q = 0; q < 2; ++q) tmem_st16(taddr + 16 * q, n.win + 16 * q);
    } else {
      tmem_st32(taddr, n.win);
    }
    if constexpr (kTailEarly) {
      if (DDB_TMEM_TAIL_ALWAYS || n.nv > 8) tmem_st8(taddr + 32, n.tail);
    } else if constexpr (kTail > 0) {
      // columns 32.. of the widest window (alignment + SPAN + W): an x8,
      // x16 or x32 store sized at compile time keeps the extra live
      // registers to what the variant can need
      if (n.nv > 8) {
        // reuse the head's registers once the x32 store has read them
        const float* pa = n.base + 32;
        float* hi = n.win;
#ifdef DDB_CHECKED
        chk.check(pa, 4 * static_cast<int>(min(n.nv - 8u, static_cast<uint32_t>(kTail / 4))));
#endif
        // nv > 8: the first tail vector is always needed
#pragma unroll
        for (int i = 0; i < kTail / 4; ++i)
          lds128_maybe(i == 0 || static_cast<uint32_t>(i) < n.nv - 8, pa + 4 * i, hi[4 * i],
                       hi[4 * i + 1], hi[4 * i + 2], hi[4 * i + 3]);
        if constexpr (kTail == 8) tmem_st8(taddr + 32, hi);
        else if constexpr (kTail == 16) tmem_st16(taddr + 32, hi);
        else tmem_st32(taddr + 32, hi);
      }
    }
    tmem_wait_st();
  }

  __device__ __forceinline__ void accumulate(const uint32_t (&off)[K], bool fast,
                                             const float* base, uint32_t buf = 0) {
    const uint32_t taddr = this->taddr + buf;
    if (fast) {
      // (ptxas schedules the loads itself: with the staging registers free
      // between channels it keeps 3-4 of them in flight).  G DMs' TMEM reads
      // per wait::ld (DDB_TMEM_GROUP, A/B builds).
      constexpr int G = (DDB_TMEM_GROUP <= K && K % DDB_TMEM_GROUP == 0) ? DDB_TMEM_GROUP : 2;
      // W = 12 read as one x16 (4 columns wasted: the window has the slack)
      // -- one TMEM address (R2UR) and one LDTM per DM instead of two
      constexpr bool kRead16 = DDB_TMEM_READ16 && W == 12 && SPAN + 3 + 16 <= COLS;
      constexpr int WB = kRead16 ? 16 : W;
#pragma unroll
      for (int k = 0; k < K; k += G) {
        float v[G][WB];
#pragma unroll
        for (int h = 0; h < G; ++h) {
          const uint32_t c = taddr + off[k + h];
          if constexpr (kRead16) {
            tmem_ld16(c, v[h]);
          } else if constexpr (W == 12 && DDB_TMEM_LD12) {
            tmem_ld12(c, v[h]);
          } else if constexpr (W == 20 && DDB_TMEM_LD20) {
            tmem_ld20(c, v[h]);
          } else {
#pragma unroll
            for (int j = 0; j + 8 <= W; j += 8) tmem_ld8(c + j, &v[h][j]);
            if constexpr (W % 8 == 4) tmem_ld4(c + (W - W % 8), &v[h][W - W % 8]);
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < G; ++h)
#pragma unroll
          for (int j = 0; j < W; j += 2) {
            const float2 s2 = fadd2(make_float2(acc[k + h][j], acc[k + h][j + 1]),
                                    make_float2(v[h][j], v[h][j + 1]));
            acc[k + h][j] = s2.x;
            acc[k + h][j + 1] = s2.y;
          }
      }
    } else {
      // slow path (a group with a DM below its first): k_plan's window
      // offsets are relative to the first DM's aligned start and wrap below
      // it, so they are applied as signed 32-bit displacements
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float* q = base + static_cast<int32_t>(off[k]);
        chk.check(q, W);
#pragma unroll
        for (int j = 0; j < W; ++j) acc[k][j] += q[j];
      }
    }
  }

  // Per channel: fetch (offsets + window from shared memory), commit
  // (window -> TMEM), accumulate (TMEM reads + FADD2).  A variant that
  // software-pipelined fetch(c+1) under accumulate(c) was measured 2x
  // slower: the extra live window registers spilled at the 168-register
  // cap that keeps two CTAs per SM.
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w) {
    Pre n;
    fetch(n, r, w);
    commit(n);
    accumulate(n.off, n.nv != 0, n.base);
  }
  // DDB_TMEM_GPREFETCH: the next channel's window geometry (its record's
  // group entry) is read before this channel's TMEM reads and adds, so the
  // next fetch starts with its window loads
  static constexpr bool kGroupPrefetch = DDB_TMEM_GPREFETCH != 0;
  uint2 gnext_ = make_uint2(0u, 0u);
  bool gvalid_ = false;
  __device__ __forceinline__ void channel(const uint32_t* r, const float* w, bool has_next) {
    Pre n;
    fetch(n, r, w);
    commit(n);
    gvalid_ = has_next;
    if (has_next)
      gnext_ = *reinterpret_cast<const uint2*>(r + a.rec_bytes / 4u + 4 + a.tile_dm +
                                               2 * (dml / K));
    accumulate(n.off, n.nv != 0, n.base);
  }
  // kStagePipe: the channels of one stage (fixed slots of win_cap floats),
  // two at a time -- fetch(c+1) | accumulate(c) | commit(c+1) -- alternating
  // between the two TMEM column blocks
  __device__ __forceinline__ void stage(const uint8_t* rbase, const float* wbase, uint32_t ncs) {
    const auto rec = [&](uint32_t cc) {
      return reinterpret_cast<const uint32_t*>(rbase + cc * a.rec_bytes);
    };
    Pre A, B;
    fetch(A, rec(0), wbase);
    commit(A, 0);
    for (uint32_t cc = 0; cc < ncs; cc += 2) {
      const bool more1 = cc + 1 < ncs, more2 = cc + 2 < ncs;
      if (more1) fetch(B, rec(cc + 1), wbase + (cc + 1) * a.win_cap);
      accumulate(A.off, A.nv != 0, A.base, 0);
      if (!more1) break;
      commit(B, COLS);
      if (more2) fetch(A, rec(cc + 2), wbase + (cc + 2) * a.win_cap);
      accumulate(B.off, B.nv != 0, B.base, COLS);
      if (more2) commit(A, 0);
    }
  }
  __device__ __forceinline__ void load(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* o = beam_out(a) + static_cast<uint64_t>(dm0 + dml + k) * a.out_pitch + t0 + col;
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = t0 + col + j < a.s ? o[j] : 0.0f;
    }
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      DDB_CHECK(dm0 + dml + k < a.num_dms);
      float* o = beam_out(a) + static_cast<uint64_t>(dm0 + dml + k) * a.out_pitch + t0 + col;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (t0 + col + j < a.s) o[j] = acc[k][j];
    }
  }
};

// TMEM columns per CTA: `cols` per consumer warp beyond the 4 lane
// quarters, rounded to the allocator's power of two (>= 32).
__device__ __forceinline__ uint32_t tmem_cols_for(uint32_t consumer_warps, uint32_t per_warp) {
  const uint32_t need = ((consumer_warps + 3) / 4) * per_warp;
  uint32_t cols = 32;
  while (cols < need) cols <<= 1;
  return cols;
}

template <int K, int W, int SPAN, int COLS, bool FULL_HEAD = true>
__device__ __forceinline__ void tmemwin_run(const TiledArgs& a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  const uint32_t consumers = blockDim.x / 32 - 1;
  using Body = TmemBody<K, W, SPAN, COLS, FULL_HEAD>;
  const uint32_t cols = tmem_cols_for(consumers, COLS * Body::kBufs);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(&tmem_base)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  staged_loop_with<Body>(a, smem, tmem_base);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(cols)
                 : "memory");
}

#if DDB_TMEM_LB2
template <int K, int W, int SPAN, int COLS>
__global__ void __maxnreg__(DDB_TMEM_LB2) k_tmemwin(const TiledArgs a) {
#else
template <int K, int W, int SPAN, int COLS>
__global__ void __launch_bounds__(288) k_tmemwin(const TiledArgs a) {
#endif
  tmemwin_run<K, W, SPAN, COLS>(a);
}

// Occupancy build for CTAs of <= 4 consumer warps + the producer: three CTAs
// per SM (<= 136 registers) instead of two.
template <int K, int W, int SPAN, int COLS>
__global__ void __launch_bounds__(160, 3) k_tmemwin_occ(const TiledArgs a) {
  tmemwin_run<K, W, SPAN, COLS, false>(a);  // predicated head: fewer live registers
}

// ---------------------------------------------------------------------
// K6: rectangles (staging "rect") for instances whose DM tiles span few
// samples per channel -- small d.  There the per-channel 1-D bulk copies of
// the staged family are tiny (T + span floats) and the CTA waits on one
// chunk's copies after another: copy count and latency, not bytes, set the
// time.  K6 stages a whole channel group per TMA operation instead: one
// 3-D tile load (samples x channels x beam) of the rectangle
// [t0 + lo_g, t0 + lo_g + rect_w) x [ch0, ch0 + rect_ch), lo_g the lowest
// shift of the group in the DM tile, so a stage is ONE copy of up to
// rect_ch x rect_w floats (rect_w <= 256, the TMA box limit), plus one bulk
// copy of the group's offsets.  The adds are K3's (SmemBody mapping: one
// shared-memory operand per add, channels ascending, one fp32 accumulator
// per output -- bit-exact).
// ---------------------------------------------------------------------
// K6 thread mapping: thread (it, id) owns times t0 + it + j*items_time
// (j < W) and the K CONSECUTIVE DMs id*K .. id*K+K-1 of the tile, so its
// per-channel offsets are one vector load (the output is mapping-invariant:
// every output still sums its channels in order into one accumulator).
template <int K>
__device__ __forceinline__ void load_offsets(const uint32_t* o, uint32_t (&v)[K]) {
  if constexpr (K % 4 == 0) {
#pragma unroll
    for (int k = 0; k < K; k += 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(o + k);
      v[k] = q.x;
      v[k + 1] = q.y;
      v[k + 2] = q.z;
      v[k + 3] = q.w;
    }
  } else if constexpr (K == 2) {
    const uint2 q = *reinterpret_cast<const uint2*>(o);
    v[0] = q.x;
    v[1] = q.y;
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = o[k];
  }
}

template <int K, int W, int IT>
struct RectBody {
  const TiledArgs& a;
  uint32_t it, id;
  float acc[K][W];
  __device__ __forceinline__ uint32_t stride() const { return IT > 0 ? IT : a.items_time; }
  __device__ RectBody(const TiledArgs& args) : a(args) {
    it = threadIdx.x % stride();
    id = threadIdx.x / stride();
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[k][j] = 0.0f;
  }
  // off: the channel's offsets (shift - lo_g) of the tile's DMs; row: this
  // thread's first sample in the channel's rectangle row
  __device__ __forceinline__ void channel(const uint32_t* off, const float* row) {
    uint32_t o[K];
    load_offsets<K>(off + id * K, o);
#pragma unroll
    for (int n = 0; n + 1 < K * W; n += 2) {
      const int k0 = n / W, j0 = n % W, k1 = (n + 1) / W, j1 = (n + 1) % W;
      const float2 r = fadd2(make_float2(acc[k0][j0], acc[k1][j1]),
                             make_float2(row[o[k0] + j0 * stride()], row[o[k1] + j1 * stride()]));
      acc[k0][j0] = r.x;
      acc[k1][j1] = r.y;
    }
    if ((K * W) & 1) acc[K - 1][W - 1] += row[o[K - 1] + (W - 1) * stride()];
  }
  __device__ __forceinline__ void load(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float* o = beam_out(a) + static_cast<uint64_t>(dm0 + id * K + k) * a.out_pitch + t0 + it;
#pragma unroll
      for (int j = 0; j < W; ++j)
        acc[k][j] = t0 + it + j * stride() < a.s ? o[j * stride()] : 0.0f;
    }
  }
  __device__ __forceinline__ void store(uint32_t dm0, uint32_t t0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      DDB_CHECK(dm0 + id * K + k < a.num_dms);
      float* o = beam_out(a) + static_cast<uint64_t>(dm0 + id * K + k) * a.out_pitch + t0 + it;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (t0 + it + j * stride() < a.s) o[j * stride()] = acc[k][j];
    }
  }
};

#ifndef DDB_RECT_PREFETCH
#define DDB_RECT_PREFETCH 0
#endif
// A/B switches, both off: measured within +-1 us at d=2..16 and mixed at
// d=64 (profiles/r02_ab_rect_lo.txt).  MIS_SMEM: the box misalignment handed
// to the consumers through shared memory (the producer already has it)
// instead of a global load of the group low per consumer thread and stage
#ifndef DDB_RECT_MIS_SMEM
#define DDB_RECT_MIS_SMEM 0
#endif
// the producer loads the next chunk's group low one chunk ahead, so the
// global load's latency overlaps its wait for the next free slot
#ifndef DDB_RECT_LO_AHEAD
#define DDB_RECT_LO_AHEAD 0
#endif

template <int K, int W, int IT>
__global__ void __launch_bounds__(1024 + 32) k_rect(const __grid_constant__ CUtensorMap tmap,
                                                    const TiledArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  __shared__ uint32_t mis_s[8];  // per slot: (t0 + lo_g) & 3 (nstage <= 8)
  // stage s: rect_ch x rect_w floats (128-byte aligned), then the offsets
  // (rec_bytes: a group's offsets, rect_ch x tile_dm u32 padded to 16 B)
  const uint32_t box_bytes = a.rect_ch * a.rect_w * 4u;
  const uint32_t stage_bytes = ((box_bytes + 127u) & ~127u) + ((a.rec_bytes + 127u) & ~127u);
  uint8_t* stages = smem + kPipeHeader;
  const uint32_t groups_dm = (a.tiles_dm + a.depth - 1) / a.depth;
  uint32_t t0, b_first;
  if (a.time_major) {
    t0 = (blockIdx.x % a.tiles_time) * a.tile_time;
    b_first = (blockIdx.x / a.tiles_time) * a.depth;
  } else {
    t0 = (blockIdx.x / groups_dm) * a.tile_time;
    b_first = (blockIdx.x % groups_dm) * a.depth;
  }
  const uint32_t ntiles = min(a.depth, a.tiles_dm - b_first);
  const uint32_t g_begin = a.ch_begin / a.rect_ch;
  const uint32_t g_end = (a.ch_end + a.rect_ch - 1) / a.rect_ch;
  const uint32_t nchunk = g_end - g_begin;
  const uint32_t total = ntiles * nchunk;
  const uint32_t consumers = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (uint32_t q = 0; q < a.nstage; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], consumers);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x >= consumers * 32) {  // producer warp: lane 0 issues
    if ((threadIdx.x & 31) != 0) return;
    const auto group_lo = [&](uint32_t g) {
      return __ldg(a.glo + (b_first + g / nchunk) * a.rect_groups + g_begin + g % nchunk);
    };
    uint32_t lo_next = (DDB_RECT_LO_AHEAD && total > 0) ? group_lo(0) : 0u;
    for (uint32_t g = 0; g < total; ++g) {
      const uint32_t slot = g % a.nstage, use = g / a.nstage;
      uint32_t lo;
      if constexpr (DDB_RECT_LO_AHEAD) {
        lo = lo_next;
        if (g + 1 < total) lo_next = group_lo(g + 1);
      } else {
        lo = 0u;
      }
      if (use > 0) mbar_wait_sleep(&empty[slot], (use - 1) & 1u);
      const uint32_t b = b_first + g / nchunk, grp = g_begin + g % nchunk;
      if constexpr (!DDB_RECT_LO_AHEAD) lo = __ldg(a.glo + b * a.rect_groups + grp);
      // the box starts at the 16-byte aligned sample at or below t0 + lo_g
      // (TMA tile loads fault on an unaligned row start); the consumers add
      // the misalignment back
      const uint32_t xs = t0 + lo;
      const int32_t x0 = static_cast<int32_t>(xs & ~3u);
      if constexpr (DDB_RECT_MIS_SMEM) mis_s[slot] = xs & 3u;  // published by the arrive below
      uint8_t* st = stages + slot * stage_bytes;
      uint64_t* bar = &full[slot];
      mbar_expect_tx(bar, box_bytes + a.rec_bytes);
      tma_load_3d(st, &tmap, x0, static_cast<int32_t>(grp * a.rect_ch),
                  static_cast<int32_t>(blockIdx.y), bar);
      if constexpr (DDB_RECT_PREFETCH > 0) {
        // warm L2 with the box DDB_RECT_PREFETCH chunks ahead
        const uint32_t gp = g + DDB_RECT_PREFETCH;
        if (gp < total) {
          const uint32_t bp = b_first + gp / nchunk, grpp = g_begin + gp % nchunk;
          const int32_t xp =
              static_cast<int32_t>((t0 + __ldg(a.glo + bp * a.rect_groups + grpp)) & ~3u);
          tma_prefetch_3d(&tmap, xp, static_cast<int32_t>(grpp * a.rect_ch),
                          static_cast<int32_t>(blockIdx.y));
        }
      }
      bulk_g2s(st + ((box_bytes + 127u) & ~127u),
               a.rec + (static_cast<uint64_t>(b) * a.rect_groups + grp) * a.rec_bytes, a.rec_bytes,
               bar);
      mbar_arrive(bar);
    }
    return;
  }
  const bool active = threadIdx.x < a.items_time * a.items_dm;
  RectBody<K, W, IT> body(a);
  for (uint32_t g = 0; g < total; ++g) {
    const uint32_t q = g % nchunk, slot = g % a.nstage;
    const uint32_t dm0 = (b_first + g / nchunk) * a.tile_dm;
    if (q == 0) {
      if (a.accumulate && active)
        body.load(dm0, t0);
      else
        body.zero();
    }
    consumer_wait(&full[slot], (g / a.nstage) & 1u);
    const uint8_t* st = stages + slot * stage_bytes;
    const uint32_t grp0 = g_begin + q;
    const uint32_t mis =
        DDB_RECT_MIS_SMEM ? mis_s[slot]
                          : ((t0 + __ldg(a.glo + (b_first + g / nchunk) * a.rect_groups + grp0)) & 3u);
    const float* rows = reinterpret_cast<const float*>(st) + mis;
    const uint32_t* offs = reinterpret_cast<const uint32_t*>(st + ((box_bytes + 127u) & ~127u));
    const uint32_t grp = grp0;
    // this launch's channels of the group (a channel-range pass may start or
    // end inside one)
    const uint32_t c_lo = max(a.ch_begin, grp * a.rect_ch) - grp * a.rect_ch;
    const uint32_t c_hi = min(a.ch_end, (grp + 1) * a.rect_ch) - grp * a.rect_ch;
    if (active) {
      // running pointers: the channel's offsets and this thread's first
      // sample of the channel's rectangle row
      const uint32_t* o = offs + c_lo * a.tile_dm;
      const float* r = rows + c_lo * a.rect_w + body.it;
      const uint32_t dof = a.tile_dm, drow = a.rect_w;
      uint32_t cc = c_lo;
      constexpr uint32_t U = K * W <= 8 ? 4 : 1;
      if constexpr (U > 1) {
        for (; cc + U <= c_hi; cc += U) {
#pragma unroll
          for (uint32_t u = 0; u < U; ++u) body.channel(o + u * dof, r + u * drow);
          o += U * dof;
          r += U * drow;
        }
      }
      for (; cc < c_hi; ++cc, o += dof, r += drow) body.channel(o, r);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[slot]);
    if (active && q == nchunk - 1) body.store(dm0, t0);
  }
}

using RectFn = void (*)(const CUtensorMap, const TiledArgs);

struct RectVariant {
  int k, w, it;
  RectFn fn;
};
#define DDB_RV(K, W, I) {K, W, I, k_rect<K, W, I>}
static const RectVariant kRectVariants[] = {
    DDB_RV(1, 1, 0), DDB_RV(1, 2, 0), DDB_RV(1, 4, 0), DDB_RV(2, 1, 0), DDB_RV(2, 2, 0),
    DDB_RV(2, 4, 0), DDB_RV(4, 1, 0), DDB_RV(4, 2, 0), DDB_RV(4, 4, 0), DDB_RV(8, 1, 0),
    DDB_RV(8, 2, 0), DDB_RV(8, 4, 0), DDB_RV(16, 1, 0), DDB_RV(16, 2, 0),
    // compile-time items_time (immediate strides) for the shapes small-d
    // sweeps pick
    DDB_RV(2, 1, 32), DDB_RV(2, 1, 64), DDB_RV(2, 1, 96), DDB_RV(2, 1, 128), DDB_RV(4, 1, 32),
    DDB_RV(4, 1, 64), DDB_RV(2, 2, 64), DDB_RV(8, 1, 32), DDB_RV(4, 2, 32),
};
#undef DDB_RV

RectFn find_rect_kernel(uint32_t k, uint32_t w, uint32_t items_time) {
  const RectVariant* generic = nullptr;
  for (const RectVariant& v : kRectVariants) {
    if (static_cast<uint32_t>(v.k) != k || static_cast<uint32_t>(v.w) != w) continue;
    if (v.it == 0 && generic == nullptr) generic = &v;
    if (items_time != 0 && static_cast<uint32_t>(v.it) == items_time) return v.fn;
  }
  return generic ? generic->fn : nullptr;
}

// ------------------------------------------------------------ dispatch --
using KernelFn = void (*)(const TiledArgs);

struct SmemVariant {
  int k, w, it;  // it = 0: items_time at run time
  KernelFn fn;
  int max_threads;
  KernelFn fn_packed;  // packed-stage build (DD_CONFIG_PACKED_STAGES); nullptr if none
};

#define DDB_V(K, W) {K, W, 0, k_smem<K, W>, smem_max_threads<K, W>(), nullptr}
#define DDB_VI(K, W, I) {K, W, I, k_smem<K, W, I>, smem_max_threads<K, W>(), nullptr}
#define DDB_VP(K, W, I) \
  {K, W, I, k_smem<K, W, I>, smem_max_threads<K, W>(), k_smem<K, W, I, true>}
#define DDB_VPT(K, W, I, MT) \
  {K, W, I, k_smem<K, W, I, false, MT>, MT, k_smem<K, W, I, true, MT>}
static const SmemVariant kSmemVariants[] = {
    DDB_V(1, 1),  DDB_V(1, 2),  DDB_V(1, 4),  DDB_V(1, 5),  DDB_V(1, 8),  DDB_V(1, 10),
    DDB_V(1, 16), DDB_V(1, 25), DDB_V(2, 1),  DDB_V(2, 2),  DDB_V(2, 4),  DDB_V(2, 5),
    DDB_V(2, 8),  DDB_V(2, 10), DDB_V(2, 16), DDB_V(2, 25), DDB_V(4, 1),  DDB_V(4, 2),
    DDB_V(4, 4),  DDB_V(4, 5),  DDB_V(4, 8),  DDB_V(4, 10), DDB_V(4, 16), DDB_V(8, 1),
    DDB_V(8, 2),  DDB_V(8, 4),  DDB_V(8, 5),  DDB_V(8, 8),  DDB_V(16, 1), DDB_V(16, 2),
    DDB_V(16, 4),
    // compile-time items_time for the shapes the sweeps select (tuning/)
    // (and packed-stage builds for the large-delay (LOFAR) shapes)
    DDB_VI(1, 5, 32), DDB_VI(2, 5, 32), DDB_VI(4, 5, 32), DDB_VI(1, 25, 8), DDB_VI(4, 10, 16),
    DDB_VP(2, 5, 160), DDB_VP(1, 25, 64), DDB_VP(2, 25, 64), DDB_VP(4, 10, 160),
    DDB_VP(2, 10, 160), DDB_VP(2, 25, 160),
    // (longer / taller LOFAR tiles -- (160,1,20,4), (160,2,10,4), (160,2,20,4)
    // -- stage fewer bytes per add but fit fewer channels per stage and
    // spill: 4.98-6.47 ms against 4.72 ms, measured round 2; not built)
};
#undef DDB_V
#undef DDB_VI
#undef DDB_VP
#undef DDB_VPT

KernelFn find_smem_kernel(uint32_t k, uint32_t w, uint32_t* max_threads, uint32_t items_time,
                          KernelFn* packed) {
  const SmemVariant* generic = nullptr;
  if (packed) *packed = nullptr;
  for (const SmemVariant& v : kSmemVariants) {
    if (static_cast<uint32_t>(v.k) != k || static_cast<uint32_t>(v.w) != w) continue;
    if (v.it == 0 && generic == nullptr) generic = &v;
    if (items_time != 0 && static_cast<uint32_t>(v.it) == items_time) {
      if (max_threads) *max_threads = static_cast<uint32_t>(v.max_threads);
      if (packed) *packed = v.fn_packed;
      return v.fn;
    }
  }
  if (generic == nullptr) return nullptr;
  if (max_threads) *max_threads = static_cast<uint32_t>(generic->max_threads);
  return generic->fn;
}

struct RegWinVariant {
  int k, w, span;
  KernelFn fn;
};

#define DDB_R(K, W, S) {K, W, S, k_regwin<K, W, S>}
static const RegWinVariant kRegWinVariants[] = {
    // scalar windows (W odd: the reference-divisible Apertif/LOFAR shapes)
    DDB_R(2, 25, 4),  DDB_R(2, 25, 8),  DDB_R(2, 25, 16), DDB_R(4, 25, 12), DDB_R(4, 25, 16),
    DDB_R(8, 5, 31),
    // vector windows (W % 4 == 0, W/4 odd; GPU tiling)
    DDB_R(2, 20, 4),  DDB_R(2, 20, 8),  DDB_R(4, 20, 12), DDB_R(4, 20, 16), DDB_R(4, 12, 12),
    DDB_R(4, 12, 16), DDB_R(8, 12, 24), DDB_R(8, 12, 28), DDB_R(2, 12, 8),
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

struct TmemVariant {
  int k, w, span;
  KernelFn fn;
  KernelFn fn_occ;  // <= 160 threads, 3 CTAs/SM; nullptr when not built
};

#define DDB_T(K, W, S, C) {K, W, S, k_tmemwin<K, W, S, C>, nullptr}
#define DDB_TO(K, W, S, C) {K, W, S, k_tmemwin<K, W, S, C>, k_tmemwin_occ<K, W, S, C>}
static const TmemVariant kTmemVariants[] = {
    DDB_T(2, 12, 8, 32),  DDB_TO(4, 12, 12, 32), DDB_T(4, 12, 16, 32),
    DDB_T(8, 12, 24, 64), DDB_T(8, 12, 32, 64), DDB_T(2, 20, 8, 32),  DDB_T(4, 20, 8, 32),
    DDB_T(4, 20, 24, 64),
    DDB_T(8, 8, 32, 64),  DDB_T(16, 4, 48, 64),  DDB_TO(8, 4, 24, 32), DDB_TO(4, 4, 8, 32),
    DDB_TO(4, 8, 12, 32),
};
#undef DDB_T
#undef DDB_TO

KernelFn find_tmem_kernel(uint32_t k, uint32_t w, uint32_t group_span, uint32_t* span_out,
                          bool occ) {
  const TmemVariant* cover = nullptr;
  const TmemVariant* widest = nullptr;
  for (const TmemVariant& v : kTmemVariants) {
    if (static_cast<uint32_t>(v.k) != k || static_cast<uint32_t>(v.w) != w) continue;
    if (occ && v.fn_occ == nullptr) continue;
    if (widest == nullptr || v.span > widest->span) widest = &v;
    if (static_cast<uint32_t>(v.span) >= group_span && (cover == nullptr || v.span < cover->span))
      cover = &v;
  }
  const TmemVariant* pick = cover ? cover : widest;
  if (pick == nullptr) return nullptr;
  if (span_out) *span_out = static_cast<uint32_t>(pick->span);
  return occ ? pick->fn_occ : pick->fn;
}

bool tmem_shape_ok(uint32_t k, uint32_t w, uint32_t items_time, uint64_t block) {
  if (items_time % 32 != 0 || block > 256) return false;
  for (const TmemVariant& v : kTmemVariants)
    if (static_cast<uint32_t>(v.k) == k && static_cast<uint32_t>(v.w) == w) return true;
  return false;
}

bool tmem_has_occupancy_build(uint32_t k, uint32_t w) {
  for (const TmemVariant& v : kTmemVariants)
    if (static_cast<uint32_t>(v.k) == k && static_cast<uint32_t>(v.w) == w && v.fn_occ) return true;
  return false;
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
                        uint32_t smem, cudaStream_t st, uint32_t beams) {
  fn<<<dim3(blocks, beams), threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t debug_violations(unsigned long long* count, int* checked, int reset) {
#ifdef DDB_CHECKED
  *checked = 1;
  cudaError_t e = cudaMemcpyFromSymbol(count, g_ddb_violations, sizeof(*count));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_ddb_violations, &zero, sizeof(zero));
  }
  return e;
#else
  (void)reset;
  *checked = 0;
  *count = 0;
  return cudaSuccess;
#endif
}

cudaError_t prepare_smem(KernelFn fn, uint32_t smem) {
  // The attribute belongs to the function (per device), not to a plan: it
  // is only ever raised, so a plan created later with a smaller shared-memory
  // footprint cannot invalidate the launches of a live plan using the same
  // kernel with a larger one.
  static std::mutex mu;
  static std::map<std::pair<int, KernelFn>, uint32_t> raised;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  uint32_t& cur = raised[{dev, fn}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
  if (e == cudaSuccess) cur = smem;
  // The staged kernels never read through L1 (TMA fills shared memory,
  // outputs are streaming stores): ask for the whole unified array as
  // shared memory so the register budget, not the carveout, sets the
  // resident CTAs per SM.
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  return e;
}

cudaError_t launch_rect(RectFn fn, const CUtensorMap& tmap, const TiledArgs& a, uint32_t blocks,
                        uint32_t threads, uint32_t smem, cudaStream_t st, uint32_t beams) {
  fn<<<dim3(blocks, beams), threads, smem, st>>>(tmap, a);
  return cudaGetLastError();
}

cudaError_t prepare_rect(RectFn fn, uint32_t smem) {
  return prepare_smem(reinterpret_cast<KernelFn>(fn), smem);
}

}  // namespace ddb
