// common.cuh -- shared device helpers and launch descriptors for the
// sm_100a dedispersion kernels.  Inline PTX only (no CUTLASS/CuTe needed:
// the hot path uses 1-D bulk copies, not tensor maps).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ddb {

// ------------------------------------------------------- checked builds --
// DDB_CHECKED (build.py build(checked=True) -> libdedisp_b200_checked.so):
// every shared-memory window read, bulk-copy source/destination and output
// store of the staged kernels is bounds-checked on the device and a
// violation counted (dd_debug_violations).  The pool's GPUs do not allow
// compute-sanitizer, so this is the memcheck of the hot path
// (tools/sanitize_cases.py, tests/test_gpu_checked.py).
#ifdef DDB_CHECKED
// one counter per translation unit; the staged kernels and its reader
// (debug_violations) live in dedisp.cu
static __device__ unsigned long long g_ddb_violations = 0;
__device__ __forceinline__ void ddb_check(bool ok) {
  if (!ok) atomicAdd(&g_ddb_violations, 1ull);
}
#define DDB_CHECK(cond) ::ddb::ddb_check(static_cast<bool>(cond))
#else
#define DDB_CHECK(cond) ((void)0)
#endif

// ----------------------------------------------------------------- PTX --
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

// Make mbarrier initialisation visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Raise the phase's expected transaction bytes without arriving.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

// Plain arrival (release, CTA scope): a consumer warp hands a slot back.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// 16-byte shared load under a predicate, the destination's previous value
// declared dead: with the predicate off the registers hold unspecified
// values (for staging buffers whose unloaded tail is never read).
__device__ __forceinline__ void lds128_maybe(bool pred, const float* addr, float& x, float& y,
                                             float& z, float& w) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
      : "=f"(x), "=f"(y), "=f"(z), "=f"(w)
      : "r"(smem_addr(addr)), "r"(static_cast<int>(pred)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Producer-side wait: try_wait with a suspend-time hint parks the lane in
// hardware until the phase completes (or the hint expires) instead of
// polling, so the waiting producer does not steal issue slots from the
// consumer warps of its scheduler.
#ifndef DDB_PRODUCER_SLEEP_NS
#define DDB_PRODUCER_SLEEP_NS 0
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  if constexpr (DDB_PRODUCER_SLEEP_NS > 0) {
    // A/B: poll, then a plain timed sleep between polls
    while (!mbar_try_wait(bar, parity)) __nanosleep(DDB_PRODUCER_SLEEP_NS);
    return;
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` in bytes.
// dst/src 16-byte aligned, bytes a multiple of 16 (SASS: UBLKCP.S.G).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// 3-D TMA tile load global -> shared (SASS: UTMALDG), completion counted on
// `bar` in bytes; coordinates are signed element indices, out-of-range
// elements are zero-filled.  `tmap` is the generic address of a
// __grid_constant__ CUtensorMap kernel parameter.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}

// L2 prefetch of a 3-D TMA tile (no shared memory, no completion): lets a
// producer reach further ahead into HBM than its shared-memory stages hold.
__device__ __forceinline__ void tma_prefetch_3d(const void* tmap, int32_t c0, int32_t c1,
                                                int32_t c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tmap),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// Two IEEE round-to-nearest fp32 adds in one instruction (SASS: FADD2).
// Each lane is an independent correctly-rounded add, so the per-output
// accumulation order (and hence bit-exactness) is unchanged.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rr;\n\t"
      "mov.b64 ra, {%2, %3};\n\t"
      "mov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rr, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rr;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// ------------------------------------------------------------ launches --
// Per-(DM tile, channel) plan record, produced by k_plan (table.cu) and
// staged into shared memory next to the channel's window:
//   u32 lo, u32 span (= hi - lo), u32 pad[2], u32 off[tile_dm] (= shift - lo)
// padded to a multiple of 16 bytes.  The min/max scan is the reference's
// kernels.cpp:147-156, done once per (table, tile_dm) instead of per tile.
struct PlanRec {
  uint32_t lo;
  uint32_t span;
  uint32_t pad0, pad1;
};

// ... followed by one u32 per aligned group of `group` DMs: the spread of
// the group's offsets above its FIRST DM (0xffffffff when a later DM sits
// below it) -- the register/TMEM-window kernels' fast-path test, precomputed.
__host__ __device__ inline uint32_t plan_rec_bytes(uint32_t tile_dm, uint32_t group = 1) {
  const uint32_t groups = (tile_dm + group - 1) / group;
  return ((16u + 4u * tile_dm + 8u * groups) + 15u) & ~15u;
}

// Channels per pipeline stage: 1..kMaxCps (DD_CONFIG_CPS_* holds 1..15).
constexpr uint32_t kMaxCps = 16;
// Staged-kernel shared-memory header: full[8] and empty[8] mbarriers;
// records and windows follow.
constexpr uint32_t kPipeHeader = 128;

struct TiledArgs {
  const float* in;
  uint64_t in_pitch;  // floats, multiple of 4 for the staged families
  const uint8_t* rec; // [tiles_dm][channels] records, rec_bytes each
  const uint2* ls;    // [tiles_dm][channels] (lo, span), compact copy for the producer
  const uint32_t* shifts;  // DM-major table (direct family)
  float* out;
  uint64_t out_pitch;  // floats
  uint32_t channels, s, num_dms;
  uint32_t items_time, items_dm, work_time, work_dm;
  uint32_t tile_time, tile_dm, tiles_time, tiles_dm;
  uint32_t depth;      // DM tiles per CTA
  uint32_t time_major; // staged families: CTA raster time-fastest (else DM-fastest)
  uint32_t win_cap;    // floats per staged channel window (multiple of 4)
  uint32_t rec_bytes;
  uint32_t cps;        // channels per pipeline stage
  uint32_t nstage;
  uint32_t pack;       // tiles per CTA (direct family)
  uint32_t vthreads;   // virtual threads per CTA (direct family)
  // staged families: channel range of this launch; accumulate = 1 starts
  // every output from its current value in `out` instead of 0.0f (a pass
  // split by channel ranges then reproduces the single pass bit for bit:
  // the running fp32 sum round-trips through memory exactly)
  uint32_t ch_begin, ch_end, accumulate;
  // packed stages (DD_CONFIG_PACKED_STAGES, full channel range): stage q
  // holds channels [stage_ch[q], stage_ch[q+1]) and channel c's window sits
  // chan_off[c] floats into its stage buffer -- each channel takes its own
  // window width instead of the widest, so wide-delay instances fit more
  // channels per stage.  Otherwise stage q is cps channels of win_cap floats.
  const uint32_t* stage_ch;
  const uint32_t* chan_off;
  uint32_t packed, packed_stages;
  uint32_t stage_floats;  // floats per stage buffer (cps * win_cap unless packed)
  // staged families: independent beams (grid.y), each with its own input
  // block and output rows at these strides (floats) -- the deployment's
  // many-beams-per-GPU batching
  uint64_t in_beam_stride, out_beam_stride;
  // rectangle family (K6, small spans): per stage one TMA box of rect_ch
  // channels x rect_w samples starting at t0 + glo[dm tile][group]; plan
  // records hold, per channel, every DM's offset from the group's lo
  const uint32_t* glo;  // [tiles_dm][groups] lowest shift of the group
  uint32_t rect_w, rect_ch, rect_groups;
};

}  // namespace ddb
