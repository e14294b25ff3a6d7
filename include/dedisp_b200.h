/*
 * dedisp_b200.h -- the C-ABI boundary of the B200 dedispersion hot path.
 *
 * Plain C types only (no CUDA or torch types in any signature).  Every entry
 * point returns a dd_status; dd_last_error() gives the thread's last message.
 * The reference (/root/reference/proj/core, C++20) has no C ABI of its own;
 * each entry below names the reference function it stands in for, so the
 * reference's C++ API can be re-implemented over this layer
 * (include/dedisp/b200.hpp does exactly that; INTEGRATION.md shows the shim
 * a maintainer would add on the reference side).
 *
 * Status mapping (reference error conventions):
 *   DD_ERR_INVALID_ARGUMENT  <-> std::invalid_argument
 *                                (kernels.cpp:16-28, :58-81; setup.cpp:31-62)
 *   DD_ERR_CAPACITY          <-> dedisp::capacity_error (errors.hpp:10-13)
 *   DD_ERR_CUDA / NO_DEVICE  <-> std::runtime_error (device failure; the
 *                                reference has no device, so no analogue)
 *
 * Layouts (identical to the reference):
 *   filterbank  float32 [channels][num_samples] channel-major
 *               (filterbank.hpp:15-26); on the device rows may be padded to
 *               a pitch (in floats) -- the fast kernels need pitch % 4 == 0.
 *   shifts      uint32  [num_dms][channels] DM-major (setup.hpp:39-51)
 *   output      float32 [num_dms][samples_per_second] DM-major
 *               (kernels.hpp:16-27), optionally with a row pitch.
 *
 * Threading: a dd_context belongs to one device and one stream; calls on
 * one context must be serialised by the caller (one context per thread or a
 * lock), exactly like the reference's borrowed ThreadPool (kernels.hpp:66-71).
 */
#ifndef DEDISP_B200_H
#define DEDISP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DD_ABI_VERSION 1

typedef enum dd_status {
  DD_OK = 0,
  DD_ERR_INVALID_ARGUMENT = 1,
  DD_ERR_CAPACITY = 2,
  DD_ERR_CUDA = 3,
  DD_ERR_NO_DEVICE = 4,
  DD_ERR_INTERNAL = 5
} dd_status;

/* ObservationSetup minus its name (setup.hpp:14-33). */
typedef struct dd_setup {
  uint32_t samples_per_second;
  uint32_t channels;
  double f_min;         /* MHz, centre of channel 0 */
  double channel_width; /* MHz */
  double dm_first;      /* pc/cm^3 */
  double dm_step;       /* pc/cm^3 */
} dd_setup;

/* Input-staging strategy of a tiled launch (the paper's "local memory or
 * rely on the cache"). */
typedef enum dd_staging {
  DD_STAGING_AUTO = 0,   /* fastest kernel family that supports the config */
  DD_STAGING_SMEM = 1,   /* per-channel windows staged by TMA bulk copies   */
  DD_STAGING_DIRECT = 2, /* loads straight from global through L1/L2       */
  DD_STAGING_REGWIN = 3, /* TMA-staged windows + per-thread register window */
  DD_STAGING_TMEM = 4,   /* TMA-staged windows + per-lane TMEM windows (tcgen05) */
  DD_STAGING_RECT = 5    /* one 3-D TMA box per channel group (small spans: small d);
                            channels per stage = 16 x DD_CONFIG_CPS (0: plan's choice) */
} dd_staging;

/* KernelConfig (kernels.hpp:40-52) plus the two GPU knobs of the north star:
 * dm_tile_depth = DM tiles one CTA walks in sequence (0 or 1 = one), and the
 * staging strategy; `flags` selects GPU-only relaxations. */
typedef struct dd_config {
  uint32_t items_time;
  uint32_t items_dm;
  uint32_t work_time;
  uint32_t work_dm;
  uint32_t dm_tile_depth;
  uint32_t staging; /* dd_staging */
  uint32_t flags;   /* DD_CONFIG_* */
} dd_config;

/* GPU tiling: tile_time (items_time*work_time) need not divide s -- the
 * last time tile is predicated.  Only the staged families accept it; the
 * reference-compatible entry points (dd_validate_config without the flag,
 * dd_dedisperse) keep the reference's exact-division rule. */
#define DD_CONFIG_GPU_TILING 0x1u
/* TMEM windows: use the three-CTAs-per-SM build (<= 128 registers,
 * <= 4 consumer warps per CTA) when one exists for the shape; otherwise the
 * flag is ignored.  A tuning knob: occupancy against register pressure. */
#define DD_CONFIG_HIGH_OCCUPANCY 0x2u
/* Staged families: order the CTAs time-fastest instead of DM-fastest.  With
 * large delays (LOFAR) DM-fastest resident CTAs read windows spread over the
 * whole input block, which then streams from HBM once per time tile;
 * time-fastest keeps the resident working set to one DM group's region. */
#define DD_CONFIG_TIME_MAJOR 0x8u
/* Staged families: pack each stage with as many channels as their own
 * windows fit (instead of slots sized for the widest window), for
 * instances whose delay spread varies across the band (LOFAR).  Full
 * channel-range passes only; channel-range passes use fixed slots. */
#define DD_CONFIG_PACKED_STAGES 0x10u
/* Staged families: channels per pipeline stage in bits 8..11 (1..15; 0 lets
 * the plan choose).  A tuning knob: larger stages amortise the per-stage
 * synchronisation, smaller ones leave shared memory for more CTAs per SM. */
#define DD_CONFIG_CPS_SHIFT 8u
#define DD_CONFIG_CPS_MASK (0xfu << DD_CONFIG_CPS_SHIFT)
/* Fixed-slot staged families: twice the DD_CONFIG_CPS channels per stage
 * (up to 30; stages that wide amortise the per-stage synchronisation
 * further where shared memory allows). */
#define DD_CONFIG_WIDE_STAGES 0x20u
/* Staged families: pipeline depth (stages in flight) in bits 12..15 (2..8;
 * 0 lets the plan choose).  A tuning knob like the stage width. */
#define DD_CONFIG_NSTAGE_SHIFT 12u
#define DD_CONFIG_NSTAGE_MASK (0xfu << DD_CONFIG_NSTAGE_SHIFT)

/* KernelLimits (kernels.hpp:31-34); {0,0} means the reference defaults
 * {1024, 256}. */
typedef struct dd_limits {
  uint32_t max_block_items;
  uint32_t max_accumulators;
} dd_limits;

typedef struct dd_context dd_context;
typedef struct dd_plan dd_plan;

/* ---------------------------------------------------------------- misc */
const char* dd_last_error(void);
int dd_abi_version(void);
dd_status dd_device_count(int* count);

/* ------------------------------------------------ contexts and streams */
/* One context per device.  It owns a non-blocking stream unless
 * dd_context_set_stream() hands it a caller stream (a cudaStream_t passed
 * as void*).  Replaces the reference's ThreadPool (thread_pool.hpp:15-42). */
dd_status dd_context_create(int device, dd_context** out);
dd_status dd_context_destroy(dd_context* ctx);
dd_status dd_context_set_stream(dd_context* ctx, void* stream);
void* dd_context_stream(dd_context* ctx);
dd_status dd_context_synchronize(dd_context* ctx);
dd_status dd_context_device_info(dd_context* ctx, int* sm_count, int* smem_optin_bytes,
                                 int* cc_major, int* cc_minor);

/* -------------------------------------------------------------- memory */
dd_status dd_device_malloc(dd_context* ctx, uint64_t bytes, void** ptr);
dd_status dd_device_free(dd_context* ctx, void* ptr);
dd_status dd_host_malloc(uint64_t bytes, void** ptr); /* page-locked */
dd_status dd_host_free(void* ptr);
/* Asynchronous on the context stream. */
dd_status dd_copy_h2d(dd_context* ctx, void* dst, const void* src, uint64_t bytes);
dd_status dd_copy_d2h(dd_context* ctx, void* dst, const void* src, uint64_t bytes);
/* Upload a channel-major filterbank into a pitched device buffer
 * (dst_pitch >= num_samples floats). */
dd_status dd_upload_filterbank(dd_context* ctx, float* d_dst, uint64_t dst_pitch,
                               const float* h_src, uint32_t channels, uint64_t num_samples);

/* ---------------------------------------- L0 geometry (setup.cpp) ---- */
/* ObservationSetup::validate, setup.cpp:31-46 */
dd_status dd_setup_validate(const dd_setup* setup);
/* delay_seconds, setup.cpp:48-62 (Eq. 1, FP64, k = 4150) */
dd_status dd_delay_seconds(double dm, double f_channel_mhz, double f_highest_mhz, double* out);
/* instance_sizing, setup.cpp:112-137 */
dd_status dd_instance_sizing(const dd_setup* setup, uint32_t num_dms, uint64_t* num_samples,
                             uint64_t* flop, uint32_t* max_delay);

/* ---------------------------------------------- K1: shift table ------- */
/* build_delay_table / build_zero_delay_table (setup.cpp:86-110) computed on
 * the device in FP64: rows [dm_offset, dm_offset+num_dms) of the full table
 * are written to d_shifts (uint32 [num_dms][channels]).  max_delay (host
 * pointer, may be NULL) receives the slice maximum; that read synchronises
 * the stream.  Used directly by the DM-sharded multi-GPU driver. */
dd_status dd_delay_table_device(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                                uint32_t dm_offset, int zero, uint32_t* d_shifts,
                                uint32_t* max_delay);
/* Host-buffer drop-in for build_delay_table (setup.hpp:75-81): honours the
 * memory cap (capacity error) and returns the full table in h_shifts. */
dd_status dd_build_delay_table(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                               uint64_t memory_cap_bytes, int zero, uint32_t* h_shifts,
                               uint32_t* max_delay);

/* ------------------------------------ L1 configs (kernels.cpp:44-81) -- */
int dd_config_valid(const dd_config* cfg, uint32_t num_dms, uint32_t samples_per_second,
                    const dd_limits* limits);
dd_status dd_validate_config(const dd_config* cfg, uint32_t num_dms,
                             uint32_t samples_per_second, const dd_limits* limits);
/* Whether a device kernel family supports cfg for this instance, and which
 * (resolves DD_STAGING_AUTO).  Returns DD_OK with *family = dd_staging. */
dd_status dd_config_family(dd_context* ctx, const dd_config* cfg, uint32_t channels,
                           uint32_t num_dms, uint32_t samples_per_second, uint32_t max_span,
                           uint32_t* family);
/* count_loads, count_loads.cpp:9-68 (host arithmetic over a host table).
 * With DD_CONFIG_GPU_TILING in cfg->flags the predicated last time tile is
 * counted like a full tile (what the staging producer copies). */
dd_status dd_count_loads(const uint32_t* h_shifts, uint32_t channels, uint32_t num_dms,
                         uint32_t samples_per_second, const dd_config* cfg, uint64_t* staged,
                         uint64_t* ideal);

/* -------------------------------------- K2/K3: dedispersion plans ----- */
/* A plan binds a device shift table and a config to a kernel launch: it
 * validates (never silently falls back: an explicit staging the config cannot
 * use is DD_ERR_INVALID_ARGUMENT), runs the per-(DM tile, channel) lo/hi
 * pre-pass (the min/max scan of kernels.cpp:147-156, done once per table),
 * sizes shared memory and picks the launch.  cfg == NULL selects the
 * reference-order kernel (dedisperse_reference_into, kernels.cpp:83-108):
 * one thread per output.  Creation synchronises the context stream once. */
dd_status dd_plan_create(dd_context* ctx, const uint32_t* d_shifts, uint32_t channels,
                         uint32_t num_dms, uint32_t samples_per_second, uint64_t num_samples,
                         uint64_t in_pitch, const dd_config* cfg, const dd_limits* limits,
                         dd_plan** out);
dd_status dd_plan_destroy(dd_plan* plan);

typedef struct dd_plan_info {
  uint32_t family;        /* dd_staging actually used */
  uint32_t max_span;      /* max over (DM tile, channel) of hi - lo */
  uint32_t max_delay;     /* max shift in the table */
  uint32_t grid_x, grid_y, block_threads;
  uint32_t smem_bytes;    /* dynamic shared memory per CTA */
  uint32_t channels_per_stage, stages;
  uint32_t kernel_launches; /* launches per dd_plan_execute */
  uint64_t staged_bytes;  /* L2->SMEM bytes per execute (0 for direct) */
  uint32_t registers;     /* per thread, of the tiled kernel (0 otherwise) */
  uint32_t ctas_per_sm;   /* resident CTAs per SM by the occupancy API (0 if not
                           * staged); conservative for the tcgen05 (TMEM) kernels,
                           * which it reports as 1 while two run (ncu: ~10 warps/SM) */
  uint32_t time_major;    /* CTA raster time-fastest (DD_CONFIG_TIME_MAJOR or AUTO's pick) */
  uint32_t packed_stages; /* stages per tile when packed (DD_CONFIG_PACKED_STAGES), else 0 */
} dd_plan_info;
dd_status dd_plan_get_info(const dd_plan* plan, dd_plan_info* info);

/* Launch on the context stream, asynchronously: out[dm][j] (row pitch
 * out_pitch floats, >= samples_per_second) = sum over ch ascending of
 * in[ch][j + shift[dm][ch]], one fp32 accumulator from 0.0f per output --
 * bit-identical to dedisperse_reference for every config. */
dd_status dd_plan_execute(dd_plan* plan, const float* d_in, float* d_out, uint64_t out_pitch);

/* Staged families only: run channels [ch_begin, ch_end) of the pass.
 * accumulate = 0 starts every output at 0.0f, 1 continues from the values
 * already in d_out.  Splitting a pass into ascending channel ranges
 * (first with accumulate = 0) is bit-identical to one dd_plan_execute -- the
 * per-output fp32 running sum round-trips through memory exactly -- which
 * lets the input block stream in by channel ranges under the compute. */
dd_status dd_plan_execute_channels(dd_plan* plan, const float* d_in, float* d_out,
                                   uint64_t out_pitch, uint32_t ch_begin, uint32_t ch_end,
                                   int accumulate);

/* Staged families only: `beams` independent beams in one launch (grid.y),
 * beam b reading d_in + b*in_beam_stride (a [channels][in_pitch] block) and
 * writing d_out + b*out_beam_stride (rows of out_pitch), all with this plan's
 * shift table -- many beams per device. */
dd_status dd_plan_execute_beams(dd_plan* plan, uint32_t beams, const float* d_in,
                                uint64_t in_beam_stride, float* d_out, uint64_t out_pitch,
                                uint64_t out_beam_stride);

/* Time `repeats` executions with CUDA events on the context stream after
 * `warmup` untimed ones (benchmark_config, tuner.cpp:136-170).  seconds[i]
 * receives each run. */
dd_status dd_plan_time(dd_plan* plan, const float* d_in, float* d_out, uint64_t out_pitch,
                       uint32_t warmup, uint32_t repeats, double* seconds);
/* As dd_plan_time; flush_l2 = 1 overwrites a context buffer of twice the
 * L2 size before every timed run, outside the events (cold-L2 timing). */
dd_status dd_plan_time_ex(dd_plan* plan, const float* d_in, float* d_out, uint64_t out_pitch,
                          uint32_t warmup, uint32_t repeats, int flush_l2, double* seconds);

/* One-shot device-buffer dedispersion: plan + execute + destroy. */
dd_status dd_dedisperse_device(dd_context* ctx, const float* d_in, uint32_t channels,
                               uint64_t num_samples, uint64_t in_pitch,
                               const uint32_t* d_shifts, uint32_t num_dms,
                               uint32_t samples_per_second, const dd_config* cfg,
                               const dd_limits* limits, float* d_out);

/* Host-buffer drop-in for dedisperse_reference_into (cfg == NULL,
 * kernels.cpp:83-108) and dedisperse_tiled_into (kernels.cpp:117-206):
 * checks the pair (kernels.cpp:16-28), validates cfg against the reference
 * limits, uploads, runs, downloads h_out (num_dms x samples_per_second).
 * Synchronous.  The context keeps the device buffers and the last plan
 * between calls (the plan is reused while the table and config repeat).
 *
 * Tuned dispatch (dd_dedisperse and dd_dedisperse_device): a config with
 * staging DD_STAGING_AUTO and no flags is validated by the reference's
 * rules, then the instance's tuned schedule (dd_schedule_get) runs in its
 * place when one exists -- every schedule computes the same bits (one fp32
 * accumulator per output, channels ascending), so only the speed changes.
 * If the schedule cannot be planned for this table the config itself runs. */
dd_status dd_dedisperse(dd_context* ctx, const float* h_in, uint32_t channels,
                        uint64_t num_samples, const uint32_t* h_shifts, uint32_t num_dms,
                        uint32_t samples_per_second, const dd_config* cfg,
                        const dd_limits* limits, float* h_out);

/* ------------------------------------------------ SIGPROC ingest ------ */
/* Device transpose of a SIGPROC payload (time-major, channel 0 = highest
 * frequency, float32 [num_samples][channels]) into the channel-major,
 * lowest-first filterbank layout at d_dst (row pitch dst_pitch floats) --
 * the transpose of reference sigproc.cpp:177-189.  *first_bad receives the
 * payload index of the first non-finite sample (the reference raises
 * format_error at byte offset header_end + 4*index) or -1.  Synchronous. */
dd_status dd_sigproc_to_filterbank(dd_context* ctx, const float* d_payload, uint32_t channels,
                                   uint64_t num_samples, float* d_dst, uint64_t dst_pitch,
                                   int64_t* first_bad);

/* Streaming upload: samples [t0, t1) of every channel of a host filterbank
 * block (row pitch h_pitch floats; pinned memory for an asynchronous copy)
 * into the device block (row pitch d_pitch floats), as one 2-D copy enqueued
 * on `stream` (a cudaStream_t; NULL = the context stream).  Lets a caller
 * ship a block in time order, so the DMs whose delays fit the first part can
 * start -- and their output leave the device -- before the block's tail
 * lands. */
dd_status dd_upload_block_range(dd_context* ctx, const float* h_block, uint64_t h_pitch,
                                float* d_block, uint64_t d_pitch, uint32_t channels,
                                uint64_t t0, uint64_t t1, void* stream);

/* --------------------------------------------------- tuned schedules -- */
/* The configuration the one-shot entry points run for an AUTO config on an
 * instance of `channels` channels, `samples_per_second` and `num_dms`
 * trials: one registered with dd_schedule_set (e.g. a tuning result's best
 * record, tuner.cpp:172-179), else a built-in pick from the committed
 * sweeps (tuning/, Apertif- and LOFAR-like geometries, d = 2..4096).
 * dd_schedule_get returns DD_ERR_INVALID_ARGUMENT when there is none;
 * *builtin (may be NULL) tells which table answered. */
dd_status dd_schedule_set(uint32_t channels, uint32_t samples_per_second, uint32_t num_dms,
                          const dd_config* cfg); /* cfg == NULL forgets the entry */
dd_status dd_schedule_get(uint32_t channels, uint32_t samples_per_second, uint32_t num_dms,
                          dd_config* cfg, int* builtin);
/* The schedule the last dd_dedisperse / dd_dedisperse_device on this
 * context actually ran (the tuned one, or the caller's config). */
dd_status dd_last_run_config(dd_context* ctx, dd_config* cfg, uint32_t* family);

/* ------------------------------------------------- checked builds ---- */
/* Device bounds violations counted by a checked build of this library
 * (libdedisp_b200_checked.so, -DDDB_CHECKED: every staged window read, bulk
 * copy and output store bounds-checked on the device) on the current
 * device since the last reset; *checked = 0 and count 0 in release builds.
 * Synchronises the device. */
dd_status dd_debug_violations(uint64_t* count, int* checked, int reset);

/* ------------------------------------------------------ fingerprints -- */
/* FNV-1a 64 (basis 0xcbf29ce484222325, prime 0x100000001b3) over `bytes`
 * bytes of host memory: the fingerprint the golden fixtures use
 * (tests/golden/golden.json), so a caller can check a full output against
 * the reference's without keeping the reference's output around. */
dd_status dd_fingerprint(const void* data, uint64_t bytes, uint64_t* out);

/* ---------------------------------------------- streaming blocks ----- */
/* Consecutive seconds of a live observation (the
 * reference handles one padded block, setup.cpp:130-133).  The stream keeps
 * a device ring of the last t = instance_sizing(setup, num_dms).num_samples
 * samples per channel; every push appends one second (host [channels][s],
 * channel-major) and, once the window is full, dedisperses its first second:
 * h_out (num_dms x s, may be NULL) receives exactly what a one-shot pass over
 * the same t samples gives, *produced = 1.  cfg == NULL (or AUTO without
 * flags) runs the instance's tuned schedule.  Synchronous per push. */
typedef struct dd_block_stream dd_block_stream;
dd_status dd_block_stream_create(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                                 const dd_config* cfg, dd_block_stream** out);
dd_status dd_block_stream_push(dd_block_stream* stream, const float* h_second, float* h_out,
                               int* produced);
/* counters and the device output of the last pass (any may be NULL) */
dd_status dd_block_stream_info(const dd_block_stream* stream, uint64_t* num_samples,
                               uint64_t* pushes, uint64_t* outputs, uint64_t* compactions,
                               const float** d_out);
dd_status dd_block_stream_destroy(dd_block_stream* stream);

/* ---------------------------------------------- synthetic input ------- */
/* noise_filterbank, filterbank.cpp:60-80: mt19937_64(seed), Box-Muller,
 * channel-major fill, float(sigma * g).  Host memory; threads = 0 -> all. */
dd_status dd_noise_filterbank(uint32_t channels, uint64_t num_samples, float sigma,
                              uint64_t seed, int threads, float* h_out);

/* ------------------------------------------------------- tuner -------- */
/* enumerate_configs, tuner.cpp:103-134: the reference's divisor space.
 * Writes min(count, capacity) configs (GPU knobs zeroed). */
dd_status dd_enumerate_configs(uint32_t num_dms, uint32_t samples_per_second,
                               const dd_limits* limits, dd_config* out, uint64_t capacity,
                               uint64_t* count);

typedef struct dd_tune_options {
  dd_limits limits;
  uint32_t repeats;       /* timed runs per config (default 10) */
  uint32_t zero_dm;       /* 1: all-zero table (zero_dm_experiment) */
  uint64_t seed;          /* noise seed (TuneOptions.seed, default 1) */
  uint32_t space;         /* 0: GPU space (reference-valid 4-tuples the device
                             kernels support, x depth x staging);
                             1: the full reference divisor space */
  uint32_t max_configs;   /* 0 = no cap */
  uint32_t flush_l2;      /* 1: write a buffer larger than L2 before every
                             timed run (outside the events), so instances
                             whose input fits the 126 MB L2 are timed cold */
  uint32_t reserved;
  double* runs;           /* NULL, or repeats doubles per record (record
                             order): every timed run in seconds, the
                             reference's runs_s (report_io.cpp:70-79) */
} dd_tune_options;

/* The GPU tuning space for an instance (see dd_tune_options.space = 0). */
dd_status dd_enumerate_gpu_configs(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                                   const dd_limits* limits, dd_config* out, uint64_t capacity,
                                   uint64_t* count);

typedef struct dd_tuning_record {
  dd_config config;
  double mean_time;  /* seconds, over the timed repeats */
  double min_time;
  double max_time;
  double gflops;     /* num_dms*s*channels / mean_time / 1e9 */
  uint32_t timer_warning;
  uint32_t family;
} dd_tuning_record;

typedef struct dd_tuning_summary {
  uint64_t count;
  uint64_t best_index;     /* select_best, tuner.cpp:172-179 */
  double mean_gflops;      /* compute_stats, tuner.cpp:181-206 */
  double stddev_gflops;
  double snr_optimum;      /* NaN when degenerate */
  double chebyshev_bound;  /* NaN when degenerate */
  uint32_t degenerate;
  uint32_t realtime_pass;
  double realtime_threshold_gflops; /* analysis.cpp:40-45 */
  double clock_resolution_s;
} dd_tuning_summary;

/* tune / zero_dm_experiment (tuner.cpp:43-99, 208-216) on the device:
 * builds the table on the device, the noise input on the host, then
 * benchmarks every config of the chosen space sequentially with CUDA events.
 * records must hold `capacity` entries; summary->count is the space size. */
dd_status dd_tune(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                  const dd_tune_options* options, dd_tuning_record* records, uint64_t capacity,
                  dd_tuning_summary* summary);

/* select_best / compute_stats over caller records (pure, replayable). */
dd_status dd_select_best(const dd_tuning_record* records, uint64_t count, uint64_t* best);
dd_status dd_compute_stats(const dd_tuning_record* records, uint64_t count, uint64_t best,
                           dd_tuning_summary* summary);

#ifdef __cplusplus
}
#endif
#endif /* DEDISP_B200_H */
