// tuner.cpp -- the auto-tuner (reference tuner.cpp:19-216) on the device,
// plus the synthetic noise input (reference filterbank.cpp:22-80).
//
// Timing follows benchmark_config (tuner.cpp:136-170): one untimed warm-up,
// then `repeats` timed runs -- here with CUDA events on the context stream
// instead of steady_clock, inputs resident on the device as the paper
// assumes.  Selection, statistics and the real-time
// threshold are the reference's definitions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
#include <vector>

#include "internal.hpp"

using namespace ddb;

#define DD_TRY(call)            \
  do {                          \
    dd_status s_ = (call);      \
    if (s_ != DD_OK) return s_; \
  } while (0)

namespace {

// divisors_ascending, tuner.cpp:19-30
std::vector<uint32_t> divisors(uint32_t n) {
  std::vector<uint32_t> small, large;
  for (uint64_t k = 1; k * k <= n; ++k)
    if (n % k == 0) {
      small.push_back(static_cast<uint32_t>(k));
      if (k != n / k) large.push_back(static_cast<uint32_t>(n / k));
    }
  small.insert(small.end(), large.rbegin(), large.rend());
  return small;
}

std::vector<dd_config> reference_space(uint32_t d, uint32_t s, const dd_limits& L) {
  const std::vector<uint32_t> td = divisors(s), dd = divisors(d);
  std::vector<dd_config> out;
  for (uint32_t it : td) {
    if (it > L.max_block_items) break;
    for (uint32_t idm : dd) {
      if (static_cast<uint64_t>(it) * idm > L.max_block_items) break;
      for (uint32_t wt : td) {
        if (wt > L.max_accumulators) break;
        const uint64_t tt = static_cast<uint64_t>(it) * wt;
        if (tt > s || s % tt != 0) continue;
        for (uint32_t wd : dd) {
          if (static_cast<uint64_t>(wt) * wd > L.max_accumulators) break;
          const uint64_t tdm = static_cast<uint64_t>(idm) * wd;
          if (tdm > d || d % tdm != 0) continue;
          out.push_back(dd_config{it, idm, wt, wd, 1, DD_STAGING_AUTO});
        }
      }
    }
  }
  return out;
}

// config_preferred (tuner.cpp:35-41), extended with the two GPU knobs as a
// final tie-break so the order stays total.
bool preferred(const dd_tuning_record& a, const dd_tuning_record& b) {
  if (a.gflops != b.gflops) return a.gflops > b.gflops;
  const uint64_t ai = static_cast<uint64_t>(a.config.items_time) * a.config.items_dm;
  const uint64_t bi = static_cast<uint64_t>(b.config.items_time) * b.config.items_dm;
  if (ai != bi) return ai < bi;
  const uint32_t ka[7] = {a.config.items_time, a.config.items_dm, a.config.work_time,
                          a.config.work_dm, a.config.dm_tile_depth, a.config.staging,
                          a.config.flags};
  const uint32_t kb[7] = {b.config.items_time, b.config.items_dm, b.config.work_time,
                          b.config.work_dm, b.config.dm_tile_depth, b.config.staging,
                          b.config.flags};
  return std::lexicographical_compare(ka, ka + 7, kb, kb + 7);
}

// CUDA event resolution (the analogue of clock_resolution_seconds,
// tuner.cpp:313-330): documented as ~0.5 us.
constexpr double kEventResolution = 0.5e-6;

}  // namespace

extern "C" {

// ------------------------------------------------------------- noise ---
dd_status dd_noise_filterbank(uint32_t channels, uint64_t num_samples, float sigma, uint64_t seed,
                              int threads, float* out) {
  if (out == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "out is null");
  if (channels == 0) return fail(DD_ERR_INVALID_ARGUMENT, "channels must be >= 1");
  if (num_samples == 0) return fail(DD_ERR_INVALID_ARGUMENT, "filterbank needs at least one sample");
  if (!std::isfinite(sigma) || sigma < 0.0f)
    return fail(DD_ERR_INVALID_ARGUMENT, "noise sigma must be finite and non-negative");
  const uint64_t n = static_cast<uint64_t>(channels) * num_samples;
  if (!(sigma > 0.0f)) {
    std::memset(out, 0, n * sizeof(float));
    return DD_OK;
  }
  // The engine is inherently sequential; the Box-Muller transform is not.
  // Draw raw 64-bit words for a chunk of sample pairs on this thread, then
  // transform the chunk in parallel.  Pair p consumes draws 2p (u1) and
  // 2p+1 (u2) and yields samples 2p = r*cos and 2p+1 = r*sin, exactly the
  // reference's GaussianStream order (filterbank.cpp:26-39).
  unsigned nt = threads > 0 ? static_cast<unsigned>(threads) : std::thread::hardware_concurrency();
  nt = std::max(1u, std::min(nt, 64u));
  std::mt19937_64 engine(seed);
  const uint64_t pairs = (n + 1) / 2;
  const uint64_t chunk = 1u << 21;  // pairs per chunk
  std::vector<uint64_t> raw(2 * std::min(chunk, pairs));
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double sig = static_cast<double>(sigma);
  for (uint64_t p0 = 0; p0 < pairs; p0 += chunk) {
    const uint64_t np = std::min(chunk, pairs - p0);
    for (uint64_t i = 0; i < 2 * np; ++i) raw[i] = engine();
    auto work = [&](uint64_t a, uint64_t b) {
      for (uint64_t p = a; p < b; ++p) {
        const double u1 = 1.0 - static_cast<double>(raw[2 * p] >> 11) * 0x1.0p-53;
        const double u2 = static_cast<double>(raw[2 * p + 1] >> 11) * 0x1.0p-53;
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = two_pi * u2;
        const uint64_t idx = 2 * (p0 + p);
        out[idx] = static_cast<float>(sig * (radius * std::cos(angle)));
        if (idx + 1 < n) out[idx + 1] = static_cast<float>(sig * (radius * std::sin(angle)));
      }
    };
    if (nt == 1 || np < 4096) {
      work(0, np);
    } else {
      std::vector<std::thread> pool;
      const uint64_t per = (np + nt - 1) / nt;
      for (unsigned t = 0; t < nt; ++t) {
        const uint64_t a = t * per, b = std::min(np, a + per);
        if (a < b) pool.emplace_back(work, a, b);
      }
      for (auto& th : pool) th.join();
    }
  }
  return DD_OK;
}

// ----------------------------------------------------------- configs ---
dd_status dd_enumerate_configs(uint32_t num_dms, uint32_t s, const dd_limits* limits,
                               dd_config* out, uint64_t capacity, uint64_t* count) {
  if (count == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "count is null");
  if (num_dms == 0 || s == 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "instance dimensions must be positive");
  const std::vector<dd_config> v = reference_space(num_dms, s, effective_limits(limits));
  *count = v.size();
  if (v.empty()) return fail(DD_ERR_INVALID_ARGUMENT, "the limits leave no valid kernel configuration");
  for (uint64_t i = 0; i < v.size() && i < capacity; ++i) {
    out[i] = v[i];
    out[i].dm_tile_depth = 0;
    out[i].staging = 0;
  }
  return DD_OK;
}

// The GPU tuning space: reference-valid 4-tuples (so tuning records keep
// the reference's config identity) that map onto whole
// warps -- items_time a multiple of 32, or 8/16 lanes along time with the
// warp completed along DM.  Register-window shapes (K4) at depth {1, 2};
// shared-memory shapes (K3, 64..1024 threads, instantiated work_dm x
// work_time variant) at depth {1, 2, 4}; and the direct family for the same
// shapes at depth 1 so the paper's "rely on the cache" option is measured.
dd_status dd_enumerate_gpu_configs(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                                   const dd_limits* limits, dd_config* out, uint64_t capacity,
                                   uint64_t* count) {
  if (ctx == nullptr || count == nullptr) return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  std::string why;
  if (!setup_ok(setup, &why)) return fail(DD_ERR_INVALID_ARGUMENT, why);
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "need at least one trial DM");
  const uint32_t s = setup->samples_per_second;
  std::vector<dd_config> v;
  for (const dd_config& k : reference_space(num_dms, s, effective_limits(limits))) {
    const uint32_t block = k.items_time * k.items_dm;
    if (block < 32 || block > 1024 || block % 32 != 0) continue;
    if (!(k.items_time % 32 == 0 || k.items_time == 8 || k.items_time == 16)) continue;
    const uint32_t tiles_dm = num_dms / (k.items_dm * k.work_dm);
    if (regwin_shape_ok(k.work_dm, k.work_time, k.items_time, block)) {
      for (uint32_t cps : {8u, 15u}) {
        dd_config c = k;
        c.dm_tile_depth = 1;
        c.staging = DD_STAGING_REGWIN;
        c.flags = cps << DD_CONFIG_CPS_SHIFT;
        v.push_back(c);
      }
    }
    if (block < 64 || !smem_variant_ok(k.work_dm, k.work_time, block, k.items_time)) continue;
    for (uint32_t depth : {1u, 2u}) {
      if (depth > 1 && tiles_dm < depth * 2) continue;
      // 8 or 15 channels per stage; the time-major raster (large delays)
      // with the wide stages
      for (uint32_t flags : {8u << DD_CONFIG_CPS_SHIFT, 15u << DD_CONFIG_CPS_SHIFT,
                             (15u << DD_CONFIG_CPS_SHIFT) | DD_CONFIG_TIME_MAJOR}) {
        dd_config c = k;
        c.dm_tile_depth = depth;
        c.staging = DD_STAGING_SMEM;
        c.flags = flags;
        v.push_back(c);
      }
      if (num_dms <= 128) {  // where K3 competes: two stages of 24 channels
        dd_config c = k;
        c.dm_tile_depth = depth;
        c.staging = DD_STAGING_SMEM;
        c.flags = DD_CONFIG_WIDE_STAGES | (12u << DD_CONFIG_CPS_SHIFT) |
                  (2u << DD_CONFIG_NSTAGE_SHIFT);
        v.push_back(c);
      }
      // packed stages where a packed build exists (the large-delay shapes)
      ddb::KernelFn packed = nullptr;
      find_smem_kernel(k.work_dm, k.work_time, nullptr, k.items_time, &packed);
      if (packed != nullptr) {
        dd_config c = k;
        c.dm_tile_depth = depth;
        c.staging = DD_STAGING_SMEM;
        c.flags = DD_CONFIG_PACKED_STAGES | DD_CONFIG_TIME_MAJOR;
        v.push_back(c);
      }
    }
    dd_config c = k;
    c.dm_tile_depth = 1;
    c.staging = DD_STAGING_DIRECT;
    v.push_back(c);
  }
  // GPU-native shapes (DD_CONFIG_GPU_TILING, predicated last time tile) for
  // the window families whose W/4-odd vector loads never divide s exactly
  // (e.g. 32 x 12 samples per warp): register windows and TMEM windows.
  for (uint32_t it : {32u, 64u, 128u})
    for (uint32_t idm : {1u, 2u, 4u, 8u})
      for (uint32_t wt : {12u, 20u})
        for (uint32_t wd : {2u, 4u, 8u}) {
          const uint64_t block = static_cast<uint64_t>(it) * idm;
          if (block > 256 || num_dms % (idm * wd) != 0 || it * wt >= s * 2u) continue;
          if (s % (it * wt) == 0) continue;  // already in the reference space
          dd_config c{it, idm, wt, wd, 1, DD_STAGING_REGWIN, DD_CONFIG_GPU_TILING};
          if (tmem_shape_ok(wd, wt, it, block)) {
            // wide stages amortise the per-stage synchronisation; the
            // three-CTA builds need the narrower stages' shared memory
            for (uint32_t cps : {8u, 15u}) {
              c.staging = DD_STAGING_TMEM;
              c.flags = DD_CONFIG_GPU_TILING | (cps << DD_CONFIG_CPS_SHIFT);
              v.push_back(c);
              if (cps == 8 && block <= 128 && tmem_has_occupancy_build(wd, wt)) {
                c.flags |= DD_CONFIG_HIGH_OCCUPANCY;
                v.push_back(c);
              }
            }
            // two stages of 24 channels (measured round 2: 6.19 -> 6.01 ms
            // at Apertif d=4096 against three of 15)
            c.staging = DD_STAGING_TMEM;
            c.flags = DD_CONFIG_GPU_TILING | DD_CONFIG_WIDE_STAGES |
                      (12u << DD_CONFIG_CPS_SHIFT) | (2u << DD_CONFIG_NSTAGE_SHIFT);
            v.push_back(c);
          }
          if (regwin_shape_ok(wd, wt, it, block)) {
            c.staging = DD_STAGING_REGWIN;
            c.flags = DD_CONFIG_GPU_TILING | (8u << DD_CONFIG_CPS_SHIFT);
            v.push_back(c);
          }
        }
  // K6 rectangles for small trial counts, where a DM tile's delays span
  // few samples per channel group (the plan rejects wider spans: the
  // tuner then skips the shape); GPU tiling
  if (num_dms <= 128) {
    // time tiles of 32..128 samples, plus tiles that deal the s samples out
    // in k equal shares per SM (k = 1..4): an HBM-bound pass wants equal
    // bytes per SM, not a ragged last wave
    std::vector<uint32_t> its = {32u, 64u, 96u, 128u};
    for (uint32_t k = 1; k <= 4; ++k) {
      const uint32_t sms = static_cast<uint32_t>(std::max(1, ctx->sm_count));
      const uint32_t it = ((s + sms * k - 1) / (sms * k) + 3u) & ~3u;
      if (it >= 16 && it <= 256 && std::find(its.begin(), its.end(), it) == its.end())
        its.push_back(it);
    }
    for (uint32_t it : its)
      for (uint32_t idm : {1u, 2u, 4u, 8u, 16u})
        for (uint32_t wt : {1u, 2u})
          for (uint32_t wd : {1u, 2u, 4u, 8u, 16u}) {
            const uint64_t block = static_cast<uint64_t>(it) * idm;
            if (block < 32 || block > 512 || num_dms % (idm * wd) != 0) continue;
            if (find_rect_kernel(wd, wt, it) == nullptr) continue;
            // 32, 64 or 128 channels per TMA box (4 stages): wider boxes
            // amortise the per-box cost (measured, small d); the wide boxes
            // also with 2 stages, which leaves room for more CTAs per SM
            // (Apertif d=2: 128 channels x 2 stages 25.6 us vs x 4 35.7 us,
            // profiles/r02_rect_d2_stage_sweep.txt)
            for (uint32_t cps : {2u, 4u, 8u}) {
              dd_config c{it, idm, wt, wd, 1, DD_STAGING_RECT,
                          DD_CONFIG_GPU_TILING | (cps << DD_CONFIG_CPS_SHIFT)};
              v.push_back(c);
              if (cps >= 4) {
                c.flags |= 2u << DD_CONFIG_NSTAGE_SHIFT;
                v.push_back(c);
              }
            }
          }
  }
  *count = v.size();
  for (uint64_t i = 0; i < v.size() && i < capacity; ++i) out[i] = v[i];
  return DD_OK;
}

// ------------------------------------------------ selection / stats ----
dd_status dd_select_best(const dd_tuning_record* r, uint64_t n, uint64_t* best) {
  if (r == nullptr || best == nullptr || n == 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "no records to select from");
  uint64_t b = 0;
  for (uint64_t i = 1; i < n; ++i)
    if (preferred(r[i], r[b])) b = i;
  *best = b;
  return DD_OK;
}

// compute_stats, tuner.cpp:181-206 (population stddev, SNR, Chebyshev).
dd_status dd_compute_stats(const dd_tuning_record* r, uint64_t n, uint64_t best,
                           dd_tuning_summary* out) {
  if (r == nullptr || out == nullptr || n == 0)
    return fail(DD_ERR_INVALID_ARGUMENT, "no records to summarize");
  if (best >= n) return fail(DD_ERR_INVALID_ARGUMENT, "best_index out of range");
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) sum += r[i].gflops;
  const double mean = sum / static_cast<double>(n);
  double var = 0.0;
  for (uint64_t i = 0; i < n; ++i) var += (r[i].gflops - mean) * (r[i].gflops - mean);
  var /= static_cast<double>(n);
  out->best_index = best;
  out->mean_gflops = mean;
  out->stddev_gflops = std::sqrt(var);
  if (out->stddev_gflops > 0.0) {
    const double snr = (r[best].gflops - mean) / out->stddev_gflops;
    out->snr_optimum = snr;
    out->chebyshev_bound = std::min(1.0, 1.0 / (snr * snr));
    out->degenerate = 0;
  } else {
    out->snr_optimum = std::numeric_limits<double>::quiet_NaN();
    out->chebyshev_bound = std::numeric_limits<double>::quiet_NaN();
    out->degenerate = 1;
  }
  return DD_OK;
}

// ------------------------------------------------------------- tune ----
dd_status dd_tune(dd_context* ctx, const dd_setup* setup, uint32_t num_dms,
                  const dd_tune_options* opt, dd_tuning_record* records, uint64_t capacity,
                  dd_tuning_summary* summary) {
  if (ctx == nullptr || opt == nullptr || summary == nullptr)
    return fail(DD_ERR_INVALID_ARGUMENT, "null argument");
  std::string why;
  if (!setup_ok(setup, &why)) return fail(DD_ERR_INVALID_ARGUMENT, why);
  if (num_dms == 0) return fail(DD_ERR_INVALID_ARGUMENT, "need at least one trial DM");
  if (opt->repeats == 0) return fail(DD_ERR_INVALID_ARGUMENT, "need at least one timed repeat");
  const uint32_t s = setup->samples_per_second, c = setup->channels;

  std::vector<dd_config> space;
  uint64_t n = 0;
  if (opt->space == 1) {
    dd_status st = dd_enumerate_configs(num_dms, s, &opt->limits, nullptr, 0, &n);
    if (st != DD_OK) return st;
    space.resize(n);
    dd_enumerate_configs(num_dms, s, &opt->limits, space.data(), n, &n);
  } else {
    dd_status st = dd_enumerate_gpu_configs(ctx, setup, num_dms, &opt->limits, nullptr, 0, &n);
    if (st != DD_OK) return st;
    space.resize(n);
    dd_enumerate_gpu_configs(ctx, setup, num_dms, &opt->limits, space.data(), n, &n);
    if (space.empty())
      return fail(DD_ERR_INVALID_ARGUMENT, "the GPU space is empty for this instance");
  }
  if (opt->max_configs != 0 && space.size() > opt->max_configs) space.resize(opt->max_configs);
  if (records != nullptr && capacity < space.size())
    return fail(DD_ERR_INVALID_ARGUMENT, "record buffer too small");

  // Instance: table on the device, noise on the host (tuner.cpp:52-62).
  void *d_sh = nullptr, *d_in = nullptr, *d_out = nullptr;
  uint32_t md = 0;
  const uint64_t entries = static_cast<uint64_t>(num_dms) * c;
  dd_status st = dd_device_malloc(ctx, entries * 4, &d_sh);
  if (st == DD_OK)
    st = dd_delay_table_device(ctx, setup, num_dms, 0, opt->zero_dm ? 1 : 0,
                               static_cast<uint32_t*>(d_sh), &md);
  const uint64_t t = ((static_cast<uint64_t>(s) + md + s - 1) / s) * s;
  const uint64_t pitch = (t + 3) & ~3ull;
  std::vector<float> fb;
  if (st == DD_OK) {
    fb.resize(static_cast<size_t>(c) * t);
    st = dd_noise_filterbank(c, t, 1.0f, opt->seed, 0, fb.data());
  }
  if (st == DD_OK) st = dd_device_malloc(ctx, pitch * c * 4, &d_in);
  if (st == DD_OK) st = dd_device_malloc(ctx, static_cast<uint64_t>(num_dms) * s * 4, &d_out);
  if (st == DD_OK)
    st = dd_upload_filterbank(ctx, static_cast<float*>(d_in), pitch, fb.data(), c, t);
  if (st == DD_OK) st = dd_context_synchronize(ctx);

  std::vector<dd_tuning_record> recs;
  std::vector<double> runs(opt->repeats);
  const double flop = static_cast<double>(num_dms) * s * c;
  for (size_t i = 0; st == DD_OK && i < space.size(); ++i) {
    dd_plan* p = nullptr;
    st = dd_plan_create(ctx, static_cast<uint32_t*>(d_sh), c, num_dms, s, t, pitch, &space[i],
                        &opt->limits, &p);
    if (st == DD_ERR_INVALID_ARGUMENT && opt->space == 0) {
      st = DD_OK;  // a GPU-space shape this instance cannot stage: not a record
      continue;
    }
    if (st != DD_OK) break;
    st = dd_plan_time_ex(p, static_cast<float*>(d_in), static_cast<float*>(d_out), s, 1,
                         opt->repeats, opt->flush_l2 ? 1 : 0, runs.data());
    if (st == DD_OK && opt->runs != nullptr)
      std::copy(runs.begin(), runs.end(), opt->runs + recs.size() * opt->repeats);
    dd_plan_info info{};
    dd_plan_get_info(p, &info);
    dd_plan_destroy(p);
    if (st != DD_OK) break;
    dd_tuning_record r{};
    r.config = space[i];
    double tot = 0.0;
    r.min_time = runs[0];
    r.max_time = runs[0];
    for (double x : runs) {
      tot += x;
      r.min_time = std::min(r.min_time, x);
      r.max_time = std::max(r.max_time, x);
    }
    r.mean_time = tot / opt->repeats;
    r.timer_warning = kEventResolution > 0.01 * r.mean_time ? 1u : 0u;
    r.gflops = flop / std::max(r.mean_time, kEventResolution) / 1e9;
    r.family = info.family;
    recs.push_back(r);
  }
  dd_device_free(ctx, d_sh);
  dd_device_free(ctx, d_in);
  dd_device_free(ctx, d_out);
  if (st != DD_OK) return st;

  if (recs.empty())
    return fail(DD_ERR_INVALID_ARGUMENT, "no configuration could be planned for this instance");
  std::memset(summary, 0, sizeof(*summary));
  summary->count = recs.size();
  uint64_t best = 0;
  DD_TRY(dd_select_best(recs.data(), recs.size(), &best));
  DD_TRY(dd_compute_stats(recs.data(), recs.size(), best, summary));
  summary->count = recs.size();
  summary->realtime_threshold_gflops = flop / 1e9;  // analysis.cpp:40-45
  summary->realtime_pass = recs[summary->best_index].gflops >= flop / 1e9 ? 1u : 0u;
  summary->clock_resolution_s = kEventResolution;
  if (records != nullptr) std::copy(recs.begin(), recs.end(), records);
  return DD_OK;
}

}  // extern "C"
