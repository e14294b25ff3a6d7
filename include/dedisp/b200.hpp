// dedisp/b200.hpp -- C++ drop-in for the reference's `dedisp` core API
// (/root/reference/proj/core/include/dedisp/{setup,filterbank,kernels,
// tuner,analysis,errors}.hpp), re-implemented over the C-ABI in
// dedisp_b200.h so that every computation on the hot path runs on the B200.
//
// Same namespace, type names, field names, function names, argument meaning
// and exception types as the reference, so code written against the
// reference compiles and behaves the same (bit-identical results).
// Differences, all additive:
//   * ExecOptions gains `device`, `dm_tile_depth`, `staging` and `flags`
//     (GPU knobs); `threads` and `pool` are accepted and ignored (the CUDA
//     grid replaces the reference's ThreadPool).  With the defaults
//     (staging Auto, no flags) dedisperse_tiled validates the config by the
//     reference's rules and then runs the instance's tuned schedule (the
//     tuner's pick, register_schedule() or the built-in sweeps): every
//     schedule computes the same bits, only faster.
//   * TuningRecord carries the GPU knobs (depth, staging, flags, family)
//     next to the 4-tuple, so a tuned record replays exactly.
//   * device_error (a std::runtime_error) reports CUDA failures.
//   * SIGPROC/raw file I/O, setup files, report/manifest JSON and the CLI
//     are outside the hot path and not part of this library.
#pragma once

#include <atomic>
#include <compare>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dedisp_b200.h"

namespace dedisp {

// ---------------------------------------------------------------- errors
// Sizing above a cap or an arithmetic overflow (reference errors.hpp:10-13).
class capacity_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
// Real-time deployment sizing impossible (reference errors.hpp:29-33).
class not_real_time_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
// The device or CUDA runtime failed (no reference analogue: it has no device).
class device_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- setup
struct ObservationSetup {
  std::string name;
  std::uint32_t samples_per_second = 0;
  std::uint32_t channels = 0;
  double f_min = 0.0;          // MHz, centre of channel 0
  double channel_width = 0.0;  // MHz
  double dm_first = 0.0;       // pc/cm^3
  double dm_step = 0.0;        // pc/cm^3

  double channel_frequency(std::uint32_t ch) const {
    return f_min + static_cast<double>(ch) * channel_width;
  }
  double highest_frequency() const { return channel_frequency(channels - 1); }
  double trial_dm(std::uint32_t i) const { return dm_first + static_cast<double>(i) * dm_step; }
  void validate() const;  // std::invalid_argument on a bad field
};

struct DelayTable {
  ObservationSetup setup;
  std::uint32_t num_dms = 0;
  std::vector<std::uint32_t> shifts;  // [num_dms][channels], DM-major
  std::uint32_t max_delay = 0;

  std::uint32_t at(std::uint32_t channel, std::uint32_t dm) const {
    return shifts[static_cast<std::size_t>(dm) * setup.channels + channel];
  }
  const std::uint32_t* row(std::uint32_t dm) const {
    return shifts.data() + static_cast<std::size_t>(dm) * setup.channels;
  }
};

struct ProblemInstance {
  ObservationSetup setup;
  std::uint32_t num_dms = 0;
  std::uint64_t num_samples = 0;
  std::uint64_t flop = 0;
  std::uint32_t max_delay = 0;
};

inline constexpr std::uint64_t kDefaultDelayTableCapBytes = std::uint64_t{1} << 30;

double delay_seconds(double dm, double f_channel_mhz, double f_highest_mhz);
// Computed on the device in FP64 (K1), returned in host memory.
DelayTable build_delay_table(const ObservationSetup& setup, std::uint32_t num_dms,
                             std::uint64_t memory_cap_bytes = kDefaultDelayTableCapBytes);
DelayTable build_zero_delay_table(const ObservationSetup& setup, std::uint32_t num_dms,
                                  std::uint64_t memory_cap_bytes = kDefaultDelayTableCapBytes);
ProblemInstance instance_sizing(const ObservationSetup& setup, std::uint32_t num_dms);
const std::vector<ObservationSetup>& builtin_setups();
const ObservationSetup* find_builtin(std::string_view name);

// ----------------------------------------------------------- filterbank
struct Filterbank {
  ObservationSetup setup;
  std::uint32_t num_samples = 0;
  std::vector<float> data;  // [channels][num_samples], channel-major

  float at(std::uint32_t ch, std::uint32_t j) const {
    return data[static_cast<std::size_t>(ch) * num_samples + j];
  }
  std::span<const float> channel(std::uint32_t ch) const {
    return {data.data() + static_cast<std::size_t>(ch) * num_samples, num_samples};
  }
};

inline constexpr const char* kNoiseRngId = "mt19937_64/box-muller";
Filterbank noise_filterbank(const ObservationSetup& setup, std::uint32_t num_samples, float sigma,
                            std::uint64_t seed);

// -------------------------------------------------------------- kernels
struct DedispersedSeries {
  std::uint32_t num_dms = 0;
  std::uint32_t samples_per_second = 0;
  std::vector<float> data;  // [num_dms][samples_per_second]

  float at(std::uint32_t dm, std::uint32_t j) const {
    return data[static_cast<std::size_t>(dm) * samples_per_second + j];
  }
  const float* row(std::uint32_t dm) const {
    return data.data() + static_cast<std::size_t>(dm) * samples_per_second;
  }
};

struct KernelLimits {
  std::uint32_t max_block_items = 1024;
  std::uint32_t max_accumulators = 256;
};

struct KernelConfig {
  std::uint32_t items_time = 1;
  std::uint32_t items_dm = 1;
  std::uint32_t work_time = 1;
  std::uint32_t work_dm = 1;

  std::uint32_t tile_time() const { return items_time * work_time; }
  std::uint32_t tile_dm() const { return items_dm * work_dm; }
  std::uint32_t block_items() const { return items_time * items_dm; }
  std::uint32_t accumulators() const { return work_time * work_dm; }
  friend auto operator<=>(const KernelConfig&, const KernelConfig&) = default;
};

struct KernelStats {
  std::atomic<std::uint64_t> flop_additions{0};
  std::atomic<std::uint64_t> staged_loads{0};
  void reset() {
    flop_additions.store(0, std::memory_order_relaxed);
    staged_loads.store(0, std::memory_order_relaxed);
  }
};

class ThreadPool;  // accepted for source compatibility; never dereferenced

enum class Staging : std::uint32_t {
  Auto = DD_STAGING_AUTO,
  SharedMemory = DD_STAGING_SMEM,
  Direct = DD_STAGING_DIRECT,
  RegisterWindow = DD_STAGING_REGWIN,
  TensorMemory = DD_STAGING_TMEM,
  Rectangle = DD_STAGING_RECT,
};

struct ExecOptions {
  int threads = 0;               // ignored on the device
  KernelLimits limits{};
  KernelStats* stats = nullptr;
  ThreadPool* pool = nullptr;    // ignored on the device
  int device = 0;
  std::uint32_t dm_tile_depth = 1;
  Staging staging = Staging::Auto;
  std::uint32_t flags = 0;       // DD_CONFIG_* (GPU tiling, stage shape, raster, ...)
};

bool config_valid(const KernelConfig& cfg, std::uint32_t num_dms, std::uint32_t samples_per_second,
                  const KernelLimits& limits = {}) noexcept;
void validate_config(const KernelConfig& cfg, std::uint32_t num_dms,
                     std::uint32_t samples_per_second, const KernelLimits& limits = {});

DedispersedSeries dedisperse_reference(const Filterbank& fb, const DelayTable& table,
                                       KernelStats* stats = nullptr);
void dedisperse_reference_into(DedispersedSeries& out, const Filterbank& fb,
                               const DelayTable& table, KernelStats* stats = nullptr);
DedispersedSeries dedisperse_tiled(const Filterbank& fb, const DelayTable& table,
                                   const KernelConfig& cfg, const ExecOptions& options = {});
void dedisperse_tiled_into(DedispersedSeries& out, const Filterbank& fb, const DelayTable& table,
                           const KernelConfig& cfg, const ExecOptions& options = {});

struct LoadCounts {
  std::uint64_t staged_loads = 0;
  std::uint64_t ideal_loads = 0;
};
LoadCounts count_loads(const DelayTable& table, const KernelConfig& cfg, std::uint32_t num_dms,
                       std::uint32_t samples_per_second);

// ---------------------------------------------------------------- tuner
struct TuningRecord {
  KernelConfig config;
  std::vector<double> runs;
  double mean_time = 0.0;
  double gflops = 0.0;
  bool timer_warning = false;
  std::uint32_t dm_tile_depth = 1;
  Staging staging = Staging::Auto;
  std::uint32_t flags = 0;   // DD_CONFIG_* the record was timed with
  Staging family = Staging::Auto;  // kernel family that ran (staging Auto resolved)
  // The ExecOptions that replay this record exactly.
  ExecOptions exec_options() const {
    ExecOptions o;
    o.dm_tile_depth = dm_tile_depth;
    o.staging = staging;
    o.flags = flags;
    return o;
  }
};

struct TuningStats {
  double mean_gflops = 0.0;
  double stddev_gflops = 0.0;
  std::optional<double> snr_optimum;
  std::optional<double> chebyshev_bound;
  bool degenerate = false;
};

struct TuningResult {
  ObservationSetup setup;
  std::uint32_t num_dms = 0;
  bool zero_dm = false;
  KernelLimits limits{};
  std::uint32_t repeats = 0;
  std::uint64_t seed = 0;
  int threads = 1;
  std::string rng_id;
  double clock_resolution_s = 0.0;
  std::vector<TuningRecord> records;
  std::size_t best_index = 0;
  TuningStats stats{};
  double realtime_threshold_gflops = 0.0;
  bool realtime_pass = false;
  const TuningRecord& best() const { return records[best_index]; }
};

std::vector<KernelConfig> enumerate_configs(std::uint32_t num_dms, std::uint32_t samples_per_second,
                                            const KernelLimits& limits = {});
TuningRecord benchmark_config(const Filterbank& fb, const DelayTable& table,
                              const KernelConfig& cfg, std::uint32_t repeats = 10,
                              const ExecOptions& options = {});
std::size_t select_best(std::span<const TuningRecord> records);
TuningStats compute_stats(std::span<const TuningRecord> records, std::size_t best_index);

struct TuneOptions {
  KernelLimits limits{};
  std::uint32_t repeats = 10;
  int threads = 0;  // ignored
  std::uint64_t seed = 1;
  ThreadPool* pool = nullptr;  // ignored
  int device = 0;
  bool full_reference_space = false;  // false: the GPU space (dd_enumerate_gpu_configs)
  std::uint32_t max_configs = 0;
  bool flush_l2 = true;  // evict L2 before every timed run (cold-cache timing)
};
TuningResult tune(const ObservationSetup& setup, std::uint32_t num_dms,
                  const TuneOptions& options = {});
TuningResult zero_dm_experiment(const ObservationSetup& setup, std::uint32_t num_dms,
                                const TuneOptions& options = {});

struct FixedConfigReport {
  KernelConfig config;
  std::uint32_t dm_tile_depth = 1;  // the GPU knobs of the fixed config
  Staging staging = Staging::Auto;
  std::uint32_t flags = 0;
  double total_gflops = 0.0;
  std::vector<double> fixed_gflops;
  std::vector<double> speedup_over_fixed;
};
FixedConfigReport best_fixed_config(std::span<const TuningResult> results);
// The schedule dedisperse_tiled's Auto staging runs for the result's
// instance from now on: its best record (dd_schedule_set).
void register_schedule(const TuningResult& result);
std::vector<std::uint32_t> default_instances();
std::uint64_t estimate_instance_bytes(const ObservationSetup& setup, std::uint32_t num_dms);

// ------------------------------------------------------- analysis (metric defs)
struct AiBounds {
  double no_reuse = 0.25;
  double reuse_bound = 0.0;
};
AiBounds ai_bounds(std::uint64_t num_dms, std::uint64_t samples_per_second,
                   std::uint64_t channels);
struct MemoryTraffic {
  std::uint64_t staged_loads = 0;
  std::uint64_t output_writes = 0;
  std::uint64_t delay_reads = 0;
};
MemoryTraffic kernel_traffic(const DelayTable& table, const KernelConfig& cfg,
                             std::uint32_t num_dms, std::uint32_t samples_per_second);
double measured_ai(std::uint64_t flops, const MemoryTraffic& traffic);
double realtime_threshold_gflops(const ObservationSetup& setup, std::uint32_t num_dms);

// analysis.hpp:43-58: devices covering `beams` beams in real time given one
// pass's measured time (throws not_real_time_error for passes >= 1 s).
struct DeploymentPlan {
  std::uint32_t beams_per_device = 0;
  std::uint64_t devices = 0;
};
DeploymentPlan deployment_sizing(const ObservationSetup& setup, std::uint32_t num_dms,
                                 std::uint32_t beams, double measured_time_per_pass);

// analysis.hpp:60-82: published peaks of the paper's five cards and the
// roofline placement of an arithmetic intensity.
struct DevicePeaks {
  std::string name;
  double peak_gflops = 0.0;
  double peak_gbs = 0.0;
  double ridge_flop_per_byte() const { return peak_gflops / peak_gbs; }
};
std::span<const DevicePeaks> reference_devices();
struct RooflineVerdict {
  bool memory_bound = false;
  double ridge_flop_per_byte = 0.0;
  double attainable_gflops = 0.0;
};
RooflineVerdict classify_roofline(double ai_flop_per_byte, double peak_gflops, double peak_gbs);

// tuner.hpp:115-123: equal-width gflops histogram over [min, max].
struct HistogramBin {
  double lo = 0.0;
  double hi = 0.0;
  std::size_t count = 0;
};
std::vector<HistogramBin> make_histogram(const TuningResult& result, std::size_t bins);

}  // namespace dedisp
