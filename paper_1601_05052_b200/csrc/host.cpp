// host.cpp -- the reference's C++ API (namespace dedisp) implemented over the
// C-ABI.  Each function cites the reference function whose contract it
// keeps; all compute goes through dd_* into the CUDA kernels.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "dedisp/b200.hpp"

namespace dedisp {
namespace {

std::mutex g_mu;  // one device context per device, calls serialised

[[noreturn]] void raise(dd_status st) {
  const std::string msg = dd_last_error();
  switch (st) {
    case DD_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case DD_ERR_CAPACITY:
      throw capacity_error(msg);
    default:
      throw device_error(msg.empty() ? "device failure" : msg);
  }
}

void check(dd_status st) {
  if (st != DD_OK) raise(st);
}

dd_context* context(int device) {
  static std::map<int, dd_context*> contexts;
  auto it = contexts.find(device);
  if (it != contexts.end()) return it->second;
  dd_context* c = nullptr;
  check(dd_context_create(device, &c));
  contexts[device] = c;
  return c;
}

dd_setup to_c(const ObservationSetup& s) {
  return dd_setup{s.samples_per_second, s.channels, s.f_min, s.channel_width, s.dm_first,
                  s.dm_step};
}

dd_config to_c(const KernelConfig& k, const ExecOptions& o) {
  return dd_config{k.items_time,     k.items_dm,
                   k.work_time,      k.work_dm,
                   o.dm_tile_depth,  static_cast<uint32_t>(o.staging),
                   o.flags};
}

dd_limits to_c(const KernelLimits& l) { return dd_limits{l.max_block_items, l.max_accumulators}; }

DelayTable make_table(const ObservationSetup& setup, std::uint32_t num_dms, std::uint64_t cap,
                      int zero) {
  setup.validate();
  if (num_dms < 1) throw std::invalid_argument("num_dms must be >= 1");
  const unsigned __int128 bytes = static_cast<unsigned __int128>(num_dms) * setup.channels * 4u;
  if (bytes > cap)
    throw capacity_error("delay table of " + std::to_string(static_cast<std::uint64_t>(bytes)) +
                         " bytes exceeds the cap of " + std::to_string(cap));
  DelayTable t;
  t.setup = setup;
  t.num_dms = num_dms;
  t.shifts.resize(static_cast<std::size_t>(num_dms) * setup.channels);
  const dd_setup cs = to_c(setup);
  std::lock_guard<std::mutex> g(g_mu);
  check(dd_build_delay_table(context(0), &cs, num_dms, cap, zero, t.shifts.data(), &t.max_delay));
  return t;
}

// check_pair, reference kernels.cpp:16-28
void check_pair(const Filterbank& fb, const DelayTable& table) {
  if (fb.setup.channels != table.setup.channels ||
      fb.setup.samples_per_second != table.setup.samples_per_second)
    throw std::invalid_argument("filterbank and delay table describe different setups");
  if (table.num_dms == 0) throw std::invalid_argument("delay table holds no trials");
  const std::uint64_t needed =
      static_cast<std::uint64_t>(fb.setup.samples_per_second) + table.max_delay;
  if (fb.num_samples < needed)
    throw std::invalid_argument("filterbank too short: need " + std::to_string(needed) +
                                " samples per channel, have " + std::to_string(fb.num_samples));
  if (fb.data.size() != static_cast<std::size_t>(fb.setup.channels) * fb.num_samples)
    throw std::invalid_argument("filterbank data size does not match its shape");
}

void run(DedispersedSeries& out, const Filterbank& fb, const DelayTable& table,
         const dd_config* cfg, const dd_limits* limits, int device) {
  check_pair(fb, table);
  const std::uint32_t d = table.num_dms, s = fb.setup.samples_per_second;
  out.num_dms = d;
  out.samples_per_second = s;
  out.data.resize(static_cast<std::size_t>(d) * s);
  std::lock_guard<std::mutex> g(g_mu);
  check(dd_dedisperse(context(device), fb.data.data(), fb.setup.channels, fb.num_samples,
                      table.shifts.data(), d, s, cfg, limits, out.data.data()));
}

}  // namespace

// ---------------------------------------------------------------- setup
void ObservationSetup::validate() const {
  const dd_setup s = to_c(*this);
  if (dd_setup_validate(&s) != DD_OK) throw std::invalid_argument(dd_last_error());
}

double delay_seconds(double dm, double f_ch, double f_hi) {
  double out = 0.0;
  check(dd_delay_seconds(dm, f_ch, f_hi, &out));
  return out;
}

DelayTable build_delay_table(const ObservationSetup& setup, std::uint32_t num_dms,
                             std::uint64_t cap) {
  return make_table(setup, num_dms, cap, 0);
}

DelayTable build_zero_delay_table(const ObservationSetup& setup, std::uint32_t num_dms,
                                  std::uint64_t cap) {
  return make_table(setup, num_dms, cap, 1);
}

ProblemInstance instance_sizing(const ObservationSetup& setup, std::uint32_t num_dms) {
  const dd_setup s = to_c(setup);
  ProblemInstance p;
  p.setup = setup;
  p.num_dms = num_dms;
  check(dd_instance_sizing(&s, num_dms, &p.num_samples, &p.flop, &p.max_delay));
  return p;
}

// The two built-in telescopes, reference setup.cpp:139-147.
const std::vector<ObservationSetup>& builtin_setups() {
  static const std::vector<ObservationSetup> v = {
      ObservationSetup{"Apertif", 20000, 1024, 1420.0, 0.29, 0.0, 0.25},
      ObservationSetup{"LOFAR", 200000, 32, 138.0, 0.19, 0.0, 0.25},
  };
  return v;
}

const ObservationSetup* find_builtin(std::string_view name) {
  for (const auto& s : builtin_setups())
    if (s.name == name) return &s;
  return nullptr;
}

// ----------------------------------------------------------- filterbank
Filterbank noise_filterbank(const ObservationSetup& setup, std::uint32_t num_samples, float sigma,
                            std::uint64_t seed) {
  setup.validate();
  Filterbank fb;
  fb.setup = setup;
  fb.num_samples = num_samples;
  fb.data.resize(static_cast<std::size_t>(setup.channels) * num_samples);
  check(dd_noise_filterbank(setup.channels, num_samples, sigma, seed, 0, fb.data.data()));
  return fb;
}

// -------------------------------------------------------------- kernels
bool config_valid(const KernelConfig& cfg, std::uint32_t d, std::uint32_t s,
                  const KernelLimits& limits) noexcept {
  const dd_config c = to_c(cfg, ExecOptions{});
  const dd_limits l = to_c(limits);
  return dd_config_valid(&c, d, s, &l) != 0;
}

void validate_config(const KernelConfig& cfg, std::uint32_t d, std::uint32_t s,
                     const KernelLimits& limits) {
  const dd_config c = to_c(cfg, ExecOptions{});
  const dd_limits l = to_c(limits);
  check(dd_validate_config(&c, d, s, &l));
}

void dedisperse_reference_into(DedispersedSeries& out, const Filterbank& fb,
                               const DelayTable& table, KernelStats* stats) {
  run(out, fb, table, nullptr, nullptr, 0);
  if (stats != nullptr) {
    const std::uint64_t total =
        static_cast<std::uint64_t>(table.num_dms) * fb.setup.samples_per_second * fb.setup.channels;
    stats->flop_additions.fetch_add(total, std::memory_order_relaxed);
    stats->staged_loads.fetch_add(total, std::memory_order_relaxed);  // kernels.cpp:102-107
  }
}

DedispersedSeries dedisperse_reference(const Filterbank& fb, const DelayTable& table,
                                       KernelStats* stats) {
  DedispersedSeries out;
  dedisperse_reference_into(out, fb, table, stats);
  return out;
}

void dedisperse_tiled_into(DedispersedSeries& out, const Filterbank& fb, const DelayTable& table,
                           const KernelConfig& cfg, const ExecOptions& options) {
  check_pair(fb, table);
  // the reference's rules (kernels.cpp:58-81); GPU flags in the options
  // (a replayed tuning record) relax only what they name
  const dd_config c = to_c(cfg, options);
  const dd_limits l = to_c(options.limits);
  check(dd_validate_config(&c, table.num_dms, fb.setup.samples_per_second, &l));
  run(out, fb, table, &c, &l, options.device);
  if (options.stats != nullptr) {
    options.stats->flop_additions.fetch_add(
        static_cast<std::uint64_t>(table.num_dms) * fb.setup.samples_per_second * fb.setup.channels,
        std::memory_order_relaxed);
    // count_loads.cpp:9-68 for the config as given (a GPU-tiled one counts
    // its predicated last tile like a full one)
    std::uint64_t staged = 0, ideal = 0;
    check(dd_count_loads(table.shifts.data(), table.setup.channels, table.num_dms,
                         fb.setup.samples_per_second, &c, &staged, &ideal));
    options.stats->staged_loads.fetch_add(staged, std::memory_order_relaxed);
  }
}

DedispersedSeries dedisperse_tiled(const Filterbank& fb, const DelayTable& table,
                                   const KernelConfig& cfg, const ExecOptions& options) {
  DedispersedSeries out;
  dedisperse_tiled_into(out, fb, table, cfg, options);
  return out;
}

LoadCounts count_loads(const DelayTable& table, const KernelConfig& cfg, std::uint32_t num_dms,
                       std::uint32_t s) {
  if (num_dms == 0 || num_dms != table.num_dms)
    throw std::invalid_argument("delay table does not cover the requested trial count");
  const dd_config c = to_c(cfg, ExecOptions{});
  LoadCounts out;
  check(dd_count_loads(table.shifts.data(), table.setup.channels, num_dms, s, &c,
                       &out.staged_loads, &out.ideal_loads));
  return out;
}

// ---------------------------------------------------------------- tuner
std::vector<KernelConfig> enumerate_configs(std::uint32_t d, std::uint32_t s,
                                            const KernelLimits& limits) {
  const dd_limits l = to_c(limits);
  std::uint64_t n = 0;
  check(dd_enumerate_configs(d, s, &l, nullptr, 0, &n));
  std::vector<dd_config> buf(n);
  check(dd_enumerate_configs(d, s, &l, buf.data(), n, &n));
  std::vector<KernelConfig> out;
  out.reserve(n);
  for (const dd_config& c : buf)
    out.push_back(KernelConfig{c.items_time, c.items_dm, c.work_time, c.work_dm});
  return out;
}

// benchmark_config, tuner.cpp:136-170: 1 warm-up + `repeats` timed runs on a
// device-resident input, CUDA-event timed.
TuningRecord benchmark_config(const Filterbank& fb, const DelayTable& table,
                              const KernelConfig& cfg, std::uint32_t repeats,
                              const ExecOptions& options) {
  if (repeats == 0) throw std::invalid_argument("need at least one timed repeat");
  check_pair(fb, table);
  const std::uint32_t d = table.num_dms, s = fb.setup.samples_per_second, c = fb.setup.channels;
  const dd_config kc = to_c(cfg, options);
  const dd_limits l = to_c(options.limits);
  check(dd_validate_config(&kc, d, s, &l));
  TuningRecord rec;
  rec.config = cfg;
  rec.dm_tile_depth = options.dm_tile_depth;
  rec.staging = options.staging;
  rec.flags = options.flags;
  rec.runs.resize(repeats);

  std::lock_guard<std::mutex> g(g_mu);
  dd_context* ctx = context(options.device);
  const std::uint64_t pitch = (static_cast<std::uint64_t>(fb.num_samples) + 3) & ~3ull;
  void *din = nullptr, *dsh = nullptr, *dout = nullptr;
  dd_plan* plan = nullptr;
  dd_status st = dd_device_malloc(ctx, pitch * c * 4, &din);
  if (st == DD_OK) st = dd_device_malloc(ctx, static_cast<std::uint64_t>(d) * c * 4, &dsh);
  if (st == DD_OK) st = dd_device_malloc(ctx, static_cast<std::uint64_t>(d) * s * 4, &dout);
  if (st == DD_OK)
    st = dd_upload_filterbank(ctx, static_cast<float*>(din), pitch, fb.data.data(), c,
                              fb.num_samples);
  if (st == DD_OK) st = dd_copy_h2d(ctx, dsh, table.shifts.data(), table.shifts.size() * 4);
  if (st == DD_OK)
    st = dd_plan_create(ctx, static_cast<std::uint32_t*>(dsh), c, d, s, fb.num_samples, pitch,
                        &kc, &l, &plan);
  if (st == DD_OK)
    st = dd_plan_time(plan, static_cast<float*>(din), static_cast<float*>(dout), s, 1, repeats,
                      rec.runs.data());
  if (st == DD_OK) {
    dd_plan_info info{};
    if (dd_plan_get_info(plan, &info) == DD_OK) rec.family = static_cast<Staging>(info.family);
  }
  dd_plan_destroy(plan);
  dd_device_free(ctx, din);
  dd_device_free(ctx, dsh);
  dd_device_free(ctx, dout);
  check(st);
  double total = 0.0;
  for (double x : rec.runs) total += x;
  rec.mean_time = total / repeats;
  const double resolution = 0.5e-6;
  rec.timer_warning = resolution > 0.01 * rec.mean_time;
  rec.gflops = static_cast<double>(d) * s * c / std::max(rec.mean_time, resolution) / 1e9;
  return rec;
}

namespace {
dd_tuning_record to_c(const TuningRecord& r) {
  dd_tuning_record c{};
  c.config = dd_config{r.config.items_time, r.config.items_dm, r.config.work_time,
                       r.config.work_dm,    r.dm_tile_depth,   static_cast<uint32_t>(r.staging),
                       r.flags};
  c.mean_time = r.mean_time;
  c.gflops = r.gflops;
  c.family = static_cast<uint32_t>(r.family);
  return c;
}
}  // namespace

std::size_t select_best(std::span<const TuningRecord> records) {
  if (records.empty()) throw std::invalid_argument("no records to select from");
  std::vector<dd_tuning_record> v;
  for (const auto& r : records) v.push_back(to_c(r));
  std::uint64_t best = 0;
  check(dd_select_best(v.data(), v.size(), &best));
  return static_cast<std::size_t>(best);
}

TuningStats compute_stats(std::span<const TuningRecord> records, std::size_t best_index) {
  if (records.empty()) throw std::invalid_argument("no records to summarize");
  std::vector<dd_tuning_record> v;
  for (const auto& r : records) v.push_back(to_c(r));
  dd_tuning_summary s{};
  check(dd_compute_stats(v.data(), v.size(), best_index, &s));
  TuningStats out;
  out.mean_gflops = s.mean_gflops;
  out.stddev_gflops = s.stddev_gflops;
  out.degenerate = s.degenerate != 0;
  if (!out.degenerate) {
    out.snr_optimum = s.snr_optimum;
    out.chebyshev_bound = s.chebyshev_bound;
  }
  return out;
}

namespace {
TuningResult sweep(const ObservationSetup& setup, std::uint32_t num_dms, const TuneOptions& o,
                   bool zero) {
  setup.validate();
  if (num_dms == 0) throw std::invalid_argument("need at least one trial DM");
  if (o.repeats == 0) throw std::invalid_argument("need at least one timed repeat");
  const dd_setup cs = to_c(setup);
  dd_tune_options to{};
  to.limits = to_c(o.limits);
  to.repeats = o.repeats;
  to.zero_dm = zero ? 1 : 0;
  to.seed = o.seed;
  to.space = o.full_reference_space ? 1 : 0;
  to.max_configs = o.max_configs;
  to.flush_l2 = o.flush_l2 ? 1 : 0;
  std::lock_guard<std::mutex> g(g_mu);
  dd_context* ctx = context(o.device);
  std::uint64_t n = 0;
  if (to.space == 1) {
    check(dd_enumerate_configs(num_dms, setup.samples_per_second, &to.limits, nullptr, 0, &n));
  } else {
    check(dd_enumerate_gpu_configs(ctx, &cs, num_dms, &to.limits, nullptr, 0, &n));
  }
  if (o.max_configs != 0 && n > o.max_configs) n = o.max_configs;
  std::vector<dd_tuning_record> recs(n);
  std::vector<double> runs(n * o.repeats);
  to.runs = runs.data();  // every timed run, the reference's runs_s
  dd_tuning_summary sum{};
  check(dd_tune(ctx, &cs, num_dms, &to, recs.data(), n, &sum));
  TuningResult r;
  r.setup = setup;
  r.num_dms = num_dms;
  r.zero_dm = zero;
  r.limits = o.limits;
  r.repeats = o.repeats;
  r.seed = o.seed;
  r.threads = 1;
  r.rng_id = kNoiseRngId;
  r.clock_resolution_s = sum.clock_resolution_s;
  for (std::uint64_t i = 0; i < sum.count; ++i) {
    const dd_tuning_record& c = recs[i];
    TuningRecord t;
    t.config = KernelConfig{c.config.items_time, c.config.items_dm, c.config.work_time,
                            c.config.work_dm};
    t.dm_tile_depth = c.config.dm_tile_depth;
    t.staging = static_cast<Staging>(c.config.staging);
    t.flags = c.config.flags;
    t.family = static_cast<Staging>(c.family);
    t.runs.assign(runs.begin() + static_cast<std::ptrdiff_t>(i * o.repeats),
                  runs.begin() + static_cast<std::ptrdiff_t>((i + 1) * o.repeats));
    t.mean_time = c.mean_time;
    t.gflops = c.gflops;
    t.timer_warning = c.timer_warning != 0;
    r.records.push_back(std::move(t));
  }
  r.best_index = static_cast<std::size_t>(sum.best_index);
  r.stats.mean_gflops = sum.mean_gflops;
  r.stats.stddev_gflops = sum.stddev_gflops;
  r.stats.degenerate = sum.degenerate != 0;
  if (!r.stats.degenerate) {
    r.stats.snr_optimum = sum.snr_optimum;
    r.stats.chebyshev_bound = sum.chebyshev_bound;
  }
  r.realtime_threshold_gflops = sum.realtime_threshold_gflops;
  r.realtime_pass = sum.realtime_pass != 0;
  return r;
}
}  // namespace

TuningResult tune(const ObservationSetup& setup, std::uint32_t num_dms, const TuneOptions& o) {
  return sweep(setup, num_dms, o, false);
}

TuningResult zero_dm_experiment(const ObservationSetup& setup, std::uint32_t num_dms,
                                const TuneOptions& o) {
  return sweep(setup, num_dms, o, true);
}

// best_fixed_config, reference tuner.cpp:218-261.
FixedConfigReport best_fixed_config(std::span<const TuningResult> results) {
  if (results.empty()) throw std::invalid_argument("no tuning results given");
  const ObservationSetup& first = results.front().setup;
  for (const TuningResult& r : results) {
    if (r.setup.name != first.name || r.setup.samples_per_second != first.samples_per_second ||
        r.setup.channels != first.channels)
      throw std::invalid_argument("tuning results mix different setups");
    if (r.records.empty()) throw std::invalid_argument("a tuning result holds no records");
  }
  // config identity = the reference 4-tuple plus every GPU knob (depth,
  // staging, flags): records differing only in stage shape or raster are
  // different configurations (tuner.cpp:218-261 keys on the whole config)
  struct Key {
    KernelConfig c;
    std::uint32_t depth, staging, flags;
    bool operator<(const Key& o) const {
      if (c != o.c) return c < o.c;
      if (depth != o.depth) return depth < o.depth;
      if (staging != o.staging) return staging < o.staging;
      return flags < o.flags;
    }
  };
  std::map<Key, std::vector<double>> by;
  for (std::size_t i = 0; i < results.size(); ++i)
    for (const TuningRecord& rec : results[i].records) {
      auto& v = by[Key{rec.config, rec.dm_tile_depth, static_cast<std::uint32_t>(rec.staging),
                       rec.flags}];
      if (v.size() == i) v.push_back(rec.gflops);
    }
  bool found = false;
  FixedConfigReport rep;
  for (const auto& [k, v] : by) {
    if (v.size() != results.size()) continue;
    double tot = 0.0;
    for (double g : v) tot += g;
    if (!found || tot > rep.total_gflops) {
      found = true;
      rep.config = k.c;
      rep.dm_tile_depth = k.depth;
      rep.staging = static_cast<Staging>(k.staging);
      rep.flags = k.flags;
      rep.total_gflops = tot;
      rep.fixed_gflops = v;
    }
  }
  if (!found) throw std::invalid_argument("no configuration is valid in every instance");
  for (std::size_t i = 0; i < results.size(); ++i)
    rep.speedup_over_fixed.push_back(results[i].best().gflops / rep.fixed_gflops[i]);
  return rep;
}

void register_schedule(const TuningResult& result) {
  if (result.records.empty()) throw std::invalid_argument("a tuning result holds no records");
  const TuningRecord& b = result.best();
  const dd_config c = to_c(b.config, b.exec_options());
  check(dd_schedule_set(result.setup.channels, result.setup.samples_per_second, result.num_dms,
                        &c));
}

std::vector<std::uint32_t> default_instances() {
  std::vector<std::uint32_t> v;
  for (std::uint32_t d = 2; d <= 4096; d *= 2) v.push_back(d);
  return v;
}

std::uint64_t estimate_instance_bytes(const ObservationSetup& setup, std::uint32_t num_dms) {
  const ProblemInstance p = instance_sizing(setup, num_dms);
  const unsigned __int128 total = static_cast<unsigned __int128>(setup.channels) * p.num_samples * 4 +
                                  static_cast<unsigned __int128>(num_dms) * setup.samples_per_second * 4 +
                                  static_cast<unsigned __int128>(num_dms) * setup.channels * 4;
  return total > ~std::uint64_t{0} ? ~std::uint64_t{0} : static_cast<std::uint64_t>(total);
}

// ------------------------------------------------------------- analysis
AiBounds ai_bounds(std::uint64_t d, std::uint64_t s, std::uint64_t c) {
  if (d == 0 || s == 0 || c == 0) throw std::invalid_argument("instance dimensions must all be positive");
  AiBounds b;
  b.reuse_bound = 1.0 / (4.0 * (1.0 / static_cast<double>(d) + 1.0 / static_cast<double>(s) +
                                1.0 / static_cast<double>(c)));
  return b;
}

MemoryTraffic kernel_traffic(const DelayTable& table, const KernelConfig& cfg,
                             std::uint32_t num_dms, std::uint32_t s) {
  const LoadCounts l = count_loads(table, cfg, num_dms, s);
  MemoryTraffic t;
  t.staged_loads = l.staged_loads;
  t.output_writes = static_cast<std::uint64_t>(num_dms) * s;
  t.delay_reads = static_cast<std::uint64_t>(num_dms) * table.setup.channels;
  return t;
}

double measured_ai(std::uint64_t flops, const MemoryTraffic& t) {
  const std::uint64_t e = t.staged_loads + t.output_writes + t.delay_reads;
  if (e == 0) throw std::invalid_argument("no memory traffic to divide by");
  return static_cast<double>(flops) / (4.0 * static_cast<double>(e));
}

double realtime_threshold_gflops(const ObservationSetup& setup, std::uint32_t num_dms) {
  setup.validate();
  if (num_dms == 0) throw std::invalid_argument("need at least one trial DM");
  return static_cast<double>(num_dms) * setup.samples_per_second * setup.channels / 1e9;
}

DeploymentPlan deployment_sizing(const ObservationSetup& setup, std::uint32_t num_dms,
                                 std::uint32_t beams, double t) {
  setup.validate();
  if (num_dms == 0) throw std::invalid_argument("need at least one trial DM");
  if (beams == 0) throw std::invalid_argument("need at least one beam");
  if (!std::isfinite(t) || t <= 0.0)
    throw std::invalid_argument("pass time must be a positive number of seconds");
  if (t >= 1.0)
    throw not_real_time_error("one pass takes " + std::to_string(t) +
                              " s; a device cannot keep up with even a single beam");
  DeploymentPlan plan;
  plan.beams_per_device = static_cast<std::uint32_t>(1.0 / t);
  plan.devices = (static_cast<std::uint64_t>(beams) + plan.beams_per_device - 1) / plan.beams_per_device;
  return plan;
}

std::span<const DevicePeaks> reference_devices() {
  // the paper's Table 1 cards (GFLOP/s, GB/s)
  static const DevicePeaks kDevices[] = {
      {"AMD HD7970", 3788.0, 264.0},        {"Intel Xeon Phi 5110P", 2022.0, 320.0},
      {"NVIDIA GTX 680", 3090.0, 192.0},    {"NVIDIA K20", 3519.0, 208.0},
      {"NVIDIA GTX Titan", 4500.0, 288.0},
  };
  return kDevices;
}

RooflineVerdict classify_roofline(double ai, double peak_gflops, double peak_gbs) {
  if (!std::isfinite(ai) || ai <= 0.0)
    throw std::invalid_argument("arithmetic intensity must be positive");
  if (!std::isfinite(peak_gflops) || peak_gflops <= 0.0 || !std::isfinite(peak_gbs) ||
      peak_gbs <= 0.0)
    throw std::invalid_argument("device peaks must be positive");
  RooflineVerdict v;
  v.ridge_flop_per_byte = peak_gflops / peak_gbs;
  v.memory_bound = ai < v.ridge_flop_per_byte;
  v.attainable_gflops = std::min(peak_gflops, ai * peak_gbs);
  return v;
}

std::vector<HistogramBin> make_histogram(const TuningResult& result, std::size_t bins) {
  if (bins == 0) throw std::invalid_argument("need at least one histogram bin");
  if (result.records.empty()) throw std::invalid_argument("no records to bin");
  double lo = result.records.front().gflops, hi = lo;
  for (const TuningRecord& r : result.records) {
    lo = std::min(lo, r.gflops);
    hi = std::max(hi, r.gflops);
  }
  const double width = (hi - lo) / static_cast<double>(bins);
  std::vector<HistogramBin> h(bins);
  for (std::size_t i = 0; i < bins; ++i) {
    h[i].lo = lo + width * static_cast<double>(i);
    h[i].hi = i + 1 == bins ? hi : lo + width * static_cast<double>(i + 1);
  }
  for (const TuningRecord& r : result.records) {
    std::size_t i = 0;  // a flat population lands in the first bin
    if (width > 0.0) i = std::min(static_cast<std::size_t>((r.gflops - lo) / width), bins - 1);
    ++h[i].count;
  }
  return h;
}

}  // namespace dedisp
