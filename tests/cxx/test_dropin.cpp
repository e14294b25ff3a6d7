// C++ drop-in test: code written against the reference's dedisp API
// (test_kernels.cpp / test_setup.cpp style) compiled against
// include/dedisp/b200.hpp and linked with libdedisp_b200.so.  The CPU oracle
// (oracle/liboracle.so, test infrastructure) is the checker.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dedisp/b200.hpp"

extern "C" int or_dedisperse_reference(const float* in, uint32_t channels, uint64_t t,
                                       const uint32_t* shifts, uint32_t num_dms, uint32_t s,
                                       float* out);

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
  }
  return false;
}

static dedisp::ObservationSetup mini(std::uint32_t rate, std::uint32_t ch, double step) {
  dedisp::ObservationSetup s;
  s.name = "mini";
  s.samples_per_second = rate;
  s.channels = ch;
  s.f_min = 100.0;
  s.channel_width = 25.0;
  s.dm_first = 0.0;
  s.dm_step = step;
  return s;
}

static bool same(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

static dedisp::TuningRecord record_with(dedisp::KernelConfig k, double gflops,
                                        std::uint32_t flags) {
  dedisp::TuningRecord r;  // test_tuner.cpp:18-25 style fake record
  r.config = k;
  r.gflops = gflops;
  r.mean_time = 1.0 / gflops;
  r.staging = dedisp::Staging::SharedMemory;
  r.flags = flags;
  return r;
}

static std::string hex64(std::uint64_t v) {
  char b[17];
  std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(v));
  return b;
}

int main(int argc, char** argv) {
  // argv[1] (optional): the reference's fingerprint of the Apertif d=4096
  // output (tests/golden/golden.json), for the full-size drop-in check
  // setup.cpp known answers (test_setup.cpp:75-88, :130-137)
  const auto* apertif = dedisp::find_builtin("Apertif");
  CHECK(apertif != nullptr);
  const auto t16 = dedisp::build_delay_table(*apertif, 16);
  CHECK(t16.at(0, 1) == 3);
  CHECK(dedisp::instance_sizing(*apertif, 1).flop == 20480000u);
  CHECK(throws<dedisp::capacity_error>([&] { dedisp::build_delay_table(*apertif, 4096, 1024); }));
  CHECK(throws<std::invalid_argument>([&] { dedisp::delay_seconds(1.0, 1800.0, 1720.0); }));

  // tiled == reference for every valid config (test_kernels.cpp:116-139)
  const auto setup = mini(48, 6, 0.5);
  const std::uint32_t d = 12;
  const auto table = dedisp::build_delay_table(setup, d);
  const auto inst = dedisp::instance_sizing(setup, d);
  const auto fb = dedisp::noise_filterbank(setup, static_cast<std::uint32_t>(inst.num_samples), 1.0f, 99);
  std::vector<float> oracle(static_cast<std::size_t>(d) * 48);
  CHECK(or_dedisperse_reference(fb.data.data(), 6, fb.num_samples, table.shifts.data(), d, 48,
                                oracle.data()) == 0);
  const auto ref = dedisp::dedisperse_reference(fb, table);
  CHECK(same(ref.data, oracle));
  dedisp::KernelLimits limits{64, 32};
  const auto configs = dedisp::enumerate_configs(d, 48, limits);
  CHECK(configs.size() > 20);
  for (const auto& cfg : configs) {
    dedisp::ExecOptions o;
    o.limits = limits;
    CHECK(same(dedisp::dedisperse_tiled(fb, table, cfg, o).data, oracle));
  }

  // counters (test_kernels.cpp:203-227) and rejection (:183-201)
  dedisp::KernelStats stats;
  dedisp::ExecOptions o;
  o.stats = &stats;
  const dedisp::KernelConfig k{8, 2, 2, 2};
  const auto setup6 = mini(64, 6, 0.5);
  const auto table6 = dedisp::build_delay_table(setup6, 8);
  const auto fb6 = dedisp::noise_filterbank(setup6, static_cast<std::uint32_t>(dedisp::instance_sizing(setup6, 8).num_samples), 1.0f, 1);
  (void)dedisp::dedisperse_tiled(fb6, table6, k, o);
  CHECK(stats.flop_additions.load() == 8ull * 64 * 6);
  CHECK(stats.staged_loads.load() == dedisp::count_loads(table6, k, 8, 64).staged_loads);
  CHECK(throws<std::invalid_argument>([&] { dedisp::dedisperse_tiled(fb6, table6, {3, 1, 1, 1}); }));

  // the tuner (tuner.cpp:43-99) on the device
  dedisp::TuneOptions to;
  to.repeats = 2;
  to.max_configs = 6;
  const auto res = dedisp::tune(*apertif, 64, to);
  CHECK(res.records.size() == 6);
  CHECK(res.best().gflops > 0.0);

  CHECK(res.records.front().runs.size() == 2);  // every timed run kept (runs_s)

  // benchmark_config (tuner.cpp:136-170): a replayable record
  {
    dedisp::ExecOptions bo;
    bo.staging = dedisp::Staging::SharedMemory;
    bo.flags = 8u << DD_CONFIG_CPS_SHIFT;
    const auto rec = dedisp::benchmark_config(fb6, table6, k, 3, bo);
    CHECK(rec.runs.size() == 3);
    CHECK(rec.mean_time > 0.0 && rec.gflops > 0.0);
    CHECK(rec.flags == bo.flags && rec.staging == dedisp::Staging::SharedMemory);
    CHECK(rec.family == dedisp::Staging::SharedMemory);
    CHECK(same(dedisp::dedisperse_tiled(fb6, table6, k, rec.exec_options()).data,
               dedisp::dedisperse_reference(fb6, table6).data));
    CHECK(throws<std::invalid_argument>([&] { dedisp::benchmark_config(fb6, table6, k, 0); }));
  }

  // best_fixed_config (tuner.cpp:218-261) keys on the whole configuration:
  // two records of one 4-tuple that differ only in flags are two configs
  {
    const dedisp::KernelConfig a{32, 1, 1, 1}, b{64, 1, 1, 1};
    auto mk = [&](std::vector<dedisp::TuningRecord> recs) {
      dedisp::TuningResult r;
      r.setup = *apertif;
      r.num_dms = 2;
      r.records = std::move(recs);
      r.best_index = dedisp::select_best(r.records);
      return r;
    };
    std::vector<dedisp::TuningResult> results = {
        mk({record_with(a, 10.0, 0), record_with(a, 30.0, 0x800), record_with(b, 20.0, 0)}),
        mk({record_with(a, 12.0, 0), record_with(b, 25.0, 0)}),
    };
    CHECK(results[0].best().flags == 0x800);  // select_best keeps the flags
    const auto rep = dedisp::best_fixed_config(results);
    CHECK(rep.config == b && rep.flags == 0);  // (a, 0x800) is not valid everywhere
    CHECK(rep.total_gflops == 45.0);
    CHECK(rep.speedup_over_fixed.size() == 2 && rep.speedup_over_fixed[0] == 1.5);
    results[1].records.push_back(record_with(a, 40.0, 0x800));
    results[1].best_index = dedisp::select_best(results[1].records);
    const auto rep2 = dedisp::best_fixed_config(results);
    CHECK(rep2.config == a && rep2.flags == 0x800 && rep2.total_gflops == 70.0);
  }

  // tuned dispatch: default ExecOptions (staging Auto, no flags) run the
  // instance's tuned schedule; a registered one takes precedence
  {
    const auto t64 = dedisp::build_delay_table(*apertif, 64);
    const auto fb64 = dedisp::noise_filterbank(
        *apertif, static_cast<std::uint32_t>(dedisp::instance_sizing(*apertif, 64).num_samples),
        1.0f, 1);
    const auto ref64 = dedisp::dedisperse_reference(fb64, t64);
    dd_config ran{};
    int builtin = 0;
    CHECK(dd_schedule_get(1024, 20000, 64, &ran, &builtin) == DD_OK && builtin == 1);
    CHECK(same(dedisp::dedisperse_tiled(fb64, t64, {32, 8, 1, 8}).data, ref64.data));
    dd_config last{};
    dd_context* ctx0 = nullptr;
    (void)ctx0;
    dedisp::TuningResult tr;
    tr.setup = *apertif;
    tr.num_dms = 64;
    auto rec = record_with({32, 8, 1, 8}, 1.0, 8u << DD_CONFIG_CPS_SHIFT);
    rec.staging = dedisp::Staging::RegisterWindow;
    rec.config = {32, 4, 25, 4};
    tr.records = {rec};
    tr.best_index = 0;
    dedisp::register_schedule(tr);
    CHECK(dd_schedule_get(1024, 20000, 64, &last, &builtin) == DD_OK && builtin == 0);
    CHECK(last.staging == DD_STAGING_REGWIN && last.work_time == 25);
    CHECK(same(dedisp::dedisperse_tiled(fb64, t64, {32, 8, 1, 8}).data, ref64.data));
    CHECK(dd_schedule_set(1024, 20000, 64, nullptr) == DD_OK);  // forget it again
    // an explicit staging runs exactly the config asked for
    dedisp::ExecOptions so;
    so.staging = dedisp::Staging::SharedMemory;
    CHECK(same(dedisp::dedisperse_tiled(fb64, t64, {32, 8, 1, 8}, so).data, ref64.data));
  }

  // full size through the drop-in: Apertif d=4096 with default options runs
  // the tuned TMEM-window kernel (K5) and reproduces the reference's bits
  if (argc > 1) {
    const auto t4k = dedisp::build_delay_table(*apertif, 4096);
    const auto fb4k = dedisp::noise_filterbank(
        *apertif, static_cast<std::uint32_t>(dedisp::instance_sizing(*apertif, 4096).num_samples),
        1.0f, 1);
    dedisp::DedispersedSeries out;
    dedisp::dedisperse_tiled_into(out, fb4k, t4k, {125, 8, 8, 1});  // the reference CPU config
    std::uint64_t h = 0;
    CHECK(dd_fingerprint(out.data.data(), out.data.size() * 4, &h) == DD_OK);
    CHECK(hex64(h) == argv[1]);
    dd_config cfg{};
    int b = 0;
    CHECK(dd_schedule_get(1024, 20000, 4096, &cfg, &b) == DD_OK && cfg.staging == DD_STAGING_TMEM);
    std::printf("dropin: Apertif d=4096 fingerprint %s (golden %s)\n", hex64(h).c_str(), argv[1]);
  }

  std::printf(failures ? "dropin: %d failure(s)\n" : "dropin: ok\n", failures);
  return failures ? 1 : 0;
}
