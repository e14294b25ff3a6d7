// C++ drop-in test: code written against the reference's dedisp API
// (test_kernels.cpp / test_setup.cpp style) compiled against
// include/dedisp/b200.hpp and linked with libdedisp_b200.so.  The CPU oracle
// (oracle/liboracle.so, test infrastructure) is the checker.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
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

int main() {
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

  std::printf(failures ? "dropin: %d failure(s)\n" : "dropin: ok\n", failures);
  return failures ? 1 : 0;
}
