// C++ drop-in, analysis layer (no device needed): the reference's
// analysis.hpp / tuner.hpp helpers through include/dedisp/b200.hpp, with the
// known answers of proj/tests/test_analysis.cpp and test_tuner.cpp.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "dedisp/b200.hpp"

static int failures = 0;
#define CHECK(c)                                               \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                              \
    }                                                          \
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

static dedisp::TuningRecord rec(double g) {
  dedisp::TuningRecord r;
  r.config = {1, 1, 1, 1};
  r.gflops = g;
  return r;
}

int main() {
  const dedisp::ObservationSetup* ap = dedisp::find_builtin("Apertif");
  CHECK(ap != nullptr);
  // test_analysis.cpp:102-120
  const dedisp::DeploymentPlan p = dedisp::deployment_sizing(*ap, 2000, 450, 0.106);
  CHECK(p.beams_per_device == 9 && p.devices == 50);
  CHECK(dedisp::deployment_sizing(*ap, 2000, 9, 0.106).devices == 1);
  CHECK(dedisp::deployment_sizing(*ap, 2000, 10, 0.106).devices == 2);
  CHECK(dedisp::deployment_sizing(*ap, 2000, 450, 0.5).beams_per_device == 2);
  CHECK(throws<dedisp::not_real_time_error>([&] { dedisp::deployment_sizing(*ap, 2000, 450, 1.0); }));
  CHECK(throws<std::invalid_argument>([&] { dedisp::deployment_sizing(*ap, 2000, 0, 0.106); }));
  CHECK(throws<std::invalid_argument>([&] { dedisp::deployment_sizing(*ap, 2000, 450, 0.0); }));
  // test_analysis.cpp:122-140
  const auto devs = dedisp::reference_devices();
  CHECK(devs.size() == 5 && devs[0].name == "AMD HD7970" && devs[0].peak_gflops == 3788.0 &&
        devs[4].name == "NVIDIA GTX Titan" && devs[4].peak_gbs == 288.0);
  const dedisp::RooflineVerdict v = dedisp::classify_roofline(0.25, 3788.0, 264.0);
  CHECK(v.memory_bound && std::fabs(v.attainable_gflops - 66.0) < 1e-9);
  CHECK(!dedisp::classify_roofline(100.0, 3788.0, 264.0).memory_bound);
  CHECK(throws<std::invalid_argument>([] { dedisp::classify_roofline(0.0, 1.0, 1.0); }));
  // test_tuner.cpp:255-270
  dedisp::TuningResult r;
  for (double g : {1.0, 2.0, 3.0, 4.0}) r.records.push_back(rec(g));
  const auto bins = dedisp::make_histogram(r, 3);
  CHECK(bins.size() == 3 && std::fabs(bins[0].lo - 1.0) < 1e-12 && std::fabs(bins[2].hi - 4.0) < 1e-12);
  CHECK(bins[0].count == 1 && bins[1].count == 1 && bins[2].count == 2);
  dedisp::TuningResult flat;
  for (int i = 0; i < 3; ++i) flat.records.push_back(rec(5.0));
  std::size_t total = 0;
  for (const auto& b : dedisp::make_histogram(flat, 4)) total += b.count;
  CHECK(total == 3);
  CHECK(throws<std::invalid_argument>([&] { dedisp::make_histogram(flat, 0); }));
  // test_analysis.cpp:12-28
  CHECK(std::fabs(dedisp::ai_bounds(2048, 20000, 1024).reuse_bound - 165.03) < 0.02);
  CHECK(std::fabs(dedisp::realtime_threshold_gflops(*ap, 2000) - 40.96) < 1e-9);
  if (failures == 0) std::printf("analysis: ok\n");
  return failures == 0 ? 0 : 1;
}
