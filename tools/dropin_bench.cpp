// dropin_bench.cpp -- the end-to-end path a reference client takes: code
// written against the reference's dedisp API (dedisperse_tiled_into with
// host std::vector buffers and default ExecOptions) linked against
// libdedisp_b200.so instead of the reference library.  Each timed call
// uploads the filterbank, runs the tuned schedule and downloads the whole
// output into the caller's vector (pageable host memory, as the reference
// API hands it over).  Prints one JSON line.
//
//   g++ -std=c++20 -O2 -Iinclude tools/dropin_bench.cpp -Lpaper_1601_05052_b200 \
//       -ldedisp_b200 -Wl,-rpath,$PWD/paper_1601_05052_b200 -o /tmp/dropin_bench
//   /tmp/dropin_bench [Apertif|LOFAR] [num_dms] [repeats]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dedisp/b200.hpp"

int main(int argc, char** argv) {
  const std::string name = argc > 1 ? argv[1] : "Apertif";
  const std::uint32_t d = argc > 2 ? static_cast<std::uint32_t>(std::atoi(argv[2])) : 4096u;
  const int repeats = argc > 3 ? std::atoi(argv[3]) : 10;
  const dedisp::ObservationSetup* setup = dedisp::find_builtin(name);
  if (setup == nullptr) return 2;
  const auto table = dedisp::build_delay_table(*setup, d);
  const auto inst = dedisp::instance_sizing(*setup, d);
  const auto fb = dedisp::noise_filterbank(*setup, static_cast<std::uint32_t>(inst.num_samples),
                                           1.0f, 1);
  // the reference's CPU config for Apertif (a reference-valid 4-tuple); the
  // default ExecOptions let the library run the instance's tuned schedule
  const dedisp::KernelConfig cfg =
      name == "Apertif" ? dedisp::KernelConfig{125, 8, 8, 1} : dedisp::KernelConfig{1000, 1, 1, 4};
  dedisp::DedispersedSeries out;
  dedisp::dedisperse_tiled_into(out, fb, table, cfg);  // warm-up: buffers, plan
  double best = 1e30, total = 0.0;
  for (int i = 0; i < repeats; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    dedisp::dedisperse_tiled_into(out, fb, table, cfg);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    total += s;
    best = s < best ? s : best;
  }
  const double mean = total / repeats;
  std::uint64_t h = 0;
  dd_fingerprint(out.data.data(), out.data.size() * 4, &h);
  dd_config ran{};
  int builtin = 0;
  dd_schedule_get(setup->channels, setup->samples_per_second, d, &ran, &builtin);
  const double flop = static_cast<double>(inst.flop);
  std::printf(
      "{\"path\": \"dedisp::dedisperse_tiled_into (reference C++ API, pageable std::vector "
      "buffers, default ExecOptions)\", \"setup\": \"%s\", \"num_dms\": %u, \"repeats\": %d, "
      "\"mean_ms\": %.3f, \"best_ms\": %.3f, \"gflops\": %.1f, \"h2d_bytes\": %llu, "
      "\"d2h_bytes\": %llu, \"fingerprint\": \"%016llx\", \"schedule\": [%u, %u, %u, %u, %u, %u, "
      "%u], \"schedule_builtin\": %d}\n",
      name.c_str(), d, repeats, mean * 1e3, best * 1e3, flop / mean / 1e9,
      static_cast<unsigned long long>(fb.data.size() * 4),
      static_cast<unsigned long long>(out.data.size() * 4), static_cast<unsigned long long>(h),
      ran.items_time, ran.items_dm, ran.work_time, ran.work_dm, ran.dm_tile_depth, ran.staging,
      ran.flags, builtin);
  return 0;
}
