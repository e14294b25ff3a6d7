// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI face over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libdedisp_ref.so).  No reference source is
// copied here: this file only includes the reference's public headers and
// forwards to its functions so that Python (tests/, bench.py --impl
// reference) can call them through ctypes.  Entry points cited:
//   build_delay_table / build_zero_delay_table  setup.hpp:75-81
//   instance_sizing                             setup.hpp:85
//   noise_filterbank                            filterbank.hpp:59-60
//   dedisperse_reference_into                   kernels.hpp:90-91
//   dedisperse_tiled_into                       kernels.hpp:102-104
//   count_loads                                 kernels.hpp:114-115
//   enumerate_configs                           tuner.hpp:61-63
//   parse_sigproc                               filterbank.hpp:69 (sigproc.cpp:83-191)
//   tuning_result_from_json / _to_json          report_io.hpp:11-14 (report_io.cpp:58-157)
#include <cstdint>
#include <span>
#include <string>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>

#include "dedisp/errors.hpp"
#include "dedisp/filterbank.hpp"
#include "dedisp/kernels.hpp"
#include "dedisp/setup.hpp"
#include "dedisp/thread_pool.hpp"
#include "dedisp/tuner.hpp"
#ifdef REF_HAVE_JSON
#include "dedisp/report_io.hpp"
#endif

namespace {

struct ref_setup {
  std::uint32_t samples_per_second;
  std::uint32_t channels;
  double f_min, channel_width, dm_first, dm_step;
};

struct ref_config {
  std::uint32_t items_time, items_dm, work_time, work_dm;
};

dedisp::ObservationSetup to_setup(const ref_setup* s) {
  dedisp::ObservationSetup o;
  o.name = "shim";
  o.samples_per_second = s->samples_per_second;
  o.channels = s->channels;
  o.f_min = s->f_min;
  o.channel_width = s->channel_width;
  o.dm_first = s->dm_first;
  o.dm_step = s->dm_step;
  return o;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const dedisp::capacity_error&) {
    return 2;
  } catch (...) {
    return 3;
  }
}

// The reference kernels take whole value types; these wrap raw buffers.
dedisp::Filterbank wrap_fb(const ref_setup* s, const float* in, std::uint64_t t) {
  dedisp::Filterbank fb;
  fb.setup = to_setup(s);
  fb.num_samples = static_cast<std::uint32_t>(t);
  fb.data.assign(in, in + static_cast<std::size_t>(s->channels) * t);
  return fb;
}

dedisp::DelayTable wrap_table(const ref_setup* s, const std::uint32_t* shifts,
                              std::uint32_t num_dms) {
  dedisp::DelayTable table;
  table.setup = to_setup(s);
  table.num_dms = num_dms;
  table.shifts.assign(shifts, shifts + static_cast<std::size_t>(num_dms) * s->channels);
  std::uint32_t mx = 0;
  for (std::uint32_t v : table.shifts) mx = v > mx ? v : mx;
  table.max_delay = mx;
  return table;
}

}  // namespace

extern "C" {

int ref_build_delay_table(const ref_setup* s, std::uint32_t num_dms, std::uint64_t cap,
                          int zero, std::uint32_t* shifts, std::uint32_t* max_delay) {
  return guarded([&] {
    const dedisp::DelayTable t = zero ? dedisp::build_zero_delay_table(to_setup(s), num_dms, cap)
                                      : dedisp::build_delay_table(to_setup(s), num_dms, cap);
    std::memcpy(shifts, t.shifts.data(), t.shifts.size() * sizeof(std::uint32_t));
    *max_delay = t.max_delay;
  });
}

int ref_instance_sizing(const ref_setup* s, std::uint32_t num_dms, std::uint64_t* num_samples,
                        std::uint64_t* flop, std::uint32_t* max_delay) {
  return guarded([&] {
    const dedisp::ProblemInstance p = dedisp::instance_sizing(to_setup(s), num_dms);
    *num_samples = p.num_samples;
    *flop = p.flop;
    *max_delay = p.max_delay;
  });
}

int ref_noise_filterbank(const ref_setup* s, std::uint32_t num_samples, float sigma,
                         std::uint64_t seed, float* out) {
  return guarded([&] {
    const dedisp::Filterbank fb = dedisp::noise_filterbank(to_setup(s), num_samples, sigma, seed);
    std::memcpy(out, fb.data.data(), fb.data.size() * sizeof(float));
  });
}

int ref_dedisperse_reference(const ref_setup* s, const float* in, std::uint64_t t,
                             const std::uint32_t* shifts, std::uint32_t num_dms, float* out) {
  return guarded([&] {
    const dedisp::Filterbank fb = wrap_fb(s, in, t);
    const dedisp::DelayTable table = wrap_table(s, shifts, num_dms);
    dedisp::DedispersedSeries o;
    dedisp::dedisperse_reference_into(o, fb, table);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

// Persistent pool + prepared inputs so timed CPU-baseline runs exclude the
// wrapping copies, exactly as the reference tuner times only
// dedisperse_tiled_into (tuner.cpp:151-159).
struct ref_job {
  dedisp::Filterbank fb;
  dedisp::DelayTable table;
  dedisp::DedispersedSeries out;
  dedisp::ThreadPool* pool = nullptr;
};

void* ref_job_create(const ref_setup* s, const float* in, std::uint64_t t,
                     const std::uint32_t* shifts, std::uint32_t num_dms, int threads) {
  try {
    auto* j = new ref_job;
    j->fb = wrap_fb(s, in, t);
    j->table = wrap_table(s, shifts, num_dms);
    j->pool = new dedisp::ThreadPool(threads > 0 ? static_cast<unsigned>(threads) : 0u);
    return j;
  } catch (...) {
    return nullptr;
  }
}

int ref_job_threads(void* job) {
  return static_cast<int>(static_cast<ref_job*>(job)->pool->worker_count());
}

int ref_job_run_tiled(void* job, const ref_config* k) {
  auto* j = static_cast<ref_job*>(job);
  return guarded([&] {
    dedisp::ExecOptions opt;
    opt.pool = j->pool;
    dedisp::KernelConfig cfg{k->items_time, k->items_dm, k->work_time, k->work_dm};
    dedisp::dedisperse_tiled_into(j->out, j->fb, j->table, cfg, opt);
  });
}

int ref_job_run_reference(void* job) {
  auto* j = static_cast<ref_job*>(job);
  return guarded([&] { dedisp::dedisperse_reference_into(j->out, j->fb, j->table); });
}

const float* ref_job_output(void* job) { return static_cast<ref_job*>(job)->out.data.data(); }

void ref_job_destroy(void* job) {
  auto* j = static_cast<ref_job*>(job);
  delete j->pool;
  delete j;
}

int ref_dedisperse_tiled(const ref_setup* s, const float* in, std::uint64_t t,
                         const std::uint32_t* shifts, std::uint32_t num_dms, const ref_config* k,
                         int threads, float* out) {
  return guarded([&] {
    const dedisp::Filterbank fb = wrap_fb(s, in, t);
    const dedisp::DelayTable table = wrap_table(s, shifts, num_dms);
    dedisp::ExecOptions opt;
    opt.threads = threads;
    dedisp::KernelConfig cfg{k->items_time, k->items_dm, k->work_time, k->work_dm};
    dedisp::DedispersedSeries o;
    dedisp::dedisperse_tiled_into(o, fb, table, cfg, opt);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

int ref_count_loads(const ref_setup* s, const std::uint32_t* shifts, std::uint32_t num_dms,
                    const ref_config* k, std::uint64_t* staged, std::uint64_t* ideal) {
  return guarded([&] {
    const dedisp::DelayTable table = wrap_table(s, shifts, num_dms);
    dedisp::KernelConfig cfg{k->items_time, k->items_dm, k->work_time, k->work_dm};
    const dedisp::LoadCounts c = dedisp::count_loads(table, cfg, num_dms, s->samples_per_second);
    *staged = c.staged_loads;
    *ideal = c.ideal_loads;
  });
}

std::int64_t ref_enumerate_configs(std::uint32_t num_dms, std::uint32_t s,
                                   std::uint32_t max_block_items, std::uint32_t max_accumulators,
                                   ref_config* out, std::uint64_t cap) {
  try {
    dedisp::KernelLimits lim{max_block_items, max_accumulators};
    const auto v = dedisp::enumerate_configs(num_dms, s, lim);
    for (std::size_t i = 0; i < v.size() && i < cap; ++i)
      out[i] = ref_config{v[i].items_time, v[i].items_dm, v[i].work_time, v[i].work_dm};
    return static_cast<std::int64_t>(v.size());
  } catch (...) {
    return -1;
  }
}

// parse_sigproc over an in-memory stream.  Returns 0 and the parsed
// channel-major data (lowest channel first) when `out` holds channels x
// samples floats (call once with out = NULL for the sizes); 4 on a
// format_error, whose byte offset lands in *bad_offset.
int ref_parse_sigproc(const std::uint8_t* bytes, std::uint64_t n, std::uint32_t* channels,
                      std::uint64_t* samples, float* out, std::uint64_t* bad_offset,
                      double* f_min, double* channel_width, std::uint32_t* rate) {
  try {
    const dedisp::Filterbank fb = dedisp::parse_sigproc(std::span<const std::uint8_t>(bytes, n));
    *channels = fb.setup.channels;
    *samples = fb.num_samples;
    *f_min = fb.setup.f_min;
    *channel_width = fb.setup.channel_width;
    *rate = fb.setup.samples_per_second;
    if (out != nullptr) std::memcpy(out, fb.data.data(), fb.data.size() * sizeof(float));
    return 0;
  } catch (const dedisp::format_error& e) {
    *bad_offset = e.byte_offset();
    return 4;
  } catch (...) {
    return 3;
  }
}

#ifdef REF_HAVE_JSON
// tuning_result_from_json, then a summary of what the reference read and
// its own re-serialisation (tuning_result_to_json) into `json_out`
// (capacity cap; *json_len = the needed size).  Returns 4 on format_error.
int ref_tuning_roundtrip(const char* text, std::uint32_t* num_records, std::uint64_t* best_index,
                         std::uint32_t* best_config, double* best_gflops,
                         std::uint32_t* num_dms, char* json_out, std::uint64_t cap,
                         std::uint64_t* json_len) {
  try {
    const dedisp::TuningResult r = dedisp::tuning_result_from_json(text);
    *num_records = static_cast<std::uint32_t>(r.records.size());
    *best_index = r.best_index;
    const dedisp::TuningRecord& b = r.best();
    best_config[0] = b.config.items_time;
    best_config[1] = b.config.items_dm;
    best_config[2] = b.config.work_time;
    best_config[3] = b.config.work_dm;
    *best_gflops = b.gflops;
    *num_dms = r.num_dms;
    const std::string j = dedisp::tuning_result_to_json(r);
    *json_len = j.size();
    if (json_out != nullptr && cap > 0) {
      const std::size_t k = j.size() < cap - 1 ? j.size() : static_cast<std::size_t>(cap - 1);
      std::memcpy(json_out, j.data(), k);
      json_out[k] = 0;
    }
    return 0;
  } catch (const dedisp::format_error&) {
    return 4;
  } catch (...) {
    return 3;
  }
}
#endif

}  // extern "C"
