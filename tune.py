"""Auto-tuner front end (the reference CLI's `tune` subcommand,
dedisp_tune.cpp:464-535, on the device).

    python tune.py --setup Apertif --dms 4096 [--dms 64 ...] [--repeats 10]
                   [--space gpu|reference] [--max-configs N] [--zero-dm]

For every instance it benchmarks every configuration of the chosen space on
the GPU (1 warm-up + `repeats` CUDA-event-timed runs, tuner.cpp:136-170),
selects the optimum (tuner.cpp:172-179), computes the population statistics
(tuner.cpp:181-206), and writes tuning/<setup>_<d>.json.  With several
instances it also reports best_fixed_config and the tuned-vs-fixed speedups
(tuner.cpp:218-261; BASELINE config 5) in tuning/<setup>_summary.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1601_05052_b200 import api  # noqa: E402


def record_json(r: api.TuningRecord) -> dict:
    c = r.config
    return {"items_time": c.items_time, "items_dm": c.items_dm, "work_time": c.work_time,
            "work_dm": c.work_dm, "dm_tile_depth": r.dm_tile_depth, "staging": r.staging,
            "flags": r.flags, "stage_channels": r.stage_channels,
            "family": r.family, "mean_time": r.mean_time, "gflops": r.gflops,
            "timer_warning": r.timer_warning}


def result_json(res: api.TuningResult, hbm_gbs: float, seconds: float) -> dict:
    d, s, c = res.num_dms, res.setup.samples_per_second, res.setup.channels
    best = record_json(res.best())
    best["hbm_roofline_gflops"] = api.roofline_gflops(d, s, c, hbm_gbs)
    best["roofline_frac"] = best["gflops"] / best["hbm_roofline_gflops"]
    return {
        "schema": "dedisp-tuning-result/1+b200",
        "setup": res.setup.__dict__, "num_dms": d, "zero_dm": res.zero_dm,
        "limits": res.limits.__dict__, "repeats": res.repeats, "seed": res.seed,
        "rng_id": res.rng_id, "clock": "cuda events", "clock_resolution_s": res.clock_resolution_s,
        "best_index": res.best_index, "best": best,
        "stats": res.stats.__dict__,
        "realtime_threshold_gflops": res.realtime_threshold_gflops,
        "realtime_pass": res.realtime_pass, "sweep_seconds": seconds,
        "records": [record_json(r) for r in res.records],
    }


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--setup", default="Apertif")
    p.add_argument("--dms", type=int, action="append")
    p.add_argument("--repeats", type=int, default=10)
    p.add_argument("--space", default="gpu", choices=["gpu", "reference"])
    p.add_argument("--max-configs", type=int, default=0)
    p.add_argument("--zero-dm", action="store_true")
    p.add_argument("--out", default=os.path.join(ROOT, "tuning"))
    a = p.parse_args()
    setup = api.find_builtin(a.setup)
    dms = a.dms or api.default_instances()
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    os.makedirs(a.out, exist_ok=True)
    results = []
    for d in dms:
        t0 = time.time()
        fn = api.zero_dm_experiment if a.zero_dm else api.tune
        res = fn(setup, d, repeats=a.repeats, full_reference_space=a.space == "reference",
                 max_configs=a.max_configs)
        dt = time.time() - t0
        results.append(res)
        j = result_json(res, hbm, dt)
        name = f"{setup.name.lower()}_{d}{'_zero' if a.zero_dm else ''}.json"
        with open(os.path.join(a.out, name), "w") as f:
            json.dump(j, f, indent=1)
        b = j["best"]
        print(f"{setup.name} d={d}: {len(res.records)} configs in {dt:.1f}s; best "
              f"({b['items_time']},{b['items_dm']},{b['work_time']},{b['work_dm']}) "
              f"depth={b['dm_tile_depth']} {b['staging']} cps={b['stage_channels']}: "
              f"{b['gflops']:.1f} GFLOP/s "
              f"({b['mean_time'] * 1e3:.3f} ms, {b['roofline_frac']:.2f}x HBM roofline); "
              f"snr={res.stats.snr_optimum}", flush=True)
    if len(results) > 1:
        rep = api.best_fixed_config(results)
        k, depth, staging, flags = rep.config
        summ = {"setup": setup.name, "instances": dms,
                "best_fixed": {"items_time": k.items_time, "items_dm": k.items_dm,
                               "work_time": k.work_time, "work_dm": k.work_dm,
                               "dm_tile_depth": depth, "staging": staging, "flags": flags},
                "fixed_gflops": rep.fixed_gflops, "tuned_gflops": [r.best().gflops for r in results],
                "speedup_over_fixed": rep.speedup_over_fixed}
        with open(os.path.join(a.out, f"{setup.name.lower()}_summary"
                               f"{'_zero' if a.zero_dm else ''}.json"), "w") as f:
            json.dump(summ, f, indent=1)
        print("best fixed:", summ["best_fixed"], "speedups:",
              [round(x, 3) for x in rep.speedup_over_fixed])


if __name__ == "__main__":
    main()
