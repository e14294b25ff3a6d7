"""Auto-tuner front end (the reference CLI's `tune` subcommand,
dedisp_tune.cpp:464-535, on the device).

    python tune.py --setup Apertif --dms 4096 [--dms 64 ...] [--repeats 10]
                   [--space gpu|reference] [--max-configs N] [--zero-dm]

For every instance it benchmarks every configuration of the chosen space on
the GPU (1 warm-up + `repeats` CUDA-event-timed runs, tuner.cpp:136-170),
selects the optimum (tuner.cpp:172-179), computes the population statistics
(tuner.cpp:181-206), and writes tuning/<setup>_<d>[_zerodm].json in the
reference's "dedisp-tuning-result/1" layout (report_io.cpp:58-102; GPU knobs
in per-record "b200" objects, roofline and sweep time in a top-level "b200"
object), so tools/analyze.py -- the reference's `analyze` -- reads them.
With several instances it also reports best_fixed_config and the
tuned-vs-fixed speedups (tuner.cpp:218-261; BASELINE config 5) in
tuning/<setup>_summary.json.
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


def result_json(res: api.TuningResult, hbm_gbs: float, seconds: float, flush: bool = True) -> dict:
    d, s, c = res.num_dms, res.setup.samples_per_second, res.setup.channels
    doc = api.tuning_result_to_dict(res)
    best = res.best()
    roof = api.roofline_gflops(d, s, c, hbm_gbs)
    doc["b200"] = {"clock": "cuda events", "sweep_seconds": seconds, "hbm_gbs": hbm_gbs,
                   "hbm_roofline_gflops": roof, "best_roofline_frac": best.gflops / roof,
                   "l2": "flushed" if flush else "warm",
                   "l2_method": "before every timed run: a buffer twice the L2 written, then "
                                "read back (clean lines), outside the CUDA events"
                   if flush else "no flush between runs"}
    return doc


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--setup", default="Apertif")
    p.add_argument("--dms", type=int, action="append")
    p.add_argument("--repeats", type=int, default=10)
    p.add_argument("--space", default="gpu", choices=["gpu", "reference"])
    p.add_argument("--max-configs", type=int, default=0)
    p.add_argument("--zero-dm", action="store_true")
    p.add_argument("--out", default=os.path.join(ROOT, "tuning"))
    p.add_argument("--warm", action="store_true", help="no L2 flush between timed runs")
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
                 max_configs=a.max_configs, flush_l2=not a.warm)
        dt = time.time() - t0
        results.append(res)
        j = result_json(res, hbm, dt, not a.warm)
        name = f"{setup.name.lower()}_{d}{'_zerodm' if a.zero_dm else ''}.json"
        with open(os.path.join(a.out, name), "w") as f:
            json.dump(j, f, indent=1)
        b, k = res.best(), res.best().config
        print(f"{setup.name} d={d}: {len(res.records)} configs in {dt:.1f}s; best "
              f"({k.items_time},{k.items_dm},{k.work_time},{k.work_dm}) "
              f"depth={b.dm_tile_depth} {b.staging} flags={b.flags:#x}: {b.gflops:.1f} GFLOP/s "
              f"({b.mean_time * 1e3:.3f} ms, {j['b200']['best_roofline_frac']:.2f}x HBM "
              f"roofline); snr={res.stats.snr_optimum}", flush=True)
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
                               f"{'_zerodm' if a.zero_dm else ''}.json"), "w") as f:
            json.dump(summ, f, indent=1)
        print("best fixed:", summ["best_fixed"], "speedups:",
              [round(x, 3) for x in rep.speedup_over_fixed])


if __name__ == "__main__":
    main()
