"""The reference CLI's `analyze` subcommand (dedisp_tune.cpp:597-742) over
tuning-result documents written by tune.py (or by the CPU reference):
best fixed configuration, per-instance tuned/fixed GFLOP/s and speedup,
real-time verdict, measured arithmetic intensity at the optimum and for the
naive (1,1,1,1) config against the ai_bounds, an optional roofline verdict,
the zero-DM contrast and deployment sizing.  Writes analysis.json
("dedisp-analysis/1", same keys and order) and analysis.csv.

    python tools/analyze.py --results tuning/apertif_*.json [--out DIR]
        [--roofline PEAK_GFLOPS,PEAK_GBS] [--beams N] [--pass-time S]

Delay tables for the traffic model come from K1 on the device
(api.build_delay_table), so this runs where a GPU is present.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1601_05052_b200 import _native as N  # noqa: E402
from paper_1601_05052_b200 import api  # noqa: E402


def parse_roofline(text: str):
    """dedisp_tune.cpp:143-158"""
    if "," not in text:
        raise SystemExit("--roofline expects peak_gflops,peak_gbs")
    a, b = text.split(",", 1)
    try:
        g, w = float(a), float(b)
    except ValueError:
        raise SystemExit(f"--roofline '{text}' is not a pair of numbers")
    if not (g > 0.0 and w > 0.0):
        raise SystemExit("--roofline peaks must be positive")
    return g, w


def cfg_str(k: api.KernelConfig) -> str:
    return f"({k.items_time},{k.items_dm},{k.work_time},{k.work_dm})"


def analyze(results, roofline=None, beams=0, pass_time=0.0):
    real = [r for r in results if not r.zero_dm]
    zero = [r for r in results if r.zero_dm]
    main = real or zero
    fixed = api.best_fixed_config(main)
    fk = fixed.config[0]
    doc = {"schema": "dedisp-analysis/1", "setup": main[0].setup.name,
           "fixed": {"items_time": fk.items_time, "items_dm": fk.items_dm,
                     "work_time": fk.work_time, "work_dm": fk.work_dm,
                     "total_gflops": fixed.total_gflops}}
    print(f"analyze: {len(results)} result(s), setup {main[0].setup.name}")
    print(f"best fixed configuration {cfg_str(fk)}, summed {fixed.total_gflops:.3f} GFLOP/s")
    csv = ["num_dms,best_gflops,fixed_gflops,threshold_gflops,realtime_pass"]
    instances = []
    for i, r in enumerate(main):
        best = r.best()
        table = (api.build_zero_delay_table if r.zero_dm else api.build_delay_table)(r.setup,
                                                                                     r.num_dms)
        s, c = r.setup.samples_per_second, r.setup.channels
        flop = r.num_dms * s * c
        gt = best.flags & N.DD_CONFIG_GPU_TILING
        ai_best = api.measured_ai(flop, api.kernel_traffic(table, best.config, r.num_dms, s, gt))
        ai_naive = api.measured_ai(flop, api.kernel_traffic(table, api.KernelConfig(1, 1, 1, 1),
                                                            r.num_dms, s))
        no_reuse, reuse = api.ai_bounds(r.num_dms, s, c)
        k = best.config
        node = {"num_dms": r.num_dms,
                "best": {"items_time": k.items_time, "items_dm": k.items_dm,
                         "work_time": k.work_time, "work_dm": k.work_dm},
                "gflops": best.gflops, "fixed_gflops": fixed.fixed_gflops[i],
                "speedup_over_fixed": fixed.speedup_over_fixed[i],
                "threshold_gflops": r.realtime_threshold_gflops,
                "realtime_pass": r.realtime_pass,
                "ai": {"at_best": ai_best, "naive": ai_naive, "no_reuse_bound": no_reuse,
                       "reuse_bound": reuse}}
        if roofline is not None:
            v = api.classify_roofline(ai_best, *roofline)
            node["roofline"] = {"memory_bound": v.memory_bound,
                                "ridge_flop_per_byte": v.ridge_flop_per_byte,
                                "attainable_gflops": v.attainable_gflops}
        node["b200"] = {"dm_tile_depth": best.dm_tile_depth, "staging": best.staging,
                        "family": best.family, "flags": best.flags}
        instances.append(node)
        csv.append(f"{r.num_dms},{best.gflops:.9g},{fixed.fixed_gflops[i]:.9g},"
                   f"{r.realtime_threshold_gflops:.9g},{1 if r.realtime_pass else 0}")
        print(f"d={r.num_dms} tuned {best.gflops:.3f} GFLOP/s, fixed {fixed.fixed_gflops[i]:.3f}, "
              f"speedup {fixed.speedup_over_fixed[i]:.2f}x, threshold "
              f"{r.realtime_threshold_gflops:.3f}, real-time "
              f"{'pass' if r.realtime_pass else 'FAIL'}")
    doc["instances"] = instances
    if zero and real:
        zg = {r.num_dms: r.best().gflops for r in zero}
        contrast = []
        for r in real:
            if r.num_dms not in zg:
                continue
            ratio = zg[r.num_dms] / r.best().gflops
            contrast.append({"num_dms": r.num_dms, "real_gflops": r.best().gflops,
                             "zero_dm_gflops": zg[r.num_dms], "ratio": ratio})
            print(f"d={r.num_dms} zero-DM {zg[r.num_dms]:.3f} vs real {r.best().gflops:.3f} "
                  f"GFLOP/s ({ratio:.2f}x)")
        doc["zero_dm_contrast"] = contrast
    if beams > 0:
        largest = max(main, key=lambda r: r.num_dms)
        t = pass_time if pass_time > 0.0 else largest.best().mean_time
        plan = api.deployment_sizing(largest.setup, largest.num_dms, beams, t)
        doc["deployment"] = {"beams": beams, "pass_time_s": t,
                             "beams_per_device": plan.beams_per_device, "devices": plan.devices}
        print(f"deployment: {beams} beams at {t:.4f} s/pass -> {plan.beams_per_device} "
              f"beams/device, {plan.devices} device(s)")
    doc["notes"] = ["measured AI counts staged loads, output writes, and delay reads at 4 bytes "
                    "per element; unaligned-access overhead is not modeled"]
    return doc, "\n".join(csv) + "\n"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--results", nargs="+", required=True)
    p.add_argument("--out", default=".")
    p.add_argument("--roofline", default="")
    p.add_argument("--beams", type=int, default=0)
    p.add_argument("--pass-time", type=float, default=0.0)
    a = p.parse_args()
    paths = [q for pat in a.results for q in sorted(glob.glob(pat)) or [pat]]
    paths = [q for q in paths if not q.endswith("_summary.json")]
    results = sorted((api.tuning_result_from_json(open(q).read()) for q in paths),
                     key=lambda r: (r.zero_dm, r.num_dms))
    doc, csv = analyze(results, parse_roofline(a.roofline) if a.roofline else None, a.beams,
                       a.pass_time)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "analysis.json"), "w") as f:
        f.write(json.dumps(doc, indent=2) + "\n")
    with open(os.path.join(a.out, "analysis.csv"), "w") as f:
        f.write(csv)
    print(f"wrote {a.out}/analysis.json and {a.out}/analysis.csv")


if __name__ == "__main__":
    main()
