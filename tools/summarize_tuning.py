"""Tuned vs best fixed configuration over a setup's committed sweeps
(reference tuner.cpp:218-261, BASELINE config 5), from the documents in
tuning/ -- for sweeps run in several tune.py invocations.

    python tools/summarize_tuning.py Apertif [--markdown]
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1601_05052_b200 import api  # noqa: E402


def main():
    name = sys.argv[1]
    docs = {}
    for p in glob.glob(os.path.join(ROOT, "tuning", f"{name.lower()}_*.json")):
        if p.endswith("_summary.json") or "zerodm" in p:
            continue
        with open(p) as f:
            text = f.read()
        d = json.loads(text)
        docs[d["num_dms"]] = (api.tuning_result_from_json(text), d)
    dms = sorted(docs)
    results = [docs[d][0] for d in dms]
    rep = api.best_fixed_config(results)
    k, depth, staging, flags = rep.config
    rows = []
    for d, res, fixed, sp in zip(dms, results, rep.fixed_gflops, rep.speedup_over_fixed):
        b = res.best()
        meta = docs[d][1].get("b200", {})
        rows.append({"num_dms": d, "configs": len(res.records),
                     "best": [b.config.items_time, b.config.items_dm, b.config.work_time,
                              b.config.work_dm],
                     "depth": b.dm_tile_depth, "staging": b.staging, "flags": b.flags,
                     "tuned_gflops": b.gflops, "tuned_ms": b.mean_time * 1e3,
                     "fixed_gflops": fixed, "speedup_over_fixed": sp,
                     "snr_optimum": res.stats.snr_optimum,
                     "chebyshev_bound": res.stats.chebyshev_bound,
                     "l2": meta.get("l2", "warm (round 1)")})
    summ = {"setup": name, "instances": dms,
            "best_fixed": {"items_time": k.items_time, "items_dm": k.items_dm,
                           "work_time": k.work_time, "work_dm": k.work_dm,
                           "dm_tile_depth": depth, "staging": staging, "flags": flags},
            "fixed_gflops": rep.fixed_gflops, "tuned_gflops": [r["tuned_gflops"] for r in rows],
            "speedup_over_fixed": rep.speedup_over_fixed, "per_instance": rows}
    with open(os.path.join(ROOT, "tuning", f"{name.lower()}_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    if "--markdown" in sys.argv:
        print("| d | configs | tuned config (it, id, wt, wd) depth staging flags | pass | GFLOP/s | "
              "best fixed GFLOP/s | tuned/fixed | SNR | L2 |")
        print("|---|---|---|---|---|---|---|---|---|")
        for r in rows:
            ms = r["tuned_ms"]
            t = f"{ms * 1e3:.0f} µs" if ms < 1 else f"{ms:.3f} ms"
            print(f"| {r['num_dms']} | {r['configs']} | {tuple(r['best'])} {r['depth']} "
                  f"{r['staging']} {r['flags']:#x} | {t} | {r['tuned_gflops']:.0f} | "
                  f"{r['fixed_gflops']:.0f} | {r['speedup_over_fixed']:.2f} | "
                  f"{r['snr_optimum']:.2f} | {r['l2']} |")
        print(f"\nbest fixed: {summ['best_fixed']}")


if __name__ == "__main__":
    main()
