"""The A/B and profiling scripts (tools/gpu_ab_*.sh, tools/gpu_final*.sh)
time tuned records through tools/spec_of.py -> tools/time_configs.py: the
spec must carry exactly the record's configuration and flags."""
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import spec_of  # noqa: E402


def _header_flags():
    text = open(os.path.join(ROOT, "include", "dedisp_b200.h")).read()
    return {m.group(1): int(m.group(2), 16)
            for m in re.finditer(r"#define (DD_CONFIG_\w+) (0x[0-9a-f]+)u", text)}


def test_spec_flag_bits_match_the_header():
    h = _header_flags()
    assert spec_of.flags_of_spec("1,1,1,1,1,smem,g") == h["DD_CONFIG_GPU_TILING"]
    assert spec_of.flags_of_spec("1,1,1,1,1,tmem,occ") == h["DD_CONFIG_HIGH_OCCUPANCY"]
    assert spec_of.flags_of_spec("1,1,1,1,1,smem,tm") == h["DD_CONFIG_TIME_MAJOR"]
    assert spec_of.flags_of_spec("1,1,1,1,1,smem,pk") == h["DD_CONFIG_PACKED_STAGES"]
    assert spec_of.flags_of_spec("1,1,1,1,1,smem,wide") == h["DD_CONFIG_WIDE_STAGES"]


def test_every_tuned_record_round_trips_through_its_spec():
    n = 0
    for path in glob.glob(os.path.join(ROOT, "tuning", "*_*.json")):
        if path.endswith("_summary.json"):
            continue
        doc = json.load(open(path))
        recs = sorted((r for r in doc["records"] if r["mean_time_s"] > 0),
                      key=lambda r: r["mean_time_s"])[:3]
        for r in recs:
            sp = spec_of.spec(r)
            f = sp.split(",")
            assert list(map(int, f[:5])) == [r["items_time"], r["items_dm"], r["work_time"],
                                              r["work_dm"], r["b200"]["dm_tile_depth"]]
            assert f[5] == r["b200"]["staging"]
            assert spec_of.flags_of_spec(sp) == r["b200"]["flags"], (path, sp)
            n += 1
    assert n >= 24
