"""Print the tools/time_configs.py spec of a tuning document's best record
(or of record rank N): python tools/spec_of.py tuning/apertif_4096.json [N]"""
import json
import sys


def spec(r):
    b = r["b200"]
    f = b["flags"]
    x = ["g"] if f & 1 else []
    x += ["occ"] if f & 2 else []
    x += ["tm"] if f & 8 else []
    x += ["pk"] if f & 0x10 else []
    x += ["wide"] if f & 0x20 else []
    cps = (f >> 8) & 15
    x += ["cps%d" % cps] if cps else []
    ns = (f >> 12) & 15
    x += ["ns%d" % ns] if ns else []
    return ",".join(map(str, [r["items_time"], r["items_dm"], r["work_time"], r["work_dm"],
                              b["dm_tile_depth"], b["staging"]] + x))


def flags_of_spec(spec_str):
    """The dd_config flags tools/time_configs.py builds from a spec (the
    inverse of spec() above; "cpsN" and "occ" map to the same bits the plan's
    stage_channels / high_occupancy arguments set)."""
    extra = spec_str.split(",")[6:]
    f = 1 if "g" in extra else 0
    f |= 2 if "occ" in extra else 0
    f |= 8 if "tm" in extra else 0
    f |= 0x10 if "pk" in extra else 0
    f |= 0x20 if "wide" in extra else 0
    f |= next((int(x[3:]) for x in extra if x.startswith("cps")), 0) << 8
    f |= next((int(x[2:]) for x in extra if x.startswith("ns")), 0) << 12
    return f


if __name__ == "__main__":
    d = json.load(open(sys.argv[1]))
    recs = sorted((r for r in d["records"] if r["mean_time_s"] > 0), key=lambda r: r["mean_time_s"])
    print(spec(recs[int(sys.argv[2]) if len(sys.argv) > 2 else 0]))
