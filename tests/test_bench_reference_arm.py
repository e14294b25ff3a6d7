"""bench.py's reference arm (``--impl reference``): the reference's own CPU
path (oracle/_ref, kernels.cpp:117-206) on a bounded sample, printing the
same JSON contract as our arm.  Runs without a GPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--setup", "LOFAR",
                        "--dms", "8", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "GFLOP/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"] == {"value": line["value"], "unit": "GFLOP/s",
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the same workload string our arm prints for this instance
    assert line["config"]["workload"] == \
        "LOFAR c=32 s=200000 t=400000, 8 trial DMs, 1 s block (BASELINE config 3)"
