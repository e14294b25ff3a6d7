"""Tuner front end and analysis on the device: tune.py's documents load
through the reference-layout parser and tools/analyze.py (the reference's
`analyze`, dedisp_tune.cpp:597-742) produces its report from them."""
import json
import os
import sys

import pytest

from paper_1601_05052_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if api.device_count() == 0:
        pytest.skip("no CUDA device")
    return api.context(0)


def test_tune_documents_feed_analyze(dev, tmp_path):
    import analyze
    import tune
    setup = api.ObservationSetup("mini", 64, 8, 100.0, 25.0, 0.0, 0.5)
    results = []
    for d in (4, 8):
        for zero in (False, True):
            fn = api.zero_dm_experiment if zero else api.tune
            res = fn(setup, d, repeats=2, full_reference_space=True)
            text = json.dumps(tune.result_json(res, 6549.8, 0.1))
            back = api.tuning_result_from_json(text)
            assert back.best().config == res.best().config
            assert len(back.records) == len(res.records)
            assert back.zero_dm == zero
            results.append(back)
    doc, csv = analyze.analyze(results, (4500.0, 288.0), beams=450)
    assert doc["schema"] == "dedisp-analysis/1"
    assert list(doc)[:4] == ["schema", "setup", "fixed", "instances"]
    assert [i["num_dms"] for i in doc["instances"]] == [4, 8]
    for inst in doc["instances"]:
        ai = inst["ai"]
        assert 0 < ai["naive"] < 0.25 and ai["at_best"] <= ai["reuse_bound"] + 1e-12
        assert inst["speedup_over_fixed"] >= 1.0 - 1e-12
        assert "roofline" in inst
    assert len(doc["zero_dm_contrast"]) == 2
    assert doc["deployment"]["devices"] >= 1
    assert csv.splitlines()[0] == "num_dms,best_gflops,fixed_gflops,threshold_gflops,realtime_pass"

