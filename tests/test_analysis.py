"""Analysis layer and tuning-result documents: the
reference's analysis.cpp metric functions, make_histogram, and the
"dedisp-tuning-result/1" document layout (report_io.cpp), mirrored from
proj/tests/test_analysis.cpp and test_tuner.cpp.  CPU only."""
import json
import math

import pytest

from paper_1601_05052_b200 import api
from oracle import oracle as O


def _mini(rate=64, channels=8, dm_step=0.5):
    # tests/support/oracles.hpp:132-143
    return api.ObservationSetup("mini", rate, channels, 100.0, 25.0, 0.0, dm_step)


def _table(setup, d, zero=False):
    sh, md = O.delay_table(O.Setup(setup.name, setup.samples_per_second, setup.channels,
                                   setup.f_min, setup.channel_width, setup.dm_first,
                                   setup.dm_step), d)
    if zero:
        sh[:] = 0
        md = 0
    return api.DelayTable(setup, d, sh, md)


def test_ai_bounds():
    # test_analysis.cpp:12-28
    assert api.ai_bounds(1, 1, 1)[0] == 0.25
    rb = api.ai_bounds(2048, 20000, 1024)[1]
    assert math.isclose(rb, 1.0 / (4.0 * (1 / 2048 + 1 / 20000 + 1 / 1024)), rel_tol=1e-12)
    assert math.isclose(rb, 165.03, rel_tol=1e-4)
    assert api.ai_bounds(2, 20000, 1024)[1] < rb < api.ai_bounds(4096, 20000, 1024)[1]


def test_measured_ai():
    # test_analysis.cpp:30-37
    assert math.isclose(api.measured_ai(1000, api.MemoryTraffic(50, 25, 25)), 2.5)
    with pytest.raises(ValueError):
        api.measured_ai(1000, api.MemoryTraffic(0, 0, 0))


def test_kernel_traffic():
    # test_analysis.cpp:39-61
    setup = _mini()
    table = _table(setup, 8)
    t = api.kernel_traffic(table, api.KernelConfig(4, 2, 2, 2), 8, 64)
    assert t.output_writes == 8 * 64 and t.delay_reads == 8 * 8
    assert t.staged_loads == api.count_loads(table, api.KernelConfig(4, 2, 2, 2), 8,
                                             64).staged_loads
    t1 = api.kernel_traffic(table, api.KernelConfig(1, 1, 1, 1), 8, 64)
    assert t1.staged_loads == 8 * 64 * 8
    assert api.measured_ai(8 * 64 * 8, t1) < 0.25


def test_zero_dm_whole_tile_reaches_reuse_bound():
    # test_analysis.cpp:63-73
    setup = _mini()
    table = _table(setup, 16, zero=True)
    t = api.kernel_traffic(table, api.KernelConfig(64, 16, 1, 1), 16, 64)
    ai = api.measured_ai(16 * 64 * 8, t)
    assert math.isclose(ai, api.ai_bounds(16, 64, 8)[1], rel_tol=1e-12)


def test_real_tables_never_beat_reuse_bound():
    # test_analysis.cpp:75-89
    setup = _mini(128, 12)
    table = _table(setup, 16)
    bound = api.ai_bounds(16, 128, 12)[1]
    for cfg in api.enumerate_configs(16, 128, api.KernelLimits(1 << 20, 1 << 20)):
        assert api.measured_ai(16 * 128 * 12, api.kernel_traffic(table, cfg, 16, 128)) <= bound


def test_deployment_sizing():
    # test_analysis.cpp:102-120
    ap = api.APERTIF
    p = api.deployment_sizing(ap, 2000, 450, 0.106)
    assert (p.beams_per_device, p.devices) == (9, 50)
    assert api.deployment_sizing(ap, 2000, 9, 0.106).devices == 1
    assert api.deployment_sizing(ap, 2000, 10, 0.106).devices == 2
    assert api.deployment_sizing(ap, 2000, 450, 0.5).beams_per_device == 2
    for t in (1.0, 2.5):
        with pytest.raises(api.NotRealTimeError):
            api.deployment_sizing(ap, 2000, 450, t)
    with pytest.raises(ValueError):
        api.deployment_sizing(ap, 2000, 0, 0.106)
    with pytest.raises(ValueError):
        api.deployment_sizing(ap, 2000, 450, 0.0)


def test_classify_roofline():
    # analysis.cpp:79-93
    v = api.classify_roofline(0.25, 3788.0, 264.0)
    assert v.memory_bound and math.isclose(v.ridge_flop_per_byte, 3788.0 / 264.0)
    assert math.isclose(v.attainable_gflops, 66.0)
    v = api.classify_roofline(100.0, 3788.0, 264.0)
    assert not v.memory_bound and v.attainable_gflops == 3788.0
    with pytest.raises(ValueError):
        api.classify_roofline(0.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        api.classify_roofline(1.0, 1.0, float("inf"))


def _rec(cfg, g, **kw):
    return api.TuningRecord(api.KernelConfig(*cfg), [g / 10, g / 11], 1.0 / g, g, **kw)


def test_histogram():
    # test_tuner.cpp:255-270
    res = api.TuningResult(api.APERTIF, 2, False, api.KernelLimits(), 1, 1,
                           [_rec((1, 1, 1, 1), g) for g in (1.0, 2.0, 3.0, 4.0)], 3,
                           api.TuningStats(), 0.0, False)
    bins = api.make_histogram(res, 3)
    assert len(bins) == 3 and math.isclose(bins[0].lo, 1.0) and math.isclose(bins[2].hi, 4.0)
    assert [b.count for b in bins] == [1, 1, 2]
    flat = api.TuningResult(api.APERTIF, 2, False, api.KernelLimits(), 1, 1,
                            [_rec((1, 1, 1, 1), 5.0)] * 3, 0, api.TuningStats(), 0.0, False)
    assert sum(b.count for b in api.make_histogram(flat, 4)) == 3
    with pytest.raises(ValueError):
        api.make_histogram(flat, 0)


def _result():
    recs = [_rec((32, 4, 12, 8), 9558.1, dm_tile_depth=1, staging="tmem", family="tmem",
                 flags=0x801),
            _rec((16, 16, 10, 4), 7000.5, staging="smem", family="smem", flags=0x800),
            _rec((1, 1, 1, 1), 12.25)]
    st = api.compute_stats(recs, 0)
    return api.TuningResult(api.APERTIF, 4096, False, api.KernelLimits(), 10, 1, recs, 0, st,
                            api.realtime_threshold_gflops(api.APERTIF, 4096), True)


def test_tuning_document_layout_and_round_trip():
    # report_io.cpp:58-102 key order; test_tuner.cpp:291-336 round trip
    res = _result()
    text = api.tuning_result_to_json(res)
    doc = json.loads(text)
    assert list(doc) == ["schema", "setup", "num_dms", "zero_dm", "limits", "repeats", "seed",
                         "environment", "records", "best_index", "stats", "realtime"]
    assert doc["schema"] == "dedisp-tuning-result/1"
    assert list(doc["setup"]) == ["name", "samples_per_second", "channels", "f_min_mhz",
                                  "channel_width_mhz", "dm_first", "dm_step"]
    assert list(doc["environment"]) == ["threads", "rng", "clock_resolution_s"]
    assert list(doc["records"][0])[:8] == ["items_time", "items_dm", "work_time", "work_dm",
                                           "runs_s", "mean_time_s", "gflops", "timer_warning"]
    assert list(doc["stats"]) == ["mean_gflops", "stddev_gflops", "snr_optimum",
                                  "chebyshev_bound", "degenerate"]
    back = api.tuning_result_from_json(text)
    assert back.setup == res.setup and back.num_dms == res.num_dms
    assert back.limits == res.limits and back.best_index == res.best_index
    assert back.stats == res.stats and back.rng_id == res.rng_id
    assert back.realtime_threshold_gflops == res.realtime_threshold_gflops
    for a, b in zip(back.records, res.records):
        assert (a.config, a.runs, a.mean_time, a.gflops, a.timer_warning) == \
            (b.config, b.runs, b.mean_time, b.gflops, b.timer_warning)
        assert (a.dm_tile_depth, a.staging, a.family, a.flags) == \
            (b.dm_tile_depth, b.staging, b.family, b.flags)
    # a CPU reference document (no "b200" objects) loads with default knobs
    for r in doc["records"]:
        del r["b200"]
    plain = api.tuning_result_from_json(json.dumps(doc))
    assert plain.records[0].staging == "auto" and plain.records[0].flags == 0


def test_malformed_documents_are_rejected():
    # test_tuner.cpp:338-343
    for text in ("not json", "{}", '{"schema":"bogus/9"}'):
        with pytest.raises(api.FormatError):
            api.tuning_result_from_json(text)
    doc = json.loads(api.tuning_result_to_json(_result()))
    doc["best_index"] = 3
    with pytest.raises(api.FormatError):
        api.tuning_result_from_json(json.dumps(doc))


def test_csv_lists_one_row_per_configuration():
    res = _result()
    lines = api.tuning_result_to_csv(res).splitlines()
    assert lines[0] == "items_time,items_dm,work_time,work_dm,mean_time_s,gflops"
    assert len(lines) == 1 + len(res.records)
    assert lines[1].startswith("32,4,12,8,")


def test_committed_tuning_documents_load():
    import glob
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    paths = [p for p in glob.glob(os.path.join(root, "tuning", "*.json"))
             if not p.endswith("_summary.json")]
    assert paths
    for p in paths:
        r = api.tuning_result_from_json(open(p).read())
        assert r.records and r.best().gflops > 0
        assert r.best().gflops == max(x.gflops for x in r.records)
