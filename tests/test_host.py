"""CPU-side tests of the product library: the C-ABI loads and exports every
symbol include/dedisp_b200.h declares, and its host logic (geometry, config
rules, enumeration, traffic model, tuner statistics, synthetic input) keeps
the reference's contracts.  No CUDA device is used here; calls that need one
must fail loudly (no CPU fallback)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_1601_05052_b200 import _native as N
from paper_1601_05052_b200 import api
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "dedisp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = _header_functions()
    assert len(declared) >= 35
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.SIGNATURES) == declared, set(declared) ^ set(N.SIGNATURES)
    assert lib.dd_abi_version() == 1


def test_struct_layouts_match_header():
    assert C.sizeof(N.dd_setup) == 40
    assert C.sizeof(N.dd_config) == 28
    assert C.sizeof(N.dd_tuning_record) == 32 + 32 + 8


def test_no_device_fails_loudly():
    if api.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(N.DeviceError):
        api.Context(0)


def test_argument_errors_need_no_device():
    """Argument checks run before any device work (and name the problem)."""
    L = N.lib()
    assert L.dd_upload_block_range(None, None, 0, None, 0, 1, 0, 1, None) == \
        N.DD_ERR_INVALID_ARGUMENT
    assert L.dd_plan_get_info(None, None) == N.DD_ERR_INVALID_ARGUMENT
    bad = N.dd_config(32, 4, 5, 8, 1, N.STAGING["smem"], 1 << N.DD_CONFIG_NSTAGE_SHIFT)
    assert L.dd_validate_config(C.byref(bad), 4096, 20000, None) == N.DD_ERR_INVALID_ARGUMENT
    assert "stages" in L.dd_last_error().decode()
    ok = N.dd_config(32, 4, 5, 8, 1, N.STAGING["tmem"],
                     N.DD_CONFIG_TIME_MAJOR | (15 << N.DD_CONFIG_CPS_SHIFT)
                     | (3 << N.DD_CONFIG_NSTAGE_SHIFT))
    assert L.dd_validate_config(C.byref(ok), 4096, 20000, None) == N.DD_OK


def test_geometry_known_answers(golden):
    # test_setup.cpp:15-24, :130-137
    assert math.isclose(api.delay_seconds(0.25, 1420.0, 1720.0), 1.63834524e-4, rel_tol=1e-8)
    with pytest.raises(ValueError):
        api.delay_seconds(1.0, 1800.0, 1720.0)
    with pytest.raises(ValueError):
        api.delay_seconds(float("nan"), 1.0, 2.0)
    assert api.instance_sizing(api.APERTIF, 1).flop == 20_480_000
    assert api.instance_sizing(api.LOFAR, 1).flop == 6_400_000
    for g in golden["baseline"]:
        s = g["setup"]
        setup = api.find_builtin(s["name"])
        p = api.instance_sizing(setup, g["num_dms"])
        assert (p.num_samples, p.flop, p.max_delay) == (g["num_samples"], g["flop"],
                                                       g["sizing_max_delay"])


def test_setup_validation():
    bad = api.ObservationSetup("x", 0, 4, 100.0, 1.0, 0.0, 0.5)
    with pytest.raises(ValueError):
        bad.validate()
    with pytest.raises(ValueError):
        api.ObservationSetup("x", 16, 4, -1.0, 1.0, 0.0, 0.5).validate()
    api.APERTIF.validate()


def test_noise_is_bit_identical_to_reference(golden):
    # filterbank.cpp:22-80 via the reference-produced fingerprints
    for g in golden["baseline"][:2] + golden["mini"][:20]:
        s = g["setup"]
        setup = api.ObservationSetup(s["name"], s["samples_per_second"], s["channels"], s["f_min"],
                                     s["channel_width"], s["dm_first"], s["dm_step"])
        fb = api.noise_filterbank(setup, g["num_samples"], g["sigma"], g["seed"])
        assert O.fnv1a(fb.data) == g["in_fnv"]
    # odd sample counts drop the final spare exactly like the reference
    setup = api.ObservationSetup("odd", 7, 3, 100.0, 1.0, 0.0, 0.5)
    a = api.noise_filterbank(setup, 7, 0.7, 11).data
    b = O.noise(3, 7, 0.7, 11)
    assert a.tobytes() == b.tobytes()
    assert not api.noise_filterbank(setup, 7, 0.0, 11).data.any()
    with pytest.raises(ValueError):
        api.noise_filterbank(setup, 7, -1.0, 1)


def test_config_rules():
    # test_kernels.cpp:39-61
    d, s = 16, 64
    K = api.KernelConfig
    assert api.config_valid(K(1, 1, 1, 1), d, s)
    assert api.config_valid(K(4, 2, 8, 2), d, s)
    assert api.config_valid(K(64, 16, 1, 1), d, s)
    assert not api.config_valid(K(3, 1, 1, 1), d, s)
    assert not api.config_valid(K(1, 3, 1, 1), d, s)
    assert not api.config_valid(K(0, 1, 1, 1), d, s)
    assert not api.config_valid(K(1, 1, 0, 1), d, s)
    tight = api.KernelLimits(8, 4)
    assert api.config_valid(K(4, 2, 2, 2), d, s, tight)
    assert not api.config_valid(K(8, 2, 1, 1), d, s, tight)
    assert not api.config_valid(K(1, 1, 4, 2), d, s, tight)
    with pytest.raises(ValueError, match="block limit"):
        api.validate_config(K(8, 2, 1, 1), d, s, tight)
    api.validate_config(K(4, 2, 2, 2), d, s, tight)
    c = K(4, 2, 8, 3)
    assert (c.tile_time(), c.tile_dm(), c.block_items(), c.accumulators()) == (32, 6, 8, 24)


def test_enumeration_matches_reference(golden):
    for g in golden["enumerate"]:
        cfgs = api.enumerate_configs(g["num_dms"], g["s"], api.KernelLimits(*g["limits"]))
        arr = np.array([(k.items_time, k.items_dm, k.work_time, k.work_dm) for k in cfgs], np.uint32)
        assert len(cfgs) == g["count"] and O.fnv1a(arr) == g["fnv"]
    assert cfgs == sorted(cfgs)
    with pytest.raises(ValueError):
        api.enumerate_configs(16, 64, api.KernelLimits(0, 256))  # test_tuner.cpp:52-56


def test_count_loads_matches_reference(golden):
    tables = {}
    for g in golden["count_loads"]:
        setup = api.find_builtin(g["setup"])
        if setup.name not in tables:
            sh, md = O.delay_table(O.APERTIF if setup.name == "Apertif" else O.LOFAR, 4096)
            tables[setup.name] = api.DelayTable(setup, 4096, sh, md)
        lc = api.count_loads(tables[setup.name], api.KernelConfig(*g["config"]), 4096,
                             setup.samples_per_second)
        assert (lc.staged_loads, lc.ideal_loads) == (g["staged"], g["ideal"])


def test_count_loads_random_against_oracle():
    rng = np.random.default_rng(7)
    for trial in range(10):
        setup = O.Setup("m", 16 << (trial % 3), int(rng.integers(1, 10)), 100.0, 25.0, 0.0,
                        0.2 + 0.15 * (trial % 5))
        d = int(rng.integers(1, 16))
        sh, md = O.delay_table(setup, d)
        table = api.DelayTable(api.ObservationSetup("m", setup.samples_per_second, setup.channels,
                                                    100.0, 25.0, 0.0, setup.dm_step), d, sh, md)
        for cfg in O.enumerate_configs(d, setup.samples_per_second, 1 << 20, 1 << 20)[::7]:
            got = api.count_loads(table, api.KernelConfig(*cfg), d, setup.samples_per_second)
            assert (got.staged_loads, got.ideal_loads) == O.count_loads(
                sh, setup.samples_per_second, cfg)


def _rec(cfg, g):
    return api.TuningRecord(api.KernelConfig(*cfg), [1.0], 1.0, g)


def test_select_best_and_stats():
    # test_tuner.cpp:58-118
    assert api.select_best([_rec((2, 2, 1, 1), 7.0), _rec((1, 1, 2, 1), 7.0),
                            _rec((2, 1, 1, 1), 5.0)]) == 1
    assert api.select_best([_rec((2, 1, 1, 1), 7.0), _rec((1, 2, 1, 1), 7.0)]) == 1
    st = api.compute_stats([_rec((1, 1, 1, 1), g) for g in (2.0, 4.0, 6.0, 8.0)], 3)
    assert math.isclose(st.mean_gflops, 5.0) and math.isclose(st.stddev_gflops, math.sqrt(5))
    assert math.isclose(st.chebyshev_bound, 5.0 / 9.0)
    flat = api.compute_stats([_rec((1, 1, 1, 1), 3.0)] * 5, 0)
    assert flat.degenerate and flat.snr_optimum is None
    skew = [_rec((1, 1, 1, 1), 0.0)] * 64 + [_rec((1, 1, 1, 1), 7.0)] * 25
    a = api.compute_stats(skew, api.select_best(skew))
    assert math.isclose(a.snr_optimum, 1.6, rel_tol=1e-9)
    assert math.isclose(a.chebyshev_bound, 0.390625, rel_tol=1e-9)
    spiky = [_rec((1, 1, 1, 1), 0.0)] * 20 + [_rec((1, 1, 1, 1), 7.0)]
    b = api.compute_stats(spiky, api.select_best(spiky))
    assert math.isclose(b.chebyshev_bound, 0.05, rel_tol=1e-9)


def test_best_fixed_config():
    # tuner.cpp:218-261
    def result(recs):
        return api.TuningResult(api.APERTIF, 2, False, api.KernelLimits(), 1, 1, recs,
                                api.select_best(recs), api.TuningStats(), 0.0, False)
    r1 = result([_rec((1, 1, 1, 1), 4.0), _rec((2, 1, 1, 1), 6.0)])
    r2 = result([_rec((1, 1, 1, 1), 5.0), _rec((2, 1, 1, 1), 2.0), _rec((4, 1, 1, 1), 9.0)])
    rep = api.best_fixed_config([r1, r2])
    assert rep.config[0] == api.KernelConfig(1, 1, 1, 1)
    assert rep.fixed_gflops == [4.0, 5.0]
    assert rep.speedup_over_fixed == [6.0 / 4.0, 9.0 / 5.0]
    with pytest.raises(ValueError):
        api.best_fixed_config([])


def test_roofline_definitions():
    # Apertif d=4096 -> 335.89 GB no-reuse, 1635.8 GFLOP/s at 6549.8 GB/s
    b = api.algorithmic_bytes(4096, 20000, 1024)
    assert abs(b / 1e9 - 335.89) < 0.01
    assert abs(api.roofline_gflops(4096, 20000, 1024, 6549.8) - 1635.8) < 0.5
    assert math.isclose(api.realtime_threshold_gflops(api.APERTIF, 4096), 83.88608)
    assert api.ai_bounds(4096, 20000, 1024)[0] == 0.25


def test_cxx_dropin_header_compiles_and_links(tmp_path):
    """The C++ drop-in (include/dedisp/b200.hpp) builds like reference client
    code and links against the library (running it needs a GPU)."""
    import subprocess
    exe = str(tmp_path / "dropin")
    pkg = os.path.join(ROOT, "paper_1601_05052_b200")
    O.lib()
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cxx", "test_dropin.cpp"), "-L", pkg,
                        "-ldedisp_b200", "-L", os.path.join(ROOT, "oracle"), "-loracle",
                        "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_cxx_analysis_layer(tmp_path):
    """The reference's analysis/tuner helpers through the C++ drop-in header
    (deployment sizing, device table, roofline, histogram): host-only, so it
    runs here."""
    import subprocess
    exe = str(tmp_path / "analysis")
    pkg = os.path.join(ROOT, "paper_1601_05052_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cxx", "test_analysis.cpp"), "-L", pkg,
                        "-ldedisp_b200", "-Wl,-rpath," + pkg, "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "analysis: ok" in r.stdout, r.stdout + r.stderr


def test_tuned_schedules_follow_the_committed_sweeps():
    """The built-in schedules (csrc/schedules.inc, the one-shot entry points'
    AUTO) are the tuner's picks in tuning/*.json; a registered schedule takes
    precedence and can be forgotten; an invalid one is rejected."""
    import glob
    import json
    n = 0
    for path in glob.glob(os.path.join(ROOT, "tuning", "*_*.json")):
        if path.endswith("_summary.json"):
            continue
        doc = json.load(open(path))
        best = doc["records"][doc["best_index"]]
        s = doc["setup"]
        got = api.schedule_get(s["channels"], s["samples_per_second"], doc["num_dms"])
        assert got is not None, path
        cfg, depth, staging, flags, builtin = got
        assert builtin
        assert (cfg.items_time, cfg.items_dm, cfg.work_time, cfg.work_dm) == \
            (best["items_time"], best["items_dm"], best["work_time"], best["work_dm"]), path
        assert (depth, staging, flags) == (best["b200"]["dm_tile_depth"], best["b200"]["staging"],
                                           best["b200"]["flags"]), path
        n += 1
    assert n >= 24
    assert api.schedule_get(7, 100, 3) is None
    rec = api.TuningRecord(api.KernelConfig(16, 2, 5, 2), staging="smem",
                           flags=8 << N.DD_CONFIG_CPS_SHIFT)
    api.schedule_set(7, 160, 4, rec)
    cfg, depth, staging, flags, builtin = api.schedule_get(7, 160, 4)
    assert (cfg, staging, flags, builtin) == (rec.config, "smem", rec.flags, False)
    api.schedule_set(7, 160, 4, None)
    assert api.schedule_get(7, 160, 4) is None
    with pytest.raises(ValueError):  # tile_dm 4 does not divide 6 trials
        api.schedule_set(7, 160, 6, rec)


def test_fingerprint_matches_the_fixture_hash():
    """dd_fingerprint (the bench's parity check) is the FNV-1a 64 the golden
    fixtures use (the oracle's hash), on arbitrary bytes."""
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 4096, 100003):
        a = rng.integers(0, 256, size=n, dtype=np.uint8)
        assert api.fingerprint(a) == O.fnv1a(a)
    assert api.fingerprint(np.zeros(0, np.uint8)) == "cbf29ce484222325"
