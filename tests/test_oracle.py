"""Pin the C restatement (oracle/dedisp_oracle.c) before trusting it.

Every fixture in tests/golden/golden.json was produced by the unmodified
reference (oracle/_ref, see tests/golden/make_golden.py).  The known-answer
checks restate the reference's own unit tests (file:line cited per test).
CPU only.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def _setup(d):
    return O.Setup(d["name"], d["samples_per_second"], d["channels"], d["f_min"],
                   d["channel_width"], d["dm_first"], d["dm_step"])


def test_delay_seconds_known_answer():
    # test_setup.cpp:15-24
    assert math.isclose(O.delay_seconds(0.25, 1420.0, 1720.0), 1.63834524e-4, rel_tol=1e-8)
    assert O.delay_seconds(0.0, 1420.0, 1720.0) == 0.0
    with pytest.raises(ValueError):
        O.delay_seconds(-1.0, 1420.0, 1720.0)
    with pytest.raises(ValueError):
        O.delay_seconds(1.0, 1800.0, 1720.0)


def test_builtin_table_anchors():
    # test_setup.cpp:75-88 (Apertif at(0,1)==3) and :90-102 (monotone, max_delay)
    sh, md = O.delay_table(O.APERTIF, 16)
    assert sh[1, 0] == 3
    assert np.all(np.diff(sh.astype(np.int64), axis=0) >= 0)
    assert np.all(np.diff(sh.astype(np.int64), axis=1) <= 0)
    assert np.all(sh[:, -1] == 0)
    assert md == sh.max()


def test_flop_per_dm():
    # test_setup.cpp:130-137: 20,480,000 (Apertif) and 6,400,000 (LOFAR)
    assert O.instance_sizing(O.APERTIF, 1)[1] == 20_480_000
    assert O.instance_sizing(O.LOFAR, 1)[1] == 6_400_000


def test_sizing_and_tables_match_reference_fingerprints(golden):
    for g in golden["baseline"]:
        setup = _setup(g["setup"])
        t, flop, md = O.instance_sizing(setup, g["num_dms"])
        assert (t, flop, md) == (g["num_samples"], g["flop"], g["sizing_max_delay"])
        sh, md2 = O.delay_table(setup, g["num_dms"])
        assert md2 == g["max_delay"]
        assert O.fnv1a(sh) == g["shifts_fnv"], (setup.name, g["num_dms"])


def test_mini_instances_match_reference(golden):
    for g in golden["mini"]:
        setup = _setup(g["setup"])
        sh, md = O.delay_table(setup, g["num_dms"])
        assert md == g["max_delay"] and O.fnv1a(sh) == g["shifts_fnv"]
        fb = O.noise(setup.channels, g["num_samples"], g["sigma"], g["seed"])
        assert O.fnv1a(fb) == g["in_fnv"]
        out = O.dedisperse_reference(fb, sh, setup.samples_per_second)
        assert O.fnv1a(out) == g["out_fnv"]


def test_zero_dm_matches_reference(golden):
    for g in golden["zero_dm"]:
        setup = _setup(g["setup"])
        sh, md = O.delay_table(setup, g["num_dms"], zero=True)
        assert md == 0 and not sh.any()
        fb = O.noise(setup.channels, g["num_samples"], 1.0, g["seed"])
        assert O.fnv1a(fb) == g["in_fnv"]
        out = O.dedisperse_reference(fb, sh, setup.samples_per_second)
        assert O.fnv1a(out) == g["out_fnv"]
        # test_kernels.cpp:166-181: rows are per-column channel sums
        assert all(np.array_equal(out[0], out[i]) for i in range(len(out)))


@pytest.mark.parametrize("idx", [0, 1, 4, 5])
def test_baseline_small_outputs(golden, idx):
    g = golden["baseline"][idx]
    setup = _setup(g["setup"])
    sh, _ = O.delay_table(setup, g["num_dms"])
    fb = O.noise(setup.channels, g["num_samples"], g["sigma"], g["seed"])
    assert O.fnv1a(fb) == g["in_fnv"]
    out = O.dedisperse_tiled(fb, sh, setup.samples_per_second, (1000, 1, 1, 1)
                             if setup.samples_per_second % 1000 == 0 else (1, 1, 1, 1))
    assert O.fnv1a(out) == g["out_fnv"]
    assert float(out.flat[0]) == g["out_first"] and float(out.flat[-1]) == g["out_last"]


@pytest.mark.slow
def test_apertif_4096_output(golden):
    g = golden["baseline"][2]
    setup = _setup(g["setup"])
    sh, _ = O.delay_table(setup, 4096)
    fb = O.noise(setup.channels, g["num_samples"], 1.0, 1)
    out = O.dedisperse_tiled(fb, sh, setup.samples_per_second, (250, 4, 4, 4))
    assert O.fnv1a(out) == g["out_fnv"]


def test_tiled_restatement_equals_reference_for_all_configs():
    # test_kernels.cpp:116-139: every valid config under limits {64, 32}
    setup = O.Setup("mini", 48, 6, 100.0, 25.0, 0.0, 0.5)
    d = 12
    sh, md = O.delay_table(setup, d)
    t, _, _ = O.instance_sizing(setup, d)
    fb = O.noise(setup.channels, t, 1.0, 99)
    ref = O.dedisperse_reference(fb, sh, 48)
    cfgs = O.enumerate_configs(d, 48, 64, 32)
    assert len(cfgs) > 20
    for cfg in cfgs:
        assert np.array_equal(O.dedisperse_tiled(fb, sh, 48, cfg, threads=2).view(np.uint32),
                              ref.view(np.uint32)), cfg


def test_enumeration_matches_reference(golden):
    for g in golden["enumerate"]:
        cfgs = O.enumerate_configs(g["num_dms"], g["s"], *g["limits"])
        assert len(cfgs) == g["count"]
        assert O.fnv1a(np.array(cfgs, np.uint32)) == g["fnv"]


def test_enumeration_brute_force():
    # test_tuner.cpp:29-50 / oracles.hpp:109-129
    for d, s, lim in [(2, 4, (4, 4)), (6, 12, (8, 6)), (1, 1, (1, 1))]:
        brute = []
        for it in range(1, s + 1):
            for idm in range(1, d + 1):
                for wt in range(1, s + 1):
                    for wd in range(1, d + 1):
                        if s % (it * wt) or d % (idm * wd):
                            continue
                        if it * idm > lim[0] or wt * wd > lim[1]:
                            continue
                        brute.append((it, idm, wt, wd))
        assert sorted(brute) == sorted(O.enumerate_configs(d, s, *lim))


def test_count_loads_match_reference(golden):
    tables = {}
    for g in golden["count_loads"]:
        setup = O.APERTIF if g["setup"] == "Apertif" else O.LOFAR
        if setup.name not in tables:
            tables[setup.name] = O.delay_table(setup, 4096)[0]
        st, idl = O.count_loads(tables[setup.name], setup.samples_per_second, g["config"])
        assert (st, idl) == (g["staged"], g["ideal"])


def test_restatement_agrees_with_compiled_reference_on_random_cases():
    R = O.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built here (reference absent)")
    import ctypes as C
    rng = np.random.default_rng(5)
    for i in range(10):
        setup = O.Setup("r", int(rng.choice([32, 48, 64])), int(rng.integers(1, 20)),
                        float(rng.uniform(60, 300)), float(rng.uniform(0.1, 2)), 0.0,
                        float(rng.uniform(0.1, 1.2)))
        d = int(rng.integers(1, 20))
        sh, md = O.delay_table(setup, d)
        s = setup.samples_per_second
        t = ((s + md + s - 1) // s) * s
        fb = O.noise(setup.channels, t, 0.5, i)
        a = O.dedisperse_reference(fb, sh, s)
        b = np.empty_like(a)
        f32 = C.POINTER(C.c_float)
        assert R.ref_dedisperse_reference(C.byref(setup.c()), fb.ctypes.data_as(f32), t,
                                          sh.ctypes.data_as(C.POINTER(C.c_uint32)), d,
                                          b.ctypes.data_as(f32)) == 0
        assert a.tobytes() == b.tobytes()
