"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference-produced golden fixtures.  Bit-exact everywhere (integer tables
and fp32 sums in the reference's order)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1601_05052_b200 import _native as N
from paper_1601_05052_b200 import api

pytestmark = pytest.mark.gpu

K = api.KernelConfig


def _setup(d):
    return api.ObservationSetup(d["name"], d["samples_per_second"], d["channels"], d["f_min"],
                                d["channel_width"], d["dm_first"], d["dm_step"])


def _osetup(s):
    return O.Setup(s.name, s.samples_per_second, s.channels, s.f_min, s.channel_width,
                   s.dm_first, s.dm_step)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.fixture(scope="module")
def dev():
    if api.device_count() == 0:
        pytest.skip("no CUDA device")
    return api.context(0)


# ------------------------------------------------------------- K1 table --
def test_device_table_matches_reference(dev, golden):
    for g in golden["baseline"]:
        setup = _setup(g["setup"])
        t = api.build_delay_table(setup, g["num_dms"])
        assert t.max_delay == g["max_delay"]
        assert O.fnv1a(t.shifts) == g["shifts_fnv"], (setup.name, g["num_dms"])
    for g in golden["mini"]:
        setup = _setup(g["setup"])
        t = api.build_delay_table(setup, g["num_dms"])
        assert O.fnv1a(t.shifts) == g["shifts_fnv"] and t.max_delay == g["max_delay"]


def test_device_table_slices_and_zero(dev):
    import torch
    full = api.build_delay_table(api.APERTIF, 256)
    buf = torch.empty((64, 1024), dtype=torch.int32, device="cuda")
    for off in (0, 64, 192):
        md = dev.delay_table(api.APERTIF, 64, buf.data_ptr(), dm_offset=off)
        dev.synchronize()
        got = buf.cpu().numpy().view(np.uint32)
        assert np.array_equal(got, full.shifts[off:off + 64])
        assert md == full.shifts[off:off + 64].max()
    z = api.build_zero_delay_table(api.LOFAR, 8)
    assert z.max_delay == 0 and not z.shifts.any()
    with pytest.raises(api.CapacityError):
        api.build_delay_table(api.APERTIF, 4096, memory_cap_bytes=1 << 20)
    with pytest.raises(ValueError):
        api.build_delay_table(api.APERTIF, 0)


# --------------------------------------------------- golden full outputs --
def _golden_instance(g):
    setup = _setup(g["setup"])
    table = api.build_delay_table(setup, g["num_dms"])
    fb = api.noise_filterbank(setup, g["num_samples"], g["sigma"], g["seed"])
    assert O.fnv1a(fb.data) == g["in_fnv"]
    return setup, table, fb


APERTIF_CFGS = [
    (None, 1, "auto"),                      # reference-order kernel
    (K(32, 8, 1, 8), 1, "smem"),
    (K(160, 2, 1, 4), 2, "smem"),
    (K(32, 4, 5, 4), 1, "smem"),
    (K(800, 1, 1, 1), 1, "smem"),
    (K(125, 8, 8, 1), 1, "direct"),         # the reference's CPU config
    (K(16, 4, 5, 8), 1, "auto"),
    (K(32, 4, 25, 4), 1, "regwin"),
    (K(32, 8, 5, 8), 1, "regwin"),
    (K(160, 1, 5, 8), 2, "regwin"),
    (K(32, 2, 25, 2), 1, "regwin"),
    (K(32, 2, 5, 8), 1, "regwin"),
]


@pytest.mark.parametrize("cfg,depth,staging", APERTIF_CFGS)
def test_apertif_64_golden(dev, golden, cfg, depth, staging):
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    if cfg is None:
        out = api.dedisperse_reference(fb, table)
    else:
        out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(dm_tile_depth=depth,
                                                                   staging=staging))
    assert O.fnv1a(out.data) == g["out_fnv"]
    assert float(out.data.flat[0]) == g["out_first"] and float(out.data.flat[-1]) == g["out_last"]


@pytest.mark.parametrize("cfg,staging", [(None, "auto"), (K(32, 4, 5, 1), "smem"),
                                         (K(64, 4, 1, 4), "smem"), (K(1000, 1, 1, 4), "direct"),
                                         (K(32, 4, 25, 4), "regwin"), (K(64, 2, 5, 8), "regwin")])
def test_lofar_64_golden(dev, golden, cfg, staging):
    g = golden["baseline"][1]
    setup, table, fb = _golden_instance(g)
    out = (api.dedisperse_reference(fb, table) if cfg is None else
           api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(staging=staging)))
    assert O.fnv1a(out.data) == g["out_fnv"]


@pytest.mark.parametrize("idx", [4, 5])
def test_two_dm_golden(dev, golden, idx):
    g = golden["baseline"][idx]
    setup, table, fb = _golden_instance(g)
    for cfg in (K(32, 2, 1, 1), K(160, 1, 5, 2), K(32, 1, 1, 2)):
        out = api.dedisperse_tiled(fb, table, cfg)
        assert O.fnv1a(out.data) == g["out_fnv"], cfg


def test_apertif_4096_golden(dev, golden):
    g = golden["baseline"][2]
    setup, table, fb = _golden_instance(g)
    for cfg, depth, st in ((K(32, 8, 1, 8), 1, "smem"), (K(160, 1, 5, 8), 2, "smem"),
                           (K(32, 4, 25, 4), 1, "regwin"), (K(32, 8, 5, 8), 2, "regwin")):
        out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(dm_tile_depth=depth,
                                                                   staging=st))
        assert O.fnv1a(out.data) == g["out_fnv"], cfg


def test_lofar_4096_golden(dev, golden):
    g = golden["baseline"][3]
    setup, table, fb = _golden_instance(g)
    out = api.dedisperse_tiled(fb, table, K(32, 8, 5, 2))
    assert O.fnv1a(out.data) == g["out_fnv"]


def _tuned_records(name, d, top):
    """The `top` fastest records of the committed sweep tuning/<name>_<d>.json
    (the first is the tuner's pick, the configuration bench.py times)."""
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tuning",
                        f"{name.lower()}_{d}.json")
    with open(path) as f:
        res = api.tuning_result_from_json(f.read())
    best = res.best()
    rest = sorted((r for r in res.records if r is not best), key=lambda r: -r.gflops)
    return [best] + rest[:top - 1]


@pytest.mark.parametrize("idx,name", [(2, "Apertif"), (3, "LOFAR")])
def test_tuned_configs_at_full_size(dev, golden, idx, name):
    """The exact configurations the bench times -- the tuner's pick for
    Apertif and LOFAR at d=4096 (config, depth, staging and every flag:
    GPU tiling, stage width, raster, packed stages), plus the next fastest
    records -- replayed at full size: the whole output's fingerprint equals
    the reference's (golden, from oracle/_ref)."""
    import torch
    g = golden["baseline"][idx]
    setup, table, fb = _golden_instance(g)
    d, s, c, t = g["num_dms"], setup.samples_per_second, setup.channels, g["num_samples"]
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.empty((d, s), device="cuda")
    for rec in _tuned_records(name, d, 3):
        out.fill_(float("nan"))
        p = dev.plan(sh.data_ptr(), c, d, s, t, t, rec.config, rec.dm_tile_depth, rec.staging,
                     flags=rec.flags)
        assert p.info()["family"] == (rec.family or rec.staging)
        p.execute(x.data_ptr(), out.data_ptr())
        dev.synchronize()
        assert api.fingerprint(out.cpu()) == g["out_fnv"], (rec.config, rec.staging, hex(rec.flags))
        p.close()


# ------------------------------------------------ randomised equivalence --
def test_mini_instances_all_families(dev, golden):
    rng = np.random.default_rng(1)
    checked = 0
    for g in golden["mini"]:
        setup, table, fb = _golden_instance(g)
        d, s = g["num_dms"], setup.samples_per_second
        ref = api.dedisperse_reference(fb, table)
        assert O.fnv1a(ref.data) == g["out_fnv"]
        cfgs = api.enumerate_configs(d, s)
        pick = rng.choice(len(cfgs), size=min(8, len(cfgs)), replace=False)
        for i in pick:
            for staging in ("auto", "direct"):
                out = api.dedisperse_tiled(fb, table, cfgs[i], api.ExecOptions(staging=staging))
                assert np.array_equal(_bits(out.data), _bits(ref.data)), (cfgs[i], staging)
                checked += 1
    assert checked > 300


def test_every_valid_config_is_bit_identical(dev):
    # test_kernels.cpp:116-139: every config under limits {64, 32}
    setup = api.ObservationSetup("mini", 48, 6, 100.0, 25.0, 0.0, 0.5)
    d = 12
    table = api.build_delay_table(setup, d)
    inst = api.instance_sizing(setup, d)
    fb = api.noise_filterbank(setup, inst.num_samples, 1.0, 99)
    ref = O.dedisperse_reference(fb.data, table.shifts, 48)
    lim = api.KernelLimits(64, 32)
    cfgs = api.enumerate_configs(d, 48, lim)
    assert len(cfgs) > 20
    smem_runs = 0
    for cfg in cfgs:
        for depth in (1, 2):
            out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(limits=lim,
                                                                       dm_tile_depth=depth))
            assert np.array_equal(_bits(out.data), _bits(ref)), cfg
        try:
            out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(limits=lim, staging="smem"))
            smem_runs += 1
            assert np.array_equal(_bits(out.data), _bits(ref)), cfg
        except ValueError:
            pass  # no staged variant for this shape: an explicit error, never a fallback
    assert smem_runs > 50


def test_oversize_blocks_and_many_accumulators(dev):
    # configs the reference accepts under raised limits must run too
    setup = api.ObservationSetup("wide", 2048, 5, 120.0, 3.0, 0.0, 0.4)
    d = 16
    table = api.build_delay_table(setup, d)
    t = api.instance_sizing(setup, d).num_samples
    fb = api.noise_filterbank(setup, t, 1.0, 3)
    ref = O.dedisperse_reference(fb.data, table.shifts, 2048)
    lim = api.KernelLimits(1 << 20, 1 << 20)
    for cfg in (K(2048, 2, 1, 1), K(1, 1, 256, 1), K(8, 1, 16, 16), K(1024, 4, 2, 4)):
        out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(limits=lim))
        assert np.array_equal(_bits(out.data), _bits(ref)), cfg


def test_non_monotone_and_fault_injected_tables(dev, golden):
    # the kernels assume no ordering of table entries (kernels.cpp:147-156)
    rng = np.random.default_rng(2)
    setup = api.ObservationSetup("rand", 320, 24, 300.0, 1.0, 0.0, 0.5)
    d = 32
    sh = rng.integers(0, 700, size=(d, 24), dtype=np.uint32)
    table = api.DelayTable(setup, d, sh, int(sh.max()))
    t = ((320 + int(sh.max()) + 319) // 320) * 320
    fb = api.noise_filterbank(setup, t, 1.0, 5)
    ref = O.dedisperse_reference(fb.data, sh, 320)
    for cfg, st in ((K(32, 4, 5, 2), "smem"), (K(160, 2, 1, 16), "smem"),
                    (K(32, 8, 1, 4), "direct"), (K(32, 2, 5, 8), "regwin")):
        out = api.dedisperse_tiled(fb, table, cfg, api.ExecOptions(staging=st))
        assert np.array_equal(_bits(out.data), _bits(ref)), cfg
    # near-monotone table with jitter: register-window fast and slow paths mix
    base = (np.arange(d)[:, None] * np.linspace(9, 0, 24)[None, :]).astype(np.int64)
    jit = rng.integers(0, 3, size=(d, 24)) * rng.integers(0, 2, size=(d, 24)) * 7
    sh2 = (base + jit).astype(np.uint32)
    table2 = api.DelayTable(setup, d, sh2, int(sh2.max()))
    t2 = ((320 + int(sh2.max()) + 319) // 320) * 320
    fb2 = api.noise_filterbank(setup, t2, 1.0, 6)
    ref2 = O.dedisperse_reference(fb2.data, sh2, 320)
    for cfg in (K(32, 1, 5, 8), K(32, 2, 5, 8), K(32, 4, 5, 8)):
        out = api.dedisperse_tiled(fb2, table2, cfg, api.ExecOptions(staging="regwin"))
        assert np.array_equal(_bits(out.data), _bits(ref2)), cfg
    # TMEM windows with the same jittered table (GPU tiling: 384 does not divide 320*k)
    import torch
    x = torch.from_numpy(fb2.data).cuda()
    shd = torch.from_numpy(sh2.view(np.int32)).cuda()
    outd = torch.empty((d, 320), device="cuda")
    torch.cuda.synchronize()
    for cfg in (K(32, 2, 12, 4), K(32, 1, 12, 8), K(32, 4, 12, 2)):
        p = dev.plan(shd.data_ptr(), 24, d, 320, t2, t2, cfg, 1, "tmem", gpu_tiling=True)
        p.execute(x.data_ptr(), outd.data_ptr())
        dev.synchronize()
        assert np.array_equal(_bits(outd.cpu().numpy()), _bits(ref2)), cfg
    # dedisp_tune.cpp:278-287 analogue: one corrupted entry must change the output
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    table.shifts[17, 3] += 1
    out = api.dedisperse_tiled(fb, table, K(32, 8, 1, 8))
    assert O.fnv1a(out.data) != g["out_fnv"]
    assert np.array_equal(_bits(out.data), _bits(O.dedisperse_reference(fb.data, table.shifts,
                                                                         20000)))


@pytest.mark.parametrize("spec", [
    ("regwin", K(32, 4, 20, 2), 8), ("regwin", K(32, 4, 12, 4), 4), ("regwin", K(32, 2, 12, 8), 8),
    ("regwin", K(64, 2, 20, 4), 4), ("smem", K(32, 4, 4, 4), 8), ("smem", K(96, 2, 1, 8), 2),
    ("tmem", K(32, 4, 12, 4), 8), ("tmem", K(32, 8, 12, 4), 4), ("tmem", K(64, 2, 12, 2), 8),
    ("tmem", K(32, 4, 20, 2), 8), ("tmem", K(32, 4, 12, 8), 4), ("tmem", K(32, 8, 20, 4), 8),
    ("tmem", K(32, 4, 4, 8), 8), ("tmem", K(32, 2, 4, 16), 8), ("tmem", K(32, 4, 8, 8), 4),
    ("tmem", K(32, 4, 4, 8), 8, "occ"), ("tmem", K(32, 4, 12, 4), 8, "occ"),
    ("tmem", K(32, 4, 4, 4), 4, "occ"), ("tmem", K(32, 4, 8, 4), 8, "occ"),
    ("tmem", K(32, 2, 12, 8), 3), ("tmem", K(32, 1, 12, 8), 1), ("tmem", K(32, 4, 20, 4), 2),
    ("tmem", K(32, 4, 12, 8), 15), ("tmem", K(32, 4, 12, 8), 11), ("smem", K(32, 4, 4, 4), 13),
    ("regwin", K(32, 4, 12, 4), 15), ("tmem", K(32, 4, 12, 8), 15, "tm"),
    ("smem", K(32, 4, 4, 4), 8, "tm"), ("regwin", K(32, 4, 12, 4), 4, "tm"),
    ("tmem", K(32, 4, 12, 8), 0, "packed"), ("smem", K(32, 4, 4, 4), 0, "packed"),
    ("regwin", K(32, 4, 12, 4), 0, "packed")])
def test_gpu_tiling_predicated_tail(dev, golden, spec):
    """GPU-native tiles whose tile_time does not divide s (vector register
    windows, odd smem tiles, TMEM windows incl. the three-CTA builds): the
    predicated last tile must not change a bit."""
    import torch
    staging, cfg, cps = spec[:3]
    mode = spec[3] if len(spec) > 3 else ""
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    d, s, c, t = g["num_dms"], setup.samples_per_second, setup.channels, g["num_samples"]
    assert s % cfg.tile_time() != 0
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.full((d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, 1, staging, gpu_tiling=True,
                 stage_channels=cps, high_occupancy=mode == "occ",
                 flags=(N.DD_CONFIG_TIME_MAJOR if mode == "tm" else 0)
                 | (N.DD_CONFIG_PACKED_STAGES if mode == "packed" else 0))
    info = p.info()
    assert info["family"] == staging and (mode == "packed" or info["channels_per_stage"] == cps)
    if mode == "occ":
        assert 0 < info["registers"] <= 128
    p.execute(x.data_ptr(), out.data_ptr())
    dev.synchronize()
    assert O.fnv1a(out.cpu().numpy()) == g["out_fnv"]
    with pytest.raises(ValueError):  # the reference rule still holds without the flag
        dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, 1, staging)


def test_power_of_two_scaling_is_exact(dev):
    # test_signal.cpp:169-183 / SPEC linearity: x2 input -> exactly x2 output
    setup = api.APERTIF
    table = api.build_delay_table(setup, 32)
    fb = api.noise_filterbank(setup, 40000, 1.0, 4)
    a = api.dedisperse_tiled(fb, table, K(32, 4, 5, 8))
    fb.data *= 2.0
    b = api.dedisperse_tiled(fb, table, K(32, 4, 5, 8))
    assert np.array_equal(_bits(b.data), _bits(a.data * 2.0))


def test_zero_dm_reduces_to_column_sums(dev, golden):
    for g in golden["zero_dm"]:
        setup = _setup(g["setup"])
        table = api.build_zero_delay_table(setup, g["num_dms"])
        fb = api.noise_filterbank(setup, g["num_samples"], 1.0, g["seed"])
        out = api.dedisperse_tiled(fb, table, K(32, 2, 5, 2) if setup.name == "Apertif"
                                   else K(32, 2, 1, 2))
        assert O.fnv1a(out.data) == g["out_fnv"]


def test_input_rejection_and_stats(dev):
    # test_kernels.cpp:183-227
    setup = api.ObservationSetup("mini", 32, 4, 100.0, 25.0, 0.0, 0.5)
    table = api.build_delay_table(setup, 4)
    short = api.noise_filterbank(setup, 32, 0.0, 0)
    if table.max_delay > 0:
        with pytest.raises(ValueError):
            api.dedisperse_reference(short, table)
    other = api.noise_filterbank(api.ObservationSetup("mini", 32, 8, 100.0, 25.0, 0.0, 0.5), 64,
                                 0.0, 0)
    with pytest.raises(ValueError):
        api.dedisperse_reference(other, table)
    fb = api.noise_filterbank(setup, api.instance_sizing(setup, 4).num_samples, 1.0, 1)
    with pytest.raises(ValueError):
        api.dedisperse_tiled(fb, table, K(3, 1, 1, 1))
    stats = api.KernelStats()
    setup6 = api.ObservationSetup("mini", 64, 6, 100.0, 25.0, 0.0, 0.5)
    t6 = api.build_delay_table(setup6, 8)
    fb6 = api.noise_filterbank(setup6, api.instance_sizing(setup6, 8).num_samples, 1.0, 1)
    api.dedisperse_reference(fb6, t6, stats)
    assert stats.flop_additions == 8 * 64 * 6 == stats.staged_loads
    stats.reset()
    api.dedisperse_tiled(fb6, t6, K(8, 2, 2, 2), api.ExecOptions(stats=stats))
    assert stats.flop_additions == 8 * 64 * 6
    assert stats.staged_loads == api.count_loads(t6, K(8, 2, 2, 2), 8, 64).staged_loads


def test_dm_shards_concatenate_to_full_output(dev):
    """The multi-GPU decomposition (contiguous DM ranges, table slices built
    with dm_offset) reproduces the single-device output exactly; emulated
    shard by shard on one device."""
    import torch
    setup, d, n = api.APERTIF, 512, 4
    s, c = setup.samples_per_second, setup.channels
    t = api.instance_sizing(setup, d).num_samples
    fb = api.noise_filterbank(setup, t, 1.0, 1)
    full = api.dedisperse_tiled(fb, api.build_delay_table(setup, d), K(32, 8, 1, 8))
    x = torch.from_numpy(fb.data).cuda()
    torch.cuda.synchronize()
    per = d // n
    parts = []
    for r in range(n):
        sh = torch.empty((per, c), dtype=torch.int32, device="cuda")
        dev.delay_table(setup, per, sh.data_ptr(), dm_offset=r * per)
        out = torch.empty((per, s), dtype=torch.float32, device="cuda")
        dev.synchronize()
        p = dev.plan(sh.data_ptr(), c, per, s, t, t, K(32, 8, 1, 8))
        p.execute(x.data_ptr(), out.data_ptr())
        dev.synchronize()
        parts.append(out.cpu().numpy())
    assert np.array_equal(_bits(np.concatenate(parts)), _bits(full.data))


def test_tuner_on_device(dev):
    res = api.tune(api.APERTIF, 64, repeats=2, max_configs=12)
    assert len(res.records) == 12
    assert res.best().gflops == max(r.gflops for r in res.records)
    assert res.realtime_threshold_gflops == pytest.approx(64 * 20000 * 1024 / 1e9)
    z = api.zero_dm_experiment(api.LOFAR, 8, repeats=1, max_configs=4)
    assert z.zero_dm and len(z.records) == 4


def test_sharded_driver_host_pipeline(dev, golden):
    """multi.ShardedDedisperser end to end from pinned host memory with the
    DM-chunk pipeline (kernel of chunk i+1 overlapping D2H of chunk i)."""
    import torch
    from paper_1601_05052_b200 import multi
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    dd = multi.ShardedDedisperser(setup, g["num_dms"], K(16, 8, 10, 4), 1, "smem", device=0,
                                  stage_channels=8)
    dd.pipeline(3, 4, h2d="channels")
    assert len(dd.groups) == 4
    host = torch.from_numpy(fb.data).pin_memory()
    out = torch.empty((dd.count, setup.samples_per_second), dtype=torch.float32).pin_memory()
    dd.run_host(host, out)
    torch.cuda.synchronize()
    assert O.fnv1a(out.numpy()) == g["out_fnv"]
    # time-ordered H2D (dd_upload_block_range): low-DM chunks start on a
    # prefix of the block; the uploads cover the whole block by the end
    dd.block.fill_(float("nan"))
    out.zero_()
    dd.pipeline(5, h2d="time")
    assert dd.h2d_mode == "time"
    ups = [u for u, _ in dd.uploads]
    assert ups == sorted(ups) and ups[0] < dd.num_samples and ups[-1] <= dd.num_samples
    dd.run_host(host, out)
    torch.cuda.synchronize()
    assert O.fnv1a(out.numpy()) == g["out_fnv"]
    dd.run()
    torch.cuda.synchronize()
    assert O.fnv1a(dd.out.cpu().numpy()) == g["out_fnv"]
    # streamed consecutive blocks, double-buffered: the second block is the
    # first times 2 (exact in fp32), so its output is the golden one times 2
    ref = out.numpy().copy()
    host2 = (host * 2).pin_memory()
    outs = [torch.full_like(out, float("nan")).pin_memory() for _ in range(2)]
    for steps in (5, 2):
        for o in outs:
            o.fill_(float("nan"))
        dd.stream_host([host, host2], outs, steps)
        torch.cuda.synchronize()
        last = steps - 1
        assert np.array_equal(_bits(outs[last % 2].numpy()),
                              _bits(ref * (2 if last % 2 else 1)))
        assert np.array_equal(_bits(outs[(last - 1) % 2].numpy()),
                              _bits(ref * (2 if (last - 1) % 2 else 1)))
    # the TMEM family with GPU tiling, same pipeline
    dd2 = multi.ShardedDedisperser(setup, g["num_dms"], K(32, 4, 12, 8), 1, "tmem", device=0,
                                   gpu_tiling=True, stage_channels=8)
    dd2.pipeline(2, 3)
    out.zero_()
    dd2.run_host(host, out)
    torch.cuda.synchronize()
    assert O.fnv1a(out.numpy()) == g["out_fnv"]
    # the first driver still launches on its own stream with dd2 alive (each
    # driver owns its context), so its events still cover its kernels
    assert dd.ctx.handle.value != dd2.ctx.handle.value
    for o in outs:
        o.fill_(float("nan"))
    dd.stream_host([host, host2], outs, 3)
    torch.cuda.synchronize()
    assert O.fnv1a(outs[0].numpy()) == g["out_fnv"]
    assert np.array_equal(_bits(outs[1].numpy()), _bits(ref * 2))


@pytest.mark.parametrize("staging,cfg,tiling", [("smem", K(16, 8, 10, 4), False),
                                                ("tmem", K(32, 4, 12, 8), True),
                                                ("regwin", K(32, 4, 25, 2), False)])
def test_channel_range_passes_are_bit_identical(dev, golden, staging, cfg, tiling):
    """dd_plan_execute_channels: ascending channel ranges accumulating through
    the output equal one pass bit for bit (the streamed-input e2e path)."""
    import torch
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    d, s, c, t = g["num_dms"], setup.samples_per_second, setup.channels, g["num_samples"]
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.full((d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, 1, staging, gpu_tiling=tiling)
    for i, (c0, c1) in enumerate([(0, 100), (100, 101), (101, 640), (640, 1024)]):
        p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0)
    dev.synchronize()
    assert O.fnv1a(out.cpu().numpy()) == g["out_fnv"]


@pytest.mark.parametrize("staging,cfg,tiling", [("smem", K(16, 8, 10, 4), False),
                                                ("tmem", K(32, 4, 12, 8), True),
                                                ("tm-smem", K(16, 8, 10, 4), False),
                                                ("tm-tmem", K(32, 4, 12, 8), True)])
def test_beam_batching(dev, golden, staging, cfg, tiling):
    """dd_plan_execute_beams: B independent beams in one launch equal B single
    passes.  Beam b is the golden block times 2^b (exact in fp32), so every
    beam's whole output is the reference's output times 2^b, bit for bit."""
    import torch
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    d, beams = g["num_dms"], 3
    s, c, t = setup.samples_per_second, setup.channels, g["num_samples"]
    blocks = [fb.data * np.float32(2.0 ** b) for b in range(beams)]
    x = torch.from_numpy(np.stack(blocks)).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.full((beams, d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    tm = staging.startswith("tm-")
    p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, 1, staging.replace("tm-", ""),
                 gpu_tiling=tiling, flags=N.DD_CONFIG_TIME_MAJOR if tm else 0)
    assert p.info()["time_major"] == int(tm)
    p.execute_beams(beams, x.data_ptr(), c * t, out.data_ptr(), d * s)
    dev.synchronize()
    got = out.cpu().numpy()
    assert api.fingerprint(got[0]) == g["out_fnv"]
    for b in range(1, beams):
        assert np.array_equal(_bits(got[b]), _bits(got[0] * np.float32(2.0 ** b))), b


def test_block_stream_matches_one_shot(dev):
    """stream.BlockStream: consecutive seconds pushed one at a time give, for
    every full window, exactly the one-shot pass over the same samples."""
    import torch
    from paper_1601_05052_b200.stream import BlockStream
    setup = api.ObservationSetup("strm", 320, 24, 300.0, 1.0, 0.0, 0.5)
    d = 32
    st = BlockStream(setup, d, K(32, 2, 5, 8), 1, "smem", device=0)
    s, t = setup.samples_per_second, st.t
    total = t + 6 * s
    series = api.noise_filterbank(setup, total, 1.0, 21).data
    table = api.build_delay_table(setup, d)
    outs = []
    for n in range(total // s):
        o = st.push(torch.from_numpy(series[:, n * s:(n + 1) * s]).cuda())
        if o is not None:
            st.stream.synchronize()
            outs.append(o.cpu().numpy().copy())
    assert len(outs) == (total - t) // s + 1
    for i, o in enumerate(outs):
        ref = O.dedisperse_reference(np.ascontiguousarray(series[:, i * s:i * s + t]),
                                     table.shifts, s)
        assert np.array_equal(_bits(o), _bits(ref)), i
    # the ring moved the window's tail to the front only once per R pushes
    assert st.ring and 0 < st.compactions <= (total // s) // st.rounds + 1


@pytest.mark.parametrize("t,c", [(1001, 37), (40000, 1024), (3, 1), (257, 32)])
def test_sigproc_transpose_matches_reference(dev, t, c):
    """dd_sigproc_to_filterbank against the reference's own parse_sigproc
    (oracle/_ref, sigproc.cpp:83-191) on the same generated stream: the
    channel-major lowest-first block bit for bit, and the first non-finite
    sample at the byte offset the reference's format_error reports."""
    import torch
    if O.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(t + c)
    payload = rng.standard_normal((t, c)).astype(np.float32)
    stream = O.sigproc_bytes(payload, 20000, 1716.67, -0.29)
    header_end = len(stream) - payload.nbytes
    expect, _ = O.ref_parse_sigproc(stream)
    src = torch.from_numpy(payload).cuda()
    pitch = (t + 3) // 4 * 4
    dst = torch.zeros((c, pitch), device="cuda")
    torch.cuda.synchronize()
    bad = dev.sigproc_to_filterbank(src.data_ptr(), c, t, dst.data_ptr(), pitch)
    assert bad == -1
    assert np.array_equal(_bits(dst.cpu().numpy()[:, :t]), _bits(expect))
    if t * c > 2:
        payload[t // 2, c // 2] = np.inf
        payload[-1, 0] = np.nan
        _, offset = O.ref_parse_sigproc(O.sigproc_bytes(payload, 20000, 1716.67, -0.29))
        src = torch.from_numpy(payload).cuda()
        torch.cuda.synchronize()
        first = dev.sigproc_to_filterbank(src.data_ptr(), c, t, dst.data_ptr(), pitch)
        assert header_end + 4 * first == offset


@pytest.mark.parametrize("flags", [0, "tm", "tm-ns2", "cps3-ns4", "packed", "tm-packed",
                                   "packed-ns3"])
def test_large_delay_instance_all_rasters(dev, flags):
    """LOFAR-shaped delays (hundreds of samples per DM step, a block several
    seconds long): every CTA raster and stage shape, including channel-range
    passes accumulating through the output, reproduces the reference."""
    import torch
    setup = api.ObservationSetup("lofarish", 2000, 16, 138.0, 0.19, 0.0, 25.0)
    d = 64
    table = api.build_delay_table(setup, d)
    t = api.instance_sizing(setup, d).num_samples
    s, c = setup.samples_per_second, setup.channels
    assert table.max_delay > 4 * s
    fb = api.noise_filterbank(setup, t, 1.0, 33)
    ref = O.dedisperse_reference(fb.data, table.shifts, s)
    f = 0
    if "tm" in str(flags):
        f |= N.DD_CONFIG_TIME_MAJOR
    if "ns2" in str(flags):
        f |= 2 << N.DD_CONFIG_NSTAGE_SHIFT
    if "cps3" in str(flags):
        f |= (3 << N.DD_CONFIG_CPS_SHIFT) | (4 << N.DD_CONFIG_NSTAGE_SHIFT)
    if "packed" in str(flags):
        f |= N.DD_CONFIG_PACKED_STAGES
    if "ns3" in str(flags):
        f |= 3 << N.DD_CONFIG_NSTAGE_SHIFT
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    for cfg, depth in ((K(16, 4, 25, 1), 2), (K(40, 1, 10, 4), 1), (K(25, 2, 8, 2), 1)):
        out = torch.full((d, s), float("nan"), device="cuda")
        torch.cuda.synchronize()
        p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, depth, "smem", flags=f)
        p.execute(x.data_ptr(), out.data_ptr())
        dev.synchronize()
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref)), (cfg, flags)
        out.fill_(float("nan"))
        for i, (c0, c1) in enumerate([(0, 5), (5, 6), (6, 16)]):
            p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0)
        dev.synchronize()
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref)), (cfg, flags, "channels")
    # the drop-in (AUTO) path on the same instance
    got = api.dedisperse_tiled(fb, table, K(40, 1, 10, 4))
    assert np.array_equal(_bits(got.data), _bits(ref))


@pytest.mark.parametrize("name,d", [("Apertif", 64), ("LOFAR", 64)])
def test_every_gpu_space_config_is_bit_exact(dev, golden, name, d):
    """Every configuration the GPU tuner can select (dd_enumerate_gpu_configs:
    all families, depths, stage shapes, rasters, occupancy builds) reproduces
    the reference on one instance -- the auto-tuner may pick any of them."""
    import torch
    g = [b for b in golden["baseline"] if b["setup"]["name"] == name and b["num_dms"] == d][0]
    setup, table, fb = _golden_instance(g)
    t = g["num_samples"]
    s, c = setup.samples_per_second, setup.channels
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    # the whole output of every configuration against the reference-order
    # kernel's, which is first pinned to the reference's fingerprint
    ref = torch.empty((d, s), device="cuda")
    dev.plan(sh.data_ptr(), c, d, s, t, t).execute(x.data_ptr(), ref.data_ptr())
    dev.synchronize()
    assert api.fingerprint(ref.cpu()) == g["out_fnv"]
    ref_bits = ref.view(torch.int32)
    out = torch.empty((d, s), device="cuda")
    space = api.enumerate_gpu_configs(setup, d)
    assert len(space) > 100
    families, rejected = set(), 0
    for cfg, depth, staging, flags in space:
        out.fill_(float("nan"))
        try:  # the tuner skips what the plan rejects for this table (dd_tune)
            p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, depth, staging, flags=flags)
        except ValueError:
            # K6 rectangles are enumerated for every d <= 128 and rejected by
            # the plan when a group's delay span exceeds the 256-sample TMA
            # box (all of LOFAR's): not counted against the space
            rejected += staging != "rect"
            continue
        families.add(p.info()["family"])
        p.execute(x.data_ptr(), out.data_ptr())
        dev.synchronize()
        assert torch.equal(out.view(torch.int32), ref_bits), (cfg, depth, staging, hex(flags))
        p.close()
    assert {"smem", "direct"} <= families
    assert rejected < len(space) // 4


@pytest.mark.parametrize("cfg,depth", [(K(64, 4, 25, 1), 2), (K(160, 1, 10, 4), 1),
                                       (K(64, 2, 25, 2), 1)])
def test_packed_stages_bit_exact(dev, cfg, depth):
    """DD_CONFIG_PACKED_STAGES on a wide-delay instance (LOFAR-like band):
    stages packed by each channel's own window width -- full passes, beams
    and (fixed-slot fallback) channel-range passes all reproduce the
    reference."""
    import torch
    setup = api.ObservationSetup("packed", 3200, 16, 138.0, 0.19, 0.0, 25.0)
    d = 32
    table = api.build_delay_table(setup, d)
    t = api.instance_sizing(setup, d).num_samples
    s, c = setup.samples_per_second, setup.channels
    fb = api.noise_filterbank(setup, t, 1.0, 44)
    ref = O.dedisperse_reference(fb.data, table.shifts, s)
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.full((d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p = dev.plan(sh.data_ptr(), c, d, s, t, t, cfg, depth, "smem",
                 flags=N.DD_CONFIG_PACKED_STAGES | N.DD_CONFIG_TIME_MAJOR)
    info = p.info()
    assert info["packed_stages"] > 0 and info["packed_stages"] < c
    p.execute(x.data_ptr(), out.data_ptr())
    dev.synchronize()
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref))
    out.fill_(float("nan"))
    for i, (c0, c1) in enumerate([(0, 3), (3, 11), (11, 16)]):
        p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0)
    dev.synchronize()
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref))
    xb = torch.stack([x, x * 2.0])
    ob = torch.full((2, d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p.execute_beams(2, xb.data_ptr(), c * t, ob.data_ptr(), d * s)
    dev.synchronize()
    assert np.array_equal(_bits(ob[0].cpu().numpy()), _bits(ref))
    assert np.array_equal(_bits(ob[1].cpu().numpy()), _bits(ref * 2.0))


def test_live_plan_survives_a_smaller_plan_of_the_same_kernel(dev):
    """A kernel's dynamic shared-memory attribute is per function, not per
    plan: a plan created later with narrower stages (less shared memory) on
    the same kernel must not break the launches of a live wider plan."""
    import torch
    g_setup, d = api.APERTIF, 64
    table = api.build_delay_table(g_setup, d)
    t = api.instance_sizing(g_setup, d).num_samples
    s, c = g_setup.samples_per_second, g_setup.channels
    fb = api.noise_filterbank(g_setup, t, 1.0, 1)
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    ref = torch.empty((d, s), device="cuda")
    dev.plan(sh.data_ptr(), c, d, s, t, t).execute(x.data_ptr(), ref.data_ptr())
    wide = dev.plan(sh.data_ptr(), c, d, s, t, t, K(32, 8, 5, 1), 1, "smem",
                    flags=15 << N.DD_CONFIG_CPS_SHIFT)
    narrow = dev.plan(sh.data_ptr(), c, d, s, t, t, K(32, 8, 5, 1), 1, "smem",
                      flags=(1 << N.DD_CONFIG_CPS_SHIFT) | (2 << N.DD_CONFIG_NSTAGE_SHIFT))
    assert wide.info()["smem_bytes"] > narrow.info()["smem_bytes"]
    for p in (wide, narrow, wide):
        out = torch.full((d, s), float("nan"), device="cuda")
        p.execute(x.data_ptr(), out.data_ptr())
        dev.synchronize()
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32))


@pytest.mark.parametrize("idx,cfg,flags", [
    (5, K(96, 1, 1, 2), 4 << 8), (5, K(64, 1, 2, 2), 2 << 8), (5, K(128, 1, 1, 2), 0),
    (0, K(32, 4, 1, 4), 0), (0, K(16, 8, 2, 4), 2 << 8), (0, K(32, 8, 1, 8), 0),
])
def test_rect_family_golden(dev, golden, idx, cfg, flags):
    """K6 (staging "rect", one 3-D TMA box per channel group) on the golden
    small-d instances: the whole output's fingerprint equals the
    reference's, for full passes, channel-range passes and beams."""
    import torch
    g = golden["baseline"][idx]
    setup, table, fb = _golden_instance(g)
    d, s, c, t = g["num_dms"], setup.samples_per_second, setup.channels, g["num_samples"]
    pitch = (t + 3) // 4 * 4
    x = torch.zeros((c, pitch), device="cuda")
    x[:, :t] = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
    out = torch.full((d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p = dev.plan(sh.data_ptr(), c, d, s, t, pitch, cfg, 1, "rect",
                 flags=flags | N.DD_CONFIG_GPU_TILING)
    assert p.info()["family"] == "rect"
    p.execute(x.data_ptr(), out.data_ptr())
    dev.synchronize()
    assert api.fingerprint(out.cpu()) == g["out_fnv"]
    out.fill_(float("nan"))
    for i, (c0, c1) in enumerate([(0, c // 3), (c // 3, c // 3 + 1), (c // 3 + 1, c)]):
        if c1 > c0:
            p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0)
    dev.synchronize()
    assert api.fingerprint(out.cpu()) == g["out_fnv"]
    xb = torch.stack([x, x * 2.0])
    ob = torch.full((2, d, s), float("nan"), device="cuda")
    torch.cuda.synchronize()
    p.execute_beams(2, xb.data_ptr(), c * pitch, ob.data_ptr(), d * s)
    dev.synchronize()
    assert api.fingerprint(ob[0].cpu()) == g["out_fnv"]
    assert torch.equal(ob[1].view(torch.int32), (ob[0] * 2.0).view(torch.int32))


def test_rect_family_non_monotone_table(dev):
    """K6 assumes no ordering of the shifts (group lows by min scan): a
    fault-injected table still reproduces the reference-order kernel."""
    import torch
    setup, d = api.APERTIF, 8
    table = api.build_delay_table(setup, d)
    sh_np = table.shifts.copy()
    sh_np[3, ::5] = 0
    sh_np[6, 10:40] += 9
    t = api.instance_sizing(setup, d).num_samples
    s, c = setup.samples_per_second, setup.channels
    fb = api.noise_filterbank(setup, t, 1.0, 2)
    x = torch.from_numpy(fb.data).cuda()
    sh = torch.from_numpy(sh_np.view(np.int32)).cuda()
    ref = torch.empty((d, s), device="cuda")
    dev.plan(sh.data_ptr(), c, d, s, t, t).execute(x.data_ptr(), ref.data_ptr())
    out = torch.full((d, s), float("nan"), device="cuda")
    p = dev.plan(sh.data_ptr(), c, d, s, t, t, K(64, 2, 1, 4), 1, "rect",
                 flags=N.DD_CONFIG_GPU_TILING)
    p.execute(x.data_ptr(), out.data_ptr())
    dev.synchronize()
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
    with pytest.raises(ValueError):  # spans beyond one TMA box: not this family
        dev.plan(sh.data_ptr(), c, d, s, t, t, K(256, 1, 1, 8), 1, "rect",
                 flags=N.DD_CONFIG_GPU_TILING | (1 << N.DD_CONFIG_CPS_SHIFT)).close()


@pytest.mark.parametrize("rate,cfg", [(320, None), (322, K(32, 2, 5, 8))])
def test_c_abi_block_stream(dev, rate, cfg):
    """dd_block_stream_*: the streaming-ingest entry point of the C-ABI.  Each
    pushed second yields, once the window is full, exactly the one-shot
    pass over the same samples (checked against the oracle); with s % 4 != 0
    the window is compacted through a temporary on every slide."""
    import ctypes as C
    setup = api.ObservationSetup("strm", rate, 24, 300.0, 1.0, 0.0, 0.5)
    d, s = 32, rate
    h = C.c_void_p()
    kc = None
    if cfg is not None:
        kc = N.dd_config(cfg.items_time, cfg.items_dm, cfg.work_time, cfg.work_dm, 1,
                         N.STAGING["smem"], N.DD_CONFIG_GPU_TILING)
    N.check(N.lib().dd_block_stream_create(dev.handle, C.byref(setup.c()), d,
                                           C.byref(kc) if kc is not None else None, C.byref(h)))
    t = api.instance_sizing(setup, d).num_samples
    total = t + 6 * s
    series = api.noise_filterbank(setup, total, 1.0, 23).data
    table = api.build_delay_table(setup, d)
    out = np.empty((d, s), np.float32)
    produced, got = C.c_int(), []
    for n in range(total // s):
        sec = np.ascontiguousarray(series[:, n * s:(n + 1) * s])
        N.check(N.lib().dd_block_stream_push(h, sec.ctypes.data, out.ctypes.data,
                                             C.byref(produced)))
        if produced.value:
            got.append(out.copy())
    assert len(got) == (total - t) // s + 1
    for i, o in enumerate(got):
        ref = O.dedisperse_reference(np.ascontiguousarray(series[:, i * s:i * s + t]),
                                     table.shifts, s)
        assert np.array_equal(_bits(o), _bits(ref)), i
    comp = C.c_uint64()
    N.check(N.lib().dd_block_stream_info(h, None, None, None, C.byref(comp), None))
    assert comp.value >= 1
    N.check(N.lib().dd_block_stream_destroy(h))


def test_sharded_route_on_one_rank(dev, golden):
    """The N-rank e2e route (each rank's channel-group share H2D, the
    per-group all-gather -- a no-op at N = 1 --, kernels accumulating group by
    group, per-chunk D2H) run on one GPU: one block and a double-buffered
    stream, whole outputs against the reference's fingerprint."""
    import torch
    from paper_1601_05052_b200 import multi
    g = golden["baseline"][0]
    setup, table, fb = _golden_instance(g)
    dd = multi.ShardedDedisperser(setup, g["num_dms"], K(32, 4, 12, 8), 1, "tmem", device=0,
                                  gpu_tiling=True, stage_channels=15)
    dd.pipeline(4, 4, h2d="sharded")
    assert dd.h2d_mode == "sharded" and len(dd.groups) == 4
    assert dd.h2d_bytes() == setup.channels * dd.num_samples * 4
    host = torch.from_numpy(fb.data).pin_memory()
    out = torch.full((dd.count, setup.samples_per_second), float("nan")).pin_memory()
    dd.run_host(host, out)
    torch.cuda.synchronize()
    assert O.fnv1a(out.numpy()) == g["out_fnv"]
    host2 = (host * 2).pin_memory()
    outs = [torch.full_like(out, float("nan")).pin_memory() for _ in range(2)]
    dd.stream_host([host, host2], outs, 5)
    torch.cuda.synchronize()
    assert O.fnv1a(outs[0].numpy()) == g["out_fnv"]  # block 4 = host
    ref = out.numpy()
    assert np.array_equal(_bits(outs[1].numpy()), _bits(ref * 2))  # block 3 = host2
