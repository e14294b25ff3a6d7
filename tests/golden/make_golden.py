"""Generate tests/golden/golden.json from the REFERENCE itself.

Run in the dev container (needs /root/reference to build oracle/_ref):

    python tests/golden/make_golden.py

Every number here comes from the unmodified reference core
(oracle/_ref/libdedisp_ref.so, built from /root/reference/proj/core/src by
oracle/Makefile) called through oracle/ref_shim.cpp.  The fixtures then pin
both the C restatement (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py) on the GPU box, where /root/reference is absent.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def ref_table(R, setup, d, zero=False):
    sh = np.empty((d, setup.channels), np.uint32)
    md = C.c_uint32()
    rc = R.ref_build_delay_table(C.byref(setup.c()), d, 1 << 30, int(zero),
                                 sh.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(md))
    assert rc == 0, rc
    return sh, md.value


def ref_sizing(R, setup, d):
    t, f, m = C.c_uint64(), C.c_uint64(), C.c_uint32()
    assert R.ref_instance_sizing(C.byref(setup.c()), d, C.byref(t), C.byref(f), C.byref(m)) == 0
    return t.value, f.value, m.value


def ref_noise(R, setup, t, sigma, seed):
    out = np.empty((setup.channels, t), np.float32)
    assert R.ref_noise_filterbank(C.byref(setup.c()), t, sigma, seed,
                                  out.ctypes.data_as(C.POINTER(C.c_float))) == 0
    return out


def ref_dedisp(R, setup, fb, sh, cfg=None, threads=0):
    d = sh.shape[0]
    out = np.empty((d, setup.samples_per_second), np.float32)
    f32 = C.POINTER(C.c_float)
    u32 = C.POINTER(C.c_uint32)
    if cfg is None:
        rc = R.ref_dedisperse_reference(C.byref(setup.c()), fb.ctypes.data_as(f32), fb.shape[1],
                                        sh.ctypes.data_as(u32), d, out.ctypes.data_as(f32))
    else:
        rc = R.ref_dedisperse_tiled(C.byref(setup.c()), fb.ctypes.data_as(f32), fb.shape[1],
                                    sh.ctypes.data_as(u32), d, C.byref(O.ConfigC(*cfg)),
                                    threads, out.ctypes.data_as(f32))
    assert rc == 0, rc
    return out


def setup_dict(s):
    return dict(name=s.name, samples_per_second=s.samples_per_second, channels=s.channels,
                f_min=s.f_min, channel_width=s.channel_width, dm_first=s.dm_first,
                dm_step=s.dm_step)


def main():
    R = O.ref_lib()
    assert R is not None, "oracle/_ref could not be built (is /root/reference mounted?)"
    golden = {"generator": "tests/golden/make_golden.py via oracle/_ref (unmodified reference)",
              "hash": "fnv1a64 over raw little-endian bytes", "baseline": [], "mini": [],
              "zero_dm": [], "enumerate": [], "count_loads": []}

    # BASELINE-scale fingerprints.  d=4096 outputs use
    # the reference's tiled kernel, which the reference proves bit-identical.
    for setup, d, cfg in [(O.APERTIF, 64, None), (O.LOFAR, 64, None),
                          (O.APERTIF, 4096, (125, 8, 8, 1)), (O.LOFAR, 4096, (1000, 1, 1, 4)),
                          (O.LOFAR, 2, None), (O.APERTIF, 2, None)]:
        t0 = time.time()
        t, flop, md_sz = ref_sizing(R, setup, d)
        sh, md = ref_table(R, setup, d)
        fb = ref_noise(R, setup, t, 1.0, 1)
        out = ref_dedisp(R, setup, fb, sh, cfg)
        golden["baseline"].append(dict(
            setup=setup_dict(setup), num_dms=d, num_samples=t, flop=flop, max_delay=md,
            sizing_max_delay=md_sz, sigma=1.0, seed=1, in_fnv=O.fnv1a(fb), shifts_fnv=O.fnv1a(sh),
            out_fnv=O.fnv1a(out), out_first=float(out.flat[0]), out_last=float(out.flat[-1]),
            out_sum=float(out.astype(np.float64).sum()), out_max=float(out.max()),
            shift_samples={"dm1_ch0": int(sh[1, 0]) if d > 1 else None,
                           "last_ch0": int(sh[-1, 0])},
            produced_by="dedisperse_reference" if cfg is None else f"dedisperse_tiled{cfg}"))
        print(setup.name, d, "%.1fs" % (time.time() - t0), golden["baseline"][-1]["out_fnv"])

    # Randomised mini instances, modelled on acceptance_main.cpp:38-60.
    rng = random.Random(0xACCE0001)
    rates = [24, 32, 48, 64, 96, 128, 192, 256]
    for i in range(40):
        setup = O.Setup("mini%d" % i, rng.choice(rates), rng.randint(1, 64),
                        rng.uniform(50.0, 400.0), rng.uniform(0.05, 2.0), 0.0,
                        rng.uniform(0.05, 1.5))
        d = rng.randint(1, 48)
        sh, md = ref_table(R, setup, d)
        s = setup.samples_per_second
        t = ((s + md + s - 1) // s) * s
        seed = rng.getrandbits(64)
        fb = ref_noise(R, setup, t, 1.0, seed)
        out = ref_dedisp(R, setup, fb, sh)
        golden["mini"].append(dict(setup=setup_dict(setup), num_dms=d, num_samples=t,
                                   max_delay=md, sigma=1.0, seed=seed, in_fnv=O.fnv1a(fb),
                                   shifts_fnv=O.fnv1a(sh), out_fnv=O.fnv1a(out)))

    # Zero-DM table (setup.cpp:107-110) over real noise: every row equal.
    for setup, d in [(O.APERTIF, 8), (O.LOFAR, 4)]:
        sh, md = ref_table(R, setup, d, zero=True)
        t = setup.samples_per_second
        fb = ref_noise(R, setup, t, 1.0, 7)
        out = ref_dedisp(R, setup, fb, sh)
        golden["zero_dm"].append(dict(setup=setup_dict(setup), num_dms=d, num_samples=t,
                                      seed=7, in_fnv=O.fnv1a(fb), out_fnv=O.fnv1a(out)))

    # Config-space sizes and fingerprints (tuner.cpp:103-134).
    buf = (O.ConfigC * 20000)()
    for d, s, lim in [(4096, 20000, (1024, 256)), (4096, 200000, (1024, 256)),
                      (64, 20000, (1024, 256)), (2, 20000, (1024, 256)), (12, 48, (64, 32)),
                      (2, 200000, (1024, 256))]:
        n = R.ref_enumerate_configs(d, s, lim[0], lim[1], buf, 20000)
        arr = np.array([(b.items_time, b.items_dm, b.work_time, b.work_dm) for b in buf[:n]],
                       np.uint32)
        golden["enumerate"].append(dict(num_dms=d, s=s, limits=list(lim), count=int(n),
                                        fnv=O.fnv1a(arr)))

    # count_loads at d=4096.
    for setup, cfg in [(O.APERTIF, (1000, 64, 1, 1)), (O.APERTIF, (125, 8, 8, 1)),
                       (O.APERTIF, (250, 4, 4, 4)), (O.LOFAR, (1000, 1, 1, 4)),
                       (O.LOFAR, (1000, 4, 4, 1))]:
        sh, _ = ref_table(R, setup, 4096)
        st, idl = C.c_uint64(), C.c_uint64()
        assert R.ref_count_loads(C.byref(setup.c()), sh.ctypes.data_as(C.POINTER(C.c_uint32)),
                                 4096, C.byref(O.ConfigC(*cfg)), C.byref(st), C.byref(idl)) == 0
        golden["count_loads"].append(dict(setup=setup.name, num_dms=4096, config=list(cfg),
                                          staged=st.value, ideal=idl.value))

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(golden, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
