"""Small launches of every kernel family under the bounds-checked build
(SURVEY.md §5's memcheck row; compute-sanitizer is not available on the
GPU pool):

    DDB_LIB=paper_1601_05052_b200/libdedisp_b200_checked.so python tools/sanitize_cases.py

(with compute-sanitizer where a pool allows it, the same script is its
workload: compute-sanitizer --tool memcheck|racecheck|synccheck python ...).

Apertif d=64 (K1 table, k_plan, K2 reference order, K2' direct, K3 shared
memory with fixed and packed stages, K4 register windows, K5 TMEM windows,
with GPU tiling's predicated last tile) and a LOFAR-like wide-delay instance
(time-major raster, packed stages), plus channel-range passes and beams.
Every output is compared with the reference-order kernel bit for bit; the
output sits between guard rows holding a sentinel pattern that must survive
(out-of-bounds stores); a non-monotone (fault-injected) table drives the
window kernels' slow paths; and the checked build's device-side counter of
out-of-bounds shared-memory reads, bulk copies and stores must stay 0.
`--quick` runs only the K3/K5/k_plan cases."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1601_05052_b200 import _native as N
    from paper_1601_05052_b200 import api

    import ctypes as C
    quick = "--quick" in sys.argv
    K = api.KernelConfig
    ctx = api.context(0)
    nviol, checked = C.c_uint64(), C.c_int()
    N.check(N.lib().dd_debug_violations(C.byref(nviol), C.byref(checked), 1))
    print(f"library: {N.LIB_PATH} (bounds-checked build: {bool(checked.value)})", flush=True)
    SENT = 0x7fc0dead  # a NaN payload no kernel produces
    cases = [
        ("Apertif", api.APERTIF, 64, [
            (K(32, 8, 1, 8), 1, "smem", 0),
            (K(32, 4, 12, 8), 1, "tmem", N.DD_CONFIG_GPU_TILING | (15 << 8)),
            (K(32, 4, 12, 4), 1, "tmem", N.DD_CONFIG_GPU_TILING | N.DD_CONFIG_HIGH_OCCUPANCY),
            (K(32, 4, 25, 4), 1, "regwin", 0),
            (K(125, 8, 8, 1), 1, "direct", 0),
            (K(160, 1, 5, 8), 2, "smem", N.DD_CONFIG_TIME_MAJOR),
        ]),
        ("LOFAR-like", api.ObservationSetup("lofarish", 20000, 32, 138.0, 0.19, 0.0, 0.25), 32, [
            (K(160, 1, 10, 4), 2, "smem",
             N.DD_CONFIG_PACKED_STAGES | N.DD_CONFIG_TIME_MAJOR | N.DD_CONFIG_GPU_TILING),
            (K(32, 4, 5, 2), 1, "smem", 15 << 8),
        ]),
    ]
    if quick:
        cases[0] = (cases[0][0], cases[0][1], cases[0][2], cases[0][3][:2])
        cases[1] = (cases[1][0], cases[1][1], cases[1][2], cases[1][3][:1])
    # a fault-injected copy of the Apertif table: one DM far below its
    # neighbours in some channels (non-monotone rows -> slow paths)
    jit = api.build_delay_table(api.APERTIF, 64)
    jit.shifts = jit.shifts.copy()
    jit.shifts[9, ::7] = 0
    jit.shifts[40, 100:300] += 37
    jit.max_delay = int(jit.shifts.max())
    cases.append(("Apertif-jittered", api.APERTIF, 64, [
        (K(32, 4, 12, 8), 1, "tmem", N.DD_CONFIG_GPU_TILING),
        (K(32, 4, 25, 4), 1, "regwin", 0),
        (K(32, 8, 1, 8), 1, "smem", 0)], jit))
    for case in cases:
        name, setup, d, cfgs = case[:4]
        table = case[4] if len(case) > 4 else api.build_delay_table(setup, d)
        t = api.instance_sizing(setup, d).num_samples
        s, c = setup.samples_per_second, setup.channels
        fb = api.noise_filterbank(setup, t, 1.0, 1)
        pitch = (t + 3) // 4 * 4
        x = torch.zeros((c, pitch), device="cuda")
        x[:, :t] = torch.from_numpy(fb.data).cuda()
        sh = torch.from_numpy(table.shifts.view(np.int32)).cuda()
        ref = torch.empty((d, s), device="cuda")
        ctx.plan(sh.data_ptr(), c, d, s, t, pitch).execute(x.data_ptr(), ref.data_ptr())
        guard = 2
        buf = torch.full((d + 2 * guard, s), 0.0, device="cuda")
        buf.view(torch.int32).fill_(SENT)
        out = buf[guard:guard + d]
        for cfg, depth, staging, flags in cfgs:
            out.fill_(float("nan"))
            p = ctx.plan(sh.data_ptr(), c, d, s, t, pitch, cfg, depth, staging, flags=flags)
            p.execute(x.data_ptr(), out.data_ptr())
            ctx.synchronize()
            ok = torch.equal(out.view(torch.int32), ref.view(torch.int32))
            gv = buf.view(torch.int32)
            ok = ok and bool((gv[:guard] == SENT).all()) and bool((gv[guard + d:] == SENT).all())
            print(f"{name} d={d} {cfg} depth={depth} {staging} flags={flags:#x} "
                  f"family={p.info()['family']}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
            assert ok
            if not quick and p.info()["family"] in ("smem", "tmem"):
                out.fill_(float("nan"))
                for i, (c0, c1) in enumerate([(0, c // 3), (c // 3, c)]):
                    p.execute_channels(x.data_ptr(), out.data_ptr(), c0, c1, accumulate=i > 0)
                ctx.synchronize()
                assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
            p.close()
    N.check(N.lib().dd_debug_violations(C.byref(nviol), C.byref(checked), 0))
    print(f"bounds violations: {nviol.value}", flush=True)
    assert nviol.value == 0
    print("sanitize_cases: ok", flush=True)


if __name__ == "__main__":
    main()
