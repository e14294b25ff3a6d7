"""Time a list of configs on one instance (device-resident, CUDA events).

    python tools/time_configs.py Apertif 4096 "32,4,25,4,1,regwin" "16,16,10,4,1,smem" ...

Extra fields: "g" requests GPU tiling (tile_time need not divide s),
"cpsN" pins N channels per pipeline stage, "occ" the TMEM three-CTA build,
"nsN" N pipeline stages, "tm" time-major CTA raster, "pk" packed stages,
"wide" twice the cps channels per stage.
--cold flushes L2 before every timed run (dd_plan_time_ex).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1601_05052_b200 import _native as N  # noqa: E402
from paper_1601_05052_b200 import _native as N  # noqa: E402
from paper_1601_05052_b200 import api  # noqa: E402


def main():
    cold = "--cold" in sys.argv
    sys.argv = [a for a in sys.argv if a != "--cold"]
    setup = api.find_builtin(sys.argv[1])
    d = int(sys.argv[2])
    c, s = setup.channels, setup.samples_per_second
    t = api.instance_sizing(setup, d).num_samples
    ctx = api.context(0)
    x = torch.from_numpy(api.noise_filterbank(setup, t, 1.0, 1).data).cuda()
    sh = torch.empty((d, c), dtype=torch.int32, device="cuda")
    out = torch.empty((d, s), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ctx.delay_table(setup, d, sh.data_ptr())
    flop = d * s * c
    for spec in sys.argv[3:]:
        f = spec.split(",")
        cfg = api.KernelConfig(*map(int, f[:4]))
        try:
            extra = f[6:]
            p = ctx.plan(sh.data_ptr(), c, d, s, t, t, cfg, int(f[4]), f[5],
                         gpu_tiling="g" in extra,
                         stage_channels=next((int(x[3:]) for x in extra if x.startswith("cps")), 0),
                         high_occupancy="occ" in extra,
                         flags=(next((int(x[2:]) for x in extra if x.startswith("ns")), 0)
                                << N.DD_CONFIG_NSTAGE_SHIFT)
                         | (N.DD_CONFIG_TIME_MAJOR if "tm" in extra else 0)
                         | (N.DD_CONFIG_PACKED_STAGES if "pk" in extra else 0)
                         | (N.DD_CONFIG_WIDE_STAGES if "wide" in extra else 0))
        except ValueError as e:
            print(f"{spec:28s} invalid: {e}")
            continue
        runs = p.time(x.data_ptr(), out.data_ptr(), warmup=2, repeats=10, flush_l2=cold)
        ms = sorted(runs)[len(runs) // 2] * 1e3
        i = p.info()
        print(f"{spec:28s} {i['family']:7s} {ms:8.4f} ms  {flop / ms / 1e6:9.1f} GFLOP/s  "
              f"smem={i['smem_bytes']} stages={i['stages']}x{i['channels_per_stage']} "
              f"regs={i['registers']} ctas/sm={i['ctas_per_sm']}", flush=True)


if __name__ == "__main__":
    main()
