"""Benchmark of the B200 dedispersion hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one dedispersion pass over one 1-s block of the Apertif-like setup
(1024 channels, 20000 samples/s) at 4096 trial DMs -- BASELINE config 2 at
N=1; at N>1 the same instance is DM-sharded across the ranks (config 4,
strong scaling, one NCCL broadcast of the input block before timing).
``value`` is whole-job GFLOP/s (d*s*c additions / max-over-ranks pass
time) with inputs resident in HBM; ``e2e`` is the same metric through the
C-ABI with host buffers (pinned H2D of the block + D2H of the output inside
the timed region).  ``--impl reference`` times the reference's own CPU
implementation (oracle/_ref, built from the unmodified reference sources; the
C restatement when that is absent) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dedispersion GFLOP/s + HBM GB/s (Apertif/LOFAR, 2-4096 DMs) at 1/2/4/8 B200"
DEFAULT_CFG = (16, 8, 10, 4, 1, "smem", 8 << 8)  # overridden by tuning/<setup>_<d>.json
REASON_FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--setup", default="Apertif")
    p.add_argument("--dms", type=int, default=4096)
    p.add_argument("--config", default=None,
                   help="items_time,items_dm,work_time,work_dm,depth,staging[,flags]")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--flush-mb", type=int, default=256)
    p.add_argument("--e2e-chunks", type=int, default=8)
    p.add_argument("--e2e-channel-groups", type=int, default=2)
    p.add_argument("--e2e-h2d", default="auto", choices=["auto", "time", "channels"])
    p.add_argument("--e2e-single", action="store_true",
                   help="e2e over isolated blocks instead of a double-buffered stream")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def onchip_ceilings(gflops, clocks):
    """The on-chip ceilings the staged kernels are judged against (DESIGN.md
    §3): one fp32 add per (output, channel) at 128 FP32 lanes/clk/SM, and one
    4-byte shared-memory operand per add at 128 B/clk/SM, at the SM clock
    sampled under load (max clock if no sample)."""
    import torch
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    fp32 = sms * 128 * mhz * 1e6 / 1e9
    lds = sms * 32 * mhz * 1e6 / 1e9
    return {"sm_count": sms, "sm_mhz": mhz,
            "fp32_add_gflops": round(fp32, 1), "frac_fp32_add": round(gflops / fp32, 4),
            "smem_operand_gflops": round(lds, 1), "frac_smem_operand": round(gflops / lds, 4)}


def tuned_config(setup_name, d):
    from paper_1601_05052_b200 import api
    path = os.path.join(ROOT, "tuning", f"{setup_name.lower()}_{d}.json")
    if os.path.exists(path):
        with open(path) as f:
            b = api.tuning_result_from_json(f.read()).best()
        k = b.config
        return (k.items_time, k.items_dm, k.work_time, k.work_dm, b.dm_tile_depth, b.staging,
                b.flags), path
    return DEFAULT_CFG, None


# ------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw," +
             ",".join("clocks_event_reasons." + r for r in REASON_FIELDS))
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            for name, v in zip(REASON_FIELDS, r[3:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def workload_name(setup_name, c, s, t, d, world_size):
    """The config.workload string both arms print (the same workload)."""
    n = (2 if world_size == 1 else 4) if setup_name == "Apertif" else 3
    return f"{setup_name} c={c} s={s} t={t}, {d} trial DMs, 1 s block (BASELINE config {n})"


# ------------------------------------------------------- CPU baseline --
class CpuBaseline:
    """The reference's tiled CPU kernel (ThreadPool over all host cores) on a
    bounded DM sample of the same instance: oracle/_ref (the unmodified
    reference) when built, else the C restatement ("port")."""

    def __init__(self, setup_name, d):
        import ctypes as C

        import numpy as np

        from oracle import oracle as O
        self.C, self.O = C, O
        setup = O.APERTIF if setup_name == "Apertif" else O.LOFAR
        t, _, _ = O.instance_sizing(setup, d)
        sh, _ = O.delay_table(setup, d)
        self.fb = O.noise(setup.channels, t, 1.0, 1)
        rows = min(d, 256 if setup_name == "Apertif" else 128)
        self.lo = (d - rows) // 2
        self.sub = np.ascontiguousarray(sh[self.lo:self.lo + rows])
        cfg = (125, 8, 8, 1) if setup_name == "Apertif" else (1000, 1, 1, 4)
        while rows % (cfg[1] * cfg[3]):
            cfg = (cfg[0], 1, cfg[2], 1)
        self.cfg, self.rows, self.d, self.name = cfg, rows, d, setup_name
        self.s, self.t, self.c = setup.samples_per_second, t, setup.channels
        self.flop = rows * self.s * setup.channels
        self.cores = os.cpu_count() or 1
        self.R = O.ref_lib()
        self.kind = "reference" if self.R is not None else "port"
        if self.R is not None:
            self.job = self.R.ref_job_create(C.byref(setup.c()),
                                             self.fb.ctypes.data_as(C.POINTER(C.c_float)), t,
                                             self.sub.ctypes.data_as(C.POINTER(C.c_uint32)), rows,
                                             self.cores)
            self.cores = self.R.ref_job_threads(self.job)
        self.one()  # warm-up

    def one(self):
        t0 = time.perf_counter()
        if self.R is not None:
            assert self.R.ref_job_run_tiled(self.job, self.C.byref(self.O.ConfigC(*self.cfg))) == 0
        else:
            self.O.dedisperse_tiled(self.fb, self.sub, self.s, self.cfg, self.cores)
        return time.perf_counter() - t0

    def measure(self, seconds):
        runs = []
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end or len(runs) < 2:
            runs.append(self.one())
        mean = sum(runs) / len(runs)
        return {"value": round(self.flop / mean / 1e9, 3), "unit": "GFLOP/s",
                "cores": self.cores, "kind": self.kind,
                "sample": f"{self.name} d={self.d}: DM rows [{self.lo},{self.lo + self.rows}) of "
                          f"the full table, dedisperse_tiled{self.cfg}, {len(runs)} passes, "
                          f"mean {mean:.3f} s/pass",
                "realtime_factor": round(1.0 / (mean * self.d / self.rows), 4)}


def cpu_baseline(setup_name, d, seconds):
    return CpuBaseline(setup_name, d).measure(seconds)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    base = CpuBaseline(args.setup, args.dms)
    for _ in range(max(0, args.warmup - 1)):
        base.one()
    # each step is one bounded sample of the workload (a DM subset pass)
    per = max(0.0, min(6.0, 150.0 / max(1, args.steps)))
    samples = [base.measure(per) for _ in range(max(1, args.steps))]
    v = statistics.mean(x["value"] for x in samples)
    d = args.dms
    s = 20000 if args.setup == "Apertif" else 200000
    c = 1024 if args.setup == "Apertif" else 32
    line = {"metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(d * s * c / (v * 1e9) * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(args.setup, base.c, base.s, base.t, d, args.gpus),
                       "path": "host CPU, reference dedisperse_tiled on a bounded DM sample"},
            "cpu_baseline": dict(samples[-1], value=round(v, 3)),
            "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- ours --
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1601_05052_b200 import api, multi

    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world_size > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    setup = api.find_builtin(args.setup)
    d = args.dms
    if args.config:
        f = args.config.split(",")
        cfgt, cfg_src = (int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), f[5],
                         int(f[6], 0) if len(f) > 6 else 0), "cli"
    else:
        cfgt, cfg_src = tuned_config(setup.name, d)
    cfg = api.KernelConfig(*cfgt[:4])
    flags = cfgt[6]
    dd = multi.ShardedDedisperser(setup, d, cfg, cfgt[4], cfgt[5], device=local, flags=flags)
    c, s, t = setup.channels, setup.samples_per_second, dd.num_samples
    stream = dd.stream
    torch.cuda.set_stream(stream)  # events, flushes and copies share the library's stream

    host = None
    if rank == 0:
        fb = api.noise_filterbank(setup, t, 1.0, 1)  # the reference tuner's input
        host = torch.from_numpy(fb.data).pin_memory()
    dd.load(host)
    torch.cuda.synchronize()

    flush = torch.empty(args.flush_mb << 18, dtype=torch.float32, device="cuda")
    info = dd.plan.info()
    for _ in range(max(3, args.warmup)):
        dd.run()
    torch.cuda.synchronize()
    if world_size > 1:
        dist.barrier()

    # timed region: per-step CUDA events around the single kernel launch, an
    # L2 flush (memset of a buffer larger than L2) between steps, outside them
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            dd.run()
            stops[i].record(stream)
        torch.cuda.synchronize()
        # keep the GPU busy so the sampler sees load for a few hundred ms
        t_end = time.time() + 0.6
        while time.time() < t_end:
            for _ in range(8):
                dd.run()
            torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    ms_local = statistics.mean(times)
    ms = torch.tensor([ms_local], device="cuda")
    if world_size > 1:
        dist.barrier()
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    flop_total = d * s * c
    value = flop_total / (ms * 1e-3) / 1e9

    # end to end through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        h_out = torch.empty((dd.count, s), dtype=torch.float32).pin_memory()
        dd.pipeline(args.e2e_chunks, args.e2e_channel_groups, args.e2e_h2d)
        e2e_ms = []
        for i in range(max(2, args.steps // 3) + 1):
            if world_size > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dd.run_host(host, h_out)
            torch.cuda.synchronize()
            if i > 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        single_ms = statistics.mean(e2e_ms)
        # steady state of a stream of consecutive blocks (a survey's real
        # operating mode): block i+1's H2D and kernels overlap block i's D2H,
        # double-buffered; every block is copied in and read back in full
        streamed = world_size == 1 and dd.h2d_mode == "time" and not args.e2e_single
        if streamed:
            h_outs = [h_out, torch.empty_like(h_out).pin_memory()]
            n_stream = max(4, args.steps)
            dd.stream_host([host], h_outs, 2)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dd.stream_host([host], h_outs, n_stream)
            torch.cuda.synchronize()
            e2e_ms_v = (time.perf_counter() - t0) * 1e3 / n_stream
        else:
            e2e_ms_v = single_ms
        e = torch.tensor([e2e_ms_v], device="cuda")
        if world_size > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        e2e_ms_v = float(e.item())
        per_block = ("pinned H2D of the [c][t] block in time order (2-D copies, "
                     "dd_upload_block_range), each DM chunk's kernel starting once the "
                     "samples its delays reach have landed, and D2H of each chunk's rows "
                     "overlapped with the remaining uploads and kernels"
                     if dd.h2d_mode == "time" else
                     "pinned H2D of the [c][t] block by channel groups overlapped with the "
                     "kernels of the groups already landed (accumulating through the output, "
                     "bit-exact; with N>1: H2D on rank 0 + NCCL broadcast), and D2H of each "
                     "DM chunk's rows overlapped with the remaining kernels")
        e2e = {"value": round(flop_total / (e2e_ms_v * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
               "ms_per_step": round(e2e_ms_v, 3),
               "h2d_bytes_per_step": c * t * 4 if rank == 0 else 0,
               "d2h_bytes_per_step": d * s * 4,
               "dm_chunks": len(dd.chunks), "channel_groups": len(dd.groups),
               "h2d_order": dd.h2d_mode,
               "mode": (f"streamed: {n_stream} consecutive blocks through "
                        "ShardedDedisperser.stream_host, double-buffered so block i+1's H2D "
                        "and kernels overlap block i's D2H; ms_per_step = host wall time of "
                        "the whole stream / blocks" if streamed else
                        "single block per step, synchronised at the end"),
               "single_block_ms": round(single_ms, 3),
               "single_block_value": round(flop_total / (single_ms * 1e-3) / 1e9, 2),
               "path": per_block + "; host-timed"}

    cpu = None
    if rank == 0 and world_size == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(setup.name, d, args.cpu_seconds)
        except Exception as ex:  # the baseline must never break the line
            cpu = {"value": None, "error": str(ex)[:200]}

    if rank == 0:
        hbm, src = peaks()
        alg_bytes = api.algorithmic_bytes(d, s, c)
        per_launch = api.algorithmic_bytes(dd.count, s, c)  # rank 0's launch
        achieved = per_launch / (ms_local * 1e-3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f)
            key = f"{setup.name}_{d}_" + "_".join(str(x) for x in cfgt)
            ent = tr.get(key)
            traffic = ent.get("dram_bytes_per_launch") if isinstance(ent, dict) else ent
        cs = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: noise_filterbank(sigma=1, seed=1) (the reference tuner's input), "
                    "device-built shift table",
            "config": {
                "workload": workload_name(setup.name, c, s, t, d, world_size),
                "kernel_config": {"items_time": cfgt[0], "items_dm": cfgt[1],
                                  "work_time": cfgt[2], "work_dm": cfgt[3],
                                  "dm_tile_depth": cfgt[4], "staging": cfgt[5],
                                  "stage_channels": info["channels_per_stage"],
                                  "gpu_tiling": bool(flags & 1),
                                  "source": os.path.relpath(cfg_src, ROOT)
                                  if cfg_src and cfg_src != "cli" else (cfg_src or "default")},
                "kernel_family": info["family"], "smem_bytes": info["smem_bytes"],
                "grid": info["grid_x"], "block": info["block_threads"],
                "stages": info["stages"], "registers": info["registers"],
                "cta_raster": "time-major" if info["time_major"] else "dm-major",
                "parallelism": f"dm-shard x{world_size}",
                "l2": f"flushed between timed steps ({args.flush_mb} MB memset outside the events)",
            },
            "hbm_gbs_effective": round(alg_bytes / (ms * 1e-3) / 1e9, 1),
            "realtime_factor": round(1.0 / (ms * 1e-3), 2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                         "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "peak_source": src,
                         "definition": "achieved = 4*(d*s*c + d*s + d*c) no-reuse bytes (Eq. 2) "
                                       "per launch / CUDA-event launch time"},
            "onchip_ceilings": onchip_ceilings(value, cs),
            "gpu_launches": args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": cs,
        }
        print(json.dumps(line), flush=True)
    if world_size > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
