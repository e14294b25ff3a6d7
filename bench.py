"""Benchmark of the B200 dedispersion hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one dedispersion pass over one 1-s block of the Apertif-like setup
(1024 channels, 20000 samples/s) at 4096 trial DMs -- BASELINE config 2 at
N=1; at N>1 the same instance is DM-sharded across the ranks (config 4,
strong scaling).  ``value`` is whole-job GFLOP/s (d*s*c additions /
max-over-ranks pass time) with inputs resident in HBM; ``e2e`` is the same
metric through the library with host buffers (pinned H2D of the block --
at N>1 each rank ships 1/N of it and NCCL all-gathers the rest over NVLink --
and D2H of every output row inside the timed region).  ``--impl reference``
times the reference's own CPU implementation (oracle/_ref, built from the
unmodified reference sources; the C restatement when that is absent) on all
host cores, full passes of the same instance.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU); under torchrun the
world size must equal N.  The output of the timed pass is fingerprinted once,
outside the timing, against the reference's golden fingerprint
(tests/golden/golden.json): ``parity``.
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
    p.add_argument("--e2e-h2d", default="auto", choices=["auto", "time", "channels", "sharded"])
    p.add_argument("--e2e-single", action="store_true",
                   help="e2e over isolated blocks instead of a double-buffered stream")
    p.add_argument("--plumbing-check", action="store_true",
                   help="CPU/gloo check of the N-rank launcher and C1/C2 plumbing (no GPU)")
    return p.parse_args()




def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp32_add_peak(clocks, sms):
    """The binding on-chip ceiling: FP32 adds per SM clock measured on a B200
    by tools/ubench/fadd.cu (profiles/fadd_ubench.json; the better of scalar
    FADD and paired FADD2), x SMs x the SM clock sampled under load.  Falls
    back to 128 lanes/clk/SM (derived) when the measurement is absent."""
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    per_clk, src = 128.0, "derived: 128 FP32 lanes/clk/SM"
    try:
        with open(os.path.join(ROOT, "profiles", "fadd_ubench.json")) as f:
            u = json.load(f)
        per_clk = max(float(u["fadd_adds_per_clk_sm"]), float(u["fadd2_adds_per_clk_sm"]))
        src = (f"measured: tools/ubench/fadd.cu, {per_clk:.1f} adds/clk/SM "
               f"(profiles/fadd_ubench.json)")
    except Exception:
        pass
    return per_clk * sms * mhz * 1e6 / 1e12, per_clk, mhz, src


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


def golden_fingerprint(setup_name, d):
    """The reference's output fingerprint for (setup, d) with the tuner's
    input (noise sigma 1, seed 1), from tests/golden/golden.json (made by the
    unmodified reference, tests/golden/make_golden.py); None if not there."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            g = json.load(f)
    except Exception:
        return None
    for b in g["baseline"]:
        if b["setup"]["name"] == setup_name and b["num_dms"] == d and b["seed"] == 1:
            return b["out_fnv"]
    return None


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


def workload_name(setup_name, c, s, t, d, n_gpus):
    """The config.workload string both arms print (the same workload)."""
    n = (2 if n_gpus == 1 else 4) if setup_name == "Apertif" else 3
    where = "" if n_gpus == 1 else f", DM-sharded over {n_gpus} GPUs"
    return (f"{setup_name} c={c} s={s} t={t}, {d} trial DMs, 1 s block{where} "
            f"(BASELINE config {n})")


# ------------------------------------------------------- CPU baseline --
class CpuBaseline:
    """The reference's tiled CPU kernel (dedisperse_tiled_into, its
    ThreadPool over all host cores) on the same instance: oracle/_ref (the
    unmodified reference) when built, else the C restatement ("port").
    Full passes over every DM unless a pass would exceed `max_pass_s`, in
    which case a centred DM slice (GFLOP/s is a rate)."""

    def __init__(self, setup_name, d, max_pass_s=8.0):
        import ctypes as C

        import numpy as np

        from oracle import oracle as O
        self.C, self.O, self.np = C, O, np
        setup = O.APERTIF if setup_name == "Apertif" else O.LOFAR
        self.setup = setup
        t, _, _ = O.instance_sizing(setup, d)
        self.sh, _ = O.delay_table(setup, d)
        self.fb = O.noise(setup.channels, t, 1.0, 1)
        self.cfg = (125, 8, 8, 1) if setup_name == "Apertif" else (1000, 1, 1, 4)
        self.d, self.name = d, setup_name
        self.s, self.t, self.c = setup.samples_per_second, t, setup.channels
        self.cores = os.cpu_count() or 1
        self.R = O.ref_lib()
        self.kind = "reference" if self.R is not None else "port"
        self.job = None
        self._use_rows(d)
        first = self.one()  # warm-up, and the size check
        if first > max_pass_s and d > 256:
            rows = max(256, int(d * max_pass_s / first) // 64 * 64)
            self._use_rows(rows)
            self.one()

    def _use_rows(self, rows):
        cfg = self.cfg
        while rows % (cfg[1] * cfg[3]):
            cfg = (cfg[0], 1, cfg[2], 1)
        self.cfg_used = cfg
        self.rows = rows
        self.lo = (self.d - rows) // 2
        self.sub = self.np.ascontiguousarray(self.sh[self.lo:self.lo + rows])
        self.flop = rows * self.s * self.c
        if self.R is not None:
            if self.job is not None:
                self.R.ref_job_destroy(self.job)
            C = self.C
            self.job = self.R.ref_job_create(
                C.byref(self.setup.c()), self.fb.ctypes.data_as(C.POINTER(C.c_float)), self.t,
                self.sub.ctypes.data_as(C.POINTER(C.c_uint32)), rows, self.cores)
            self.cores = self.R.ref_job_threads(self.job)

    def one(self):
        t0 = time.perf_counter()
        if self.R is not None:
            assert self.R.ref_job_run_tiled(self.job,
                                            self.C.byref(self.O.ConfigC(*self.cfg_used))) == 0
        else:
            self.O.dedisperse_tiled(self.fb, self.sub, self.s, self.cfg_used, self.cores)
        return time.perf_counter() - t0

    def describe(self, runs):
        mean = sum(runs) / len(runs)
        whole = self.rows == self.d
        what = (f"{self.name} d={self.d}: the full pass (all {self.d} DMs)" if whole else
                f"{self.name} d={self.d}: DM rows [{self.lo},{self.lo + self.rows}) of the full "
                f"table")
        return {"value": round(self.flop / mean / 1e9, 3), "unit": "GFLOP/s",
                "cores": self.cores, "kind": self.kind,
                "sample": f"{what}, dedisperse_tiled{self.cfg_used} on a {self.cores}-thread "
                          f"ThreadPool, {len(runs)} passes, mean {mean:.3f} s/pass",
                "full_pass": whole,
                "realtime_factor": round(1.0 / (mean * self.d / self.rows), 4)}

    def measure(self, seconds):
        runs = []
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end or len(runs) < 2:
            runs.append(self.one())
        return self.describe(runs)

    def oracle_config(self):
        """BASELINE config 1: Apertif d=64, the reference's single-thread
        dedisperse_reference_into (kernels.cpp:83-108), one pass."""
        O, C, np = self.O, self.C, self.np
        if self.R is None:
            return None
        setup = O.APERTIF
        t, _, _ = O.instance_sizing(setup, 64)
        sh, _ = O.delay_table(setup, 64)
        fb = O.noise(setup.channels, t, 1.0, 1)
        job = self.R.ref_job_create(C.byref(setup.c()), fb.ctypes.data_as(C.POINTER(C.c_float)),
                                    t, np.ascontiguousarray(sh).ctypes.data_as(
                                        C.POINTER(C.c_uint32)), 64, 1)
        t0 = time.perf_counter()
        assert self.R.ref_job_run_reference(job) == 0
        sec = time.perf_counter() - t0
        self.R.ref_job_destroy(job)
        flop = 64 * setup.samples_per_second * setup.channels
        return {"workload": "Apertif c=1024 s=20000 t=40000, 64 trial DMs (BASELINE config 1)",
                "path": "reference dedisperse_reference_into, 1 thread", "seconds": round(sec, 3),
                "value": round(flop / sec / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                "realtime_factor": round(1.0 / sec, 4)}


def cpu_baseline(setup_name, d, seconds):
    return CpuBaseline(setup_name, d).measure(seconds)


def run_reference(args):
    """The reference arm: the reference's own dedisperse_tiled_into on the
    host cores, full passes of the same instance (rank 0 only under
    torchrun; the other ranks exit without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    base = CpuBaseline(args.setup, args.dms)
    for _ in range(max(0, args.warmup - 1)):
        base.one()
    runs = [base.one() for _ in range(max(1, args.steps))]
    desc = base.describe(runs)
    v = desc["value"]
    d, s, c = args.dms, base.s, base.c
    line = {"metric": METRIC, "value": v, "unit": "GFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.mean(runs) * base.d / base.rows * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: noise_filterbank(sigma=1, seed=1), the reference's build_delay_table",
            "config": {"workload": workload_name(args.setup, c, s, base.t, d, args.gpus),
                       "path": "host CPU, the reference's dedisperse_tiled_into on its ThreadPool "
                               "(oracle/_ref built from /root/reference/proj/core/src)"},
            "cpu_baseline": desc,
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if args.setup == "Apertif" and not args.no_cpu:
        try:
            line["oracle_config"] = base.oracle_config()
        except Exception as ex:
            line["oracle_config"] = {"error": str(ex)[:200]}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ launcher --
def spawn(args):
    """--gpus N outside torchrun: re-launch this script with N ranks (one per
    GPU) under torch.distributed.run, rendezvous on 127.0.0.1."""
    import socket
    if not args.plumbing_check:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s)\n")
            return 2
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plumbing_check(args):
    """The N-rank path without a GPU (gloo): world size, DM shards, the
    sharded channel-group upload + all-gather (C1) and the row gather (C2)
    assembled exactly; rank 0 prints one JSON line."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1601_05052_b200 import multi
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world_size > 1:
        dist.init_process_group("gloo")
    c, t, d, s, align = 16, 96, 48, 40, 4
    rng = np.random.default_rng(7)
    host = torch.from_numpy(rng.standard_normal((c, t)).astype(np.float32))
    shifts = rng.integers(0, t - s, size=(d, c)).astype(np.int64)
    block = torch.full((c, t), float("nan"))
    groups = multi.channel_groups(c, world_size, 4)
    for c0, c1 in groups:
        p0, p1 = multi.rank_part(c0, c1, world_size, rank)
        block[p0:p1] = host[p0:p1]  # this rank's upload
        multi.allgather_channels(block, c0, c1)
    assembled = bool(torch.equal(block, host))
    off, cnt = multi.shard_range(d, world_size, rank, align)
    rows = np.arange(off, off + cnt)
    idx = np.arange(s)[None, :]
    local = torch.from_numpy(np.stack([
        sum(host.numpy()[ch, idx[0] + shifts[r, ch]].astype(np.float64) for ch in range(c))
        for r in rows]).astype(np.float32)) if cnt else torch.empty((0, s))
    full = multi.gather_rows(local, d, align)
    if rank == 0:
        ref = np.stack([sum(host.numpy()[ch, idx[0] + shifts[r, ch]].astype(np.float64)
                            for ch in range(c)) for r in range(d)]).astype(np.float32)
        print(json.dumps({"plumbing": "ok" if assembled and np.array_equal(full.numpy(), ref)
                          else "mismatch", "n_gpus": args.gpus, "world_size": world_size,
                          "channel_groups": groups, "block_assembled": assembled,
                          "rows_gathered": int(full.shape[0])}), flush=True)
    if world_size > 1:
        dist.barrier()
        dist.destroy_process_group()
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

    # every rank holds the block in pinned host memory (each ships its own
    # share in the e2e path); the tuner's input
    fb = api.noise_filterbank(setup, t, 1.0, 1)
    host = torch.from_numpy(fb.data).pin_memory()
    dd.load(host)
    torch.cuda.synchronize()

    flush = torch.empty(args.flush_mb << 18, dtype=torch.float32, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float32, device="cuda")
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
            # evict L2 (write a buffer twice its size), then read the buffer
            # back so the lines left are clean: the timed pass must not pay
            # the write-back of the flush
            flush.zero_()
            flush_sink.copy_(flush.sum())
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

    # parity: the whole output of the timed pass (all ranks' rows) against
    # the reference's fingerprint -- once, outside the timing
    dd.run()
    torch.cuda.synchronize()
    full = dd.gather()
    parity = None
    golden = golden_fingerprint(setup.name, d)
    if rank == 0:
        got = api.fingerprint(full.cpu())
        parity = {"status": "unpinned" if golden is None else
                  ("bit-exact" if got == golden else "MISMATCH"),
                  "fingerprint": got, "golden": golden,
                  "what": "FNV-1a 64 of the whole [d][s] output of the timed configuration vs "
                          "the unmodified reference's (tests/golden/golden.json)"}
    del full

    # end to end through the library with host buffers
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
        # operating mode): block i+1's input route and kernels overlap block
        # i's D2H, double-buffered
        streamed = not args.e2e_single
        n_stream = max(4, args.steps)
        h_outs = [h_out, torch.empty_like(h_out).pin_memory()]
        if streamed:
            dd.stream_host([host], h_outs, 2)  # warm-up
            torch.cuda.synchronize()
            if world_size > 1:
                dist.barrier()
            t0 = time.perf_counter()
            dd.stream_host([host], h_outs, n_stream)
            torch.cuda.synchronize()
            e2e_ms_v = (time.perf_counter() - t0) * 1e3 / n_stream
        else:
            e2e_ms_v = single_ms
        e = torch.tensor([e2e_ms_v, single_ms], device="cuda")
        h2d = torch.tensor([dd.h2d_bytes(), dd.d2h_bytes()], dtype=torch.float64, device="cuda")
        if world_size > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
            dist.all_reduce(h2d, op=dist.ReduceOp.SUM)
        e2e_ms_v, single_ms = (float(x) for x in e.tolist())
        h2d_bytes, d2h_bytes = (int(x) for x in h2d.tolist())
        # the last streamed block's output, read back into host memory, is
        # the reference's too
        last = h_outs[(n_stream - 1) % 2] if streamed else h_out
        full_host = dd_gather_host(dd, last, multi)
        e2e_parity = None
        if rank == 0:
            got = api.fingerprint(full_host)
            e2e_parity = "unpinned" if golden is None else \
                ("bit-exact" if got == golden else "MISMATCH")
        routes = {
            "time": "pinned H2D of the [c][t] block in time order (2-D copies, "
                    "dd_upload_block_range; samples past the last DM chunk's reach are not "
                    "shipped), each DM chunk's kernel starting once the samples its delays "
                    "reach have landed, and D2H of each chunk's rows overlapped with the "
                    "remaining uploads and kernels",
            "sharded": "each rank ships its 1/N share of every channel group H2D over its own "
                       "PCIe link, one NCCL all-gather per group assembles the group on every "
                       "GPU (C1), the group's kernels accumulate through the output (bit-exact) "
                       "as soon as it is complete, and each rank's DM chunks go D2H as soon as "
                       "they are final",
            "broadcast": "rank 0 ships the block H2D and NCCL broadcasts it; kernels and D2H "
                         "as in the sharded route",
            "channels": "pinned H2D by channel groups, the kernels of the groups already "
                        "landed accumulating through the output (bit-exact), D2H of each DM "
                        "chunk's rows overlapped with the remaining kernels"}
        e2e = {"value": round(flop_total / (e2e_ms_v * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
               "ms_per_step": round(e2e_ms_v, 3),
               "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
               "bytes": "whole job (sum over ranks), counted from the copies issued",
               "dm_chunks": len(dd.chunks), "channel_groups": len(dd.groups),
               "h2d_route": dd.h2d_mode,
               "mode": (f"streamed: {n_stream} consecutive blocks through "
                        "ShardedDedisperser.stream_host, double-buffered so block i+1's input "
                        "route and kernels overlap block i's D2H; ms_per_step = host wall time "
                        "of the whole stream / blocks, max over ranks" if streamed else
                        "single block per step, synchronised at the end"),
               "single_block_ms": round(single_ms, 3),
               "single_block_value": round(flop_total / (single_ms * 1e-3) / 1e9, 2),
               "parity": e2e_parity,
               "path": routes[dd.h2d_mode] + "; host-timed"}

    cpu = None
    if rank == 0 and world_size == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(setup.name, d, args.cpu_seconds)
        except Exception as ex:  # the baseline must never break the line
            cpu = {"value": None, "error": str(ex)[:200]}

    if rank == 0:
        hbm, src = peaks()
        cs = clk.summary()
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        peak_t, per_clk, mhz, peak_src = fp32_add_peak(cs, sms)
        launch_flop = dd.count * s * c  # rank 0's launch
        achieved_t = launch_flop / (ms_local * 1e-3) / 1e12
        alg_launch = api.algorithmic_bytes(dd.count, s, c)
        traffic, compulsory = None, None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                tr = json.load(f)
            key = f"{setup.name}_{d}_" + "_".join(str(x) for x in cfgt)
            ent = tr.get(key)
            if isinstance(ent, dict):
                traffic = ent.get("dram_bytes_per_launch")
                compulsory = ent.get("compulsory_bytes")
            elif ent is not None:
                traffic = ent
        roofline = {
            "bound": "fp32_add", "achieved": round(achieved_t, 3), "peak": round(peak_t, 3),
            "unit": "TFLOP/s", "frac": round(achieved_t / peak_t, 4), "traffic": traffic,
            "peak_source": peak_src,
            "definition": "achieved = d*s*c fp32 additions per launch (one per output and "
                          "channel, the bit-exact sum's minimum) / CUDA-event launch time; peak "
                          "= measured FP32 adds/clk/SM x SMs x SM clock under load",
            "hbm_noreuse_multiple": round(alg_launch / (ms_local * 1e-3) / 1e9 / hbm, 3),
            "hbm_peak_gbs": hbm, "hbm_peak_source": src,
        }
        if traffic:
            roofline["dram_frac"] = round(traffic / (ms_local * 1e-3) / 1e9 / hbm, 4)
            if compulsory:
                roofline["dram_vs_compulsory"] = round(traffic / compulsory, 3)
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
                                  "flags": cfgt[6],
                                  "stage_channels": info["channels_per_stage"],
                                  "gpu_tiling": bool(flags & 1),
                                  "source": os.path.relpath(cfg_src, ROOT)
                                  if cfg_src and cfg_src != "cli" else (cfg_src or "default")},
                "kernel_family": info["family"], "smem_bytes": info["smem_bytes"],
                "grid": info["grid_x"], "block": info["block_threads"],
                "stages": info["stages"], "registers": info["registers"],
                "cta_raster": "time-major" if info["time_major"] else "dm-major",
                "parallelism": f"dm-shard x{world_size}",
                "l2": f"flushed between timed steps ({args.flush_mb} MB memset + read-back, outside "
                      "the events: the pass starts with clean, evicted L2)",
            },
            "parity": parity,
            "hbm_gbs_effective": round(api.algorithmic_bytes(d, s, c) / (ms * 1e-3) / 1e9, 1),
            "realtime_factor": round(1.0 / (ms * 1e-3), 2),
            "roofline": roofline,
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


def dd_gather_host(dd, host_rows, multi):
    """Every rank's host output rows assembled on rank 0 (through the device
    for NCCL), for the e2e parity check; the host tensor itself at N=1."""
    import torch
    if dd.world == 1:
        return host_rows
    dev = host_rows.to(dd.device)
    full = multi.gather_rows(dev, dd.num_dms, dd.cfg.tile_dm())
    return None if full is None else full.cpu()


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return spawn(args)
    if args.plumbing_check:
        return plumbing_check(args)
    if ws is not None and int(ws) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}\n")
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
