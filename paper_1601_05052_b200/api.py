"""Python mirror of the reference's `dedisp` C++ API, over the C-ABI.

Same names, argument meaning and error behaviour as the reference's
proj/core headers (setup.hpp, filterbank.hpp, kernels.hpp, tuner.hpp,
analysis.hpp): ``std::invalid_argument`` surfaces as ``ValueError``,
``capacity_error`` as ``CapacityError``, device failures as ``DeviceError``.
Host-side value types hold numpy arrays with the reference layouts
(filterbank float32 [channels][t], table uint32 [d][channels], output
float32 [d][s]).  Every computation on the hot path runs in the CUDA library;
nothing here falls back to the CPU.

Device-resident workflows (the bench, the multi-GPU driver) use
:class:`Context` and :class:`Plan` with raw device pointers (e.g. from
``torch.Tensor.data_ptr()``).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import CapacityError, DeviceError, check, lib  # noqa: F401


# ----------------------------------------------------------------- setup --
@dataclass(frozen=True)
class ObservationSetup:
    """reference setup.hpp:14-33"""

    name: str
    samples_per_second: int
    channels: int
    f_min: float
    channel_width: float
    dm_first: float
    dm_step: float

    def channel_frequency(self, ch: int) -> float:
        return self.f_min + float(ch) * self.channel_width

    def highest_frequency(self) -> float:
        return self.channel_frequency(self.channels - 1)

    def trial_dm(self, i: int) -> float:
        return self.dm_first + float(i) * self.dm_step

    def c(self) -> N.dd_setup:
        return N.dd_setup(self.samples_per_second, self.channels, self.f_min,
                          self.channel_width, self.dm_first, self.dm_step)

    def validate(self) -> None:
        check(lib().dd_setup_validate(C.byref(self.c())))


APERTIF = ObservationSetup("Apertif", 20000, 1024, 1420.0, 0.29, 0.0, 0.25)
LOFAR = ObservationSetup("LOFAR", 200000, 32, 138.0, 0.19, 0.0, 0.25)
DEFAULT_TABLE_CAP = 1 << 30


def builtin_setups() -> List[ObservationSetup]:
    """reference setup.cpp:139-147"""
    return [APERTIF, LOFAR]


def find_builtin(name: str) -> Optional[ObservationSetup]:
    for s in builtin_setups():
        if s.name == name:
            return s
    return None


@dataclass
class DelayTable:
    """reference setup.hpp:39-51 (shifts: uint32 [num_dms][channels])."""

    setup: ObservationSetup
    num_dms: int
    shifts: np.ndarray
    max_delay: int

    def at(self, channel: int, dm: int) -> int:
        return int(self.shifts[dm, channel])


@dataclass
class ProblemInstance:
    setup: ObservationSetup
    num_dms: int
    num_samples: int
    flop: int
    max_delay: int


def delay_seconds(dm: float, f_channel_mhz: float, f_highest_mhz: float) -> float:
    out = C.c_double()
    check(lib().dd_delay_seconds(dm, f_channel_mhz, f_highest_mhz, C.byref(out)))
    return out.value


def instance_sizing(setup: ObservationSetup, num_dms: int) -> ProblemInstance:
    t, f, m = C.c_uint64(), C.c_uint64(), C.c_uint32()
    check(lib().dd_instance_sizing(C.byref(setup.c()), num_dms, C.byref(t), C.byref(f),
                                   C.byref(m)))
    return ProblemInstance(setup, num_dms, t.value, f.value, m.value)


def _table(setup, num_dms, cap, zero, device):
    if num_dms < 1:
        raise ValueError("num_dms must be >= 1")
    setup.validate()
    if num_dms * setup.channels * 4 > cap:
        raise CapacityError(f"delay table of {num_dms * setup.channels * 4} bytes exceeds the "
                            f"cap of {cap}")
    sh = np.empty((num_dms, setup.channels), np.uint32)
    md = C.c_uint32()
    check(lib().dd_build_delay_table(context(device).handle, C.byref(setup.c()), num_dms, cap,
                                     int(zero), sh.ctypes.data, C.byref(md)))
    return DelayTable(setup, num_dms, sh, md.value)


def build_delay_table(setup: ObservationSetup, num_dms: int, memory_cap_bytes: int = DEFAULT_TABLE_CAP,
                      device: int = 0) -> DelayTable:
    """reference setup.cpp:86-105, computed on the device (K1)."""
    return _table(setup, num_dms, memory_cap_bytes, False, device)


def build_zero_delay_table(setup: ObservationSetup, num_dms: int,
                           memory_cap_bytes: int = DEFAULT_TABLE_CAP, device: int = 0) -> DelayTable:
    """reference setup.cpp:107-110"""
    return _table(setup, num_dms, memory_cap_bytes, True, device)


# ------------------------------------------------------------ filterbank --
@dataclass
class Filterbank:
    """reference filterbank.hpp:15-26 (data: float32 [channels][num_samples])."""

    setup: ObservationSetup
    num_samples: int
    data: np.ndarray

    def at(self, channel: int, sample: int) -> float:
        return float(self.data[channel, sample])


def noise_filterbank(setup: ObservationSetup, num_samples: int, sigma: float, seed: int,
                     threads: int = 0) -> Filterbank:
    """reference filterbank.cpp:60-80 (mt19937_64 + Box-Muller, bit-identical)."""
    setup.validate()
    out = np.empty((setup.channels, num_samples), np.float32)
    check(lib().dd_noise_filterbank(setup.channels, num_samples, sigma, seed, threads,
                                    out.ctypes.data))
    return Filterbank(setup, num_samples, out)


# --------------------------------------------------------------- kernels --
@dataclass(frozen=True, order=True)
class KernelConfig:
    """reference kernels.hpp:40-52"""

    items_time: int = 1
    items_dm: int = 1
    work_time: int = 1
    work_dm: int = 1

    def tile_time(self) -> int:
        return self.items_time * self.work_time

    def tile_dm(self) -> int:
        return self.items_dm * self.work_dm

    def block_items(self) -> int:
        return self.items_time * self.items_dm

    def accumulators(self) -> int:
        return self.work_time * self.work_dm


@dataclass(frozen=True)
class KernelLimits:
    """reference kernels.hpp:31-34"""

    max_block_items: int = 1024
    max_accumulators: int = 256

    def c(self) -> N.dd_limits:
        return N.dd_limits(self.max_block_items, self.max_accumulators)


@dataclass
class KernelStats:
    """reference kernels.hpp:56-64"""

    flop_additions: int = 0
    staged_loads: int = 0

    def reset(self) -> None:
        self.flop_additions = 0
        self.staged_loads = 0


@dataclass
class ExecOptions:
    """reference kernels.hpp:66-71 plus the GPU knobs (threads is ignored)."""

    threads: int = 0
    limits: KernelLimits = field(default_factory=KernelLimits)
    stats: Optional[KernelStats] = None
    device: int = 0
    dm_tile_depth: int = 1
    staging: str = "auto"


@dataclass
class DedispersedSeries:
    """reference kernels.hpp:16-27 (data: float32 [num_dms][samples_per_second])."""

    num_dms: int = 0
    samples_per_second: int = 0
    data: np.ndarray = field(default_factory=lambda: np.empty((0, 0), np.float32))

    def at(self, dm: int, sample: int) -> float:
        return float(self.data[dm, sample])


@dataclass(frozen=True)
class LoadCounts:
    staged_loads: int
    ideal_loads: int


def _cfg(cfg: KernelConfig, depth: int = 1, staging: str = "auto",
         gpu_tiling: bool = False, stage_channels: int = 0,
         high_occupancy: bool = False) -> N.dd_config:
    flags = ((N.DD_CONFIG_GPU_TILING if gpu_tiling else 0)
             | (N.DD_CONFIG_HIGH_OCCUPANCY if high_occupancy else 0)
             | (stage_channels << N.DD_CONFIG_CPS_SHIFT))
    return N.dd_config(cfg.items_time, cfg.items_dm, cfg.work_time, cfg.work_dm, depth,
                       N.STAGING[staging], flags)


def config_valid(cfg: KernelConfig, num_dms: int, samples_per_second: int,
                 limits: KernelLimits = KernelLimits()) -> bool:
    return bool(lib().dd_config_valid(C.byref(_cfg(cfg)), num_dms, samples_per_second,
                                      C.byref(limits.c())))


def validate_config(cfg: KernelConfig, num_dms: int, samples_per_second: int,
                    limits: KernelLimits = KernelLimits()) -> None:
    check(lib().dd_validate_config(C.byref(_cfg(cfg)), num_dms, samples_per_second,
                                   C.byref(limits.c())))


def _check_pair(fb: Filterbank, table: DelayTable) -> None:
    """reference kernels.cpp:16-28"""
    if (fb.setup.channels != table.setup.channels
            or fb.setup.samples_per_second != table.setup.samples_per_second):
        raise ValueError("filterbank and delay table describe different setups")
    if table.num_dms == 0:
        raise ValueError("delay table holds no trials")
    need = fb.setup.samples_per_second + table.max_delay
    if fb.num_samples < need:
        raise ValueError(f"filterbank too short: need {need} samples per channel, have "
                         f"{fb.num_samples}")


def _run(out: DedispersedSeries, fb: Filterbank, table: DelayTable, cfg, limits, device) -> None:
    _check_pair(fb, table)
    d, s = table.num_dms, fb.setup.samples_per_second
    data = np.ascontiguousarray(fb.data, np.float32)
    shifts = np.ascontiguousarray(table.shifts, np.uint32)
    if out.data.shape != (d, s) or out.data.dtype != np.float32 or not out.data.flags.c_contiguous:
        out.data = np.empty((d, s), np.float32)
    out.num_dms, out.samples_per_second = d, s
    check(lib().dd_dedisperse(context(device).handle, data.ctypes.data, fb.setup.channels,
                              fb.num_samples, shifts.ctypes.data, d, s,
                              C.byref(cfg) if cfg is not None else None,
                              C.byref(limits) if limits is not None else None,
                              out.data.ctypes.data))


def dedisperse_reference_into(out: DedispersedSeries, fb: Filterbank, table: DelayTable,
                              stats: Optional[KernelStats] = None, device: int = 0) -> None:
    """reference kernels.cpp:83-108, on the device in the same per-output order."""
    _run(out, fb, table, None, None, device)
    if stats is not None:
        total = table.num_dms * fb.setup.samples_per_second * fb.setup.channels
        stats.flop_additions += total
        stats.staged_loads += total


def dedisperse_reference(fb: Filterbank, table: DelayTable,
                         stats: Optional[KernelStats] = None, device: int = 0) -> DedispersedSeries:
    out = DedispersedSeries()
    dedisperse_reference_into(out, fb, table, stats, device)
    return out


def dedisperse_tiled_into(out: DedispersedSeries, fb: Filterbank, table: DelayTable,
                          cfg: KernelConfig, options: ExecOptions = ExecOptions()) -> None:
    """reference kernels.cpp:117-206: bit-identical to dedisperse_reference."""
    _check_pair(fb, table)
    validate_config(cfg, table.num_dms, fb.setup.samples_per_second, options.limits)
    _run(out, fb, table, _cfg(cfg, options.dm_tile_depth, options.staging),
         options.limits.c(), options.device)
    if options.stats is not None:
        options.stats.flop_additions += (table.num_dms * fb.setup.samples_per_second
                                         * fb.setup.channels)
        options.stats.staged_loads += count_loads(table, cfg, table.num_dms,
                                                  fb.setup.samples_per_second).staged_loads


def dedisperse_tiled(fb: Filterbank, table: DelayTable, cfg: KernelConfig,
                     options: ExecOptions = ExecOptions()) -> DedispersedSeries:
    out = DedispersedSeries()
    dedisperse_tiled_into(out, fb, table, cfg, options)
    return out


def count_loads(table: DelayTable, cfg: KernelConfig, num_dms: int,
                samples_per_second: int, flags: int = 0) -> LoadCounts:
    """reference count_loads.cpp:9-68 (flags: DD_CONFIG_GPU_TILING counts a
    predicated last time tile like a full one)."""
    if num_dms == 0 or num_dms != table.num_dms:
        raise ValueError("delay table does not cover the requested trial count")
    sh = np.ascontiguousarray(table.shifts, np.uint32)
    st, idl = C.c_uint64(), C.c_uint64()
    kc = _cfg(cfg)
    kc.flags = flags
    check(lib().dd_count_loads(sh.ctypes.data, table.setup.channels, num_dms, samples_per_second,
                               C.byref(kc), C.byref(st), C.byref(idl)))
    return LoadCounts(st.value, idl.value)


# ------------------------------------------------- device-side objects ---
class Context:
    """One dd_context: a device and a stream (replaces the reference ThreadPool)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().dd_context_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().dd_context_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        check(lib().dd_context_set_stream(self.handle, C.c_void_p(stream_ptr or None)))

    def synchronize(self) -> None:
        check(lib().dd_context_synchronize(self.handle))

    def info(self):
        sm, smem, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().dd_context_device_info(self.handle, C.byref(sm), C.byref(smem), C.byref(ma),
                                           C.byref(mi)))
        return {"sm_count": sm.value, "smem_optin": smem.value, "cc": (ma.value, mi.value)}

    def delay_table(self, setup: ObservationSetup, num_dms: int, d_shifts: int,
                    dm_offset: int = 0, zero: bool = False) -> int:
        """K1 into a device buffer (rows dm_offset..); returns the slice max."""
        md = C.c_uint32()
        check(lib().dd_delay_table_device(self.handle, C.byref(setup.c()), num_dms, dm_offset,
                                          int(zero), C.c_void_p(d_shifts), C.byref(md)))
        return md.value

    def sigproc_to_filterbank(self, d_payload: int, channels: int, num_samples: int,
                              d_dst: int, dst_pitch: int) -> int:
        """Device transpose of a SIGPROC payload (time-major, highest channel
        first) into the channel-major lowest-first layout (reference
        sigproc.cpp:177-189).  Returns the payload index of the first
        non-finite sample, or -1."""
        bad = C.c_int64()
        check(lib().dd_sigproc_to_filterbank(self.handle, C.c_void_p(d_payload), channels,
                                             num_samples, C.c_void_p(d_dst), dst_pitch,
                                             C.byref(bad)))
        return bad.value

    def upload_block_range(self, h_block: int, h_pitch: int, d_block: int, d_pitch: int,
                           channels: int, t0: int, t1: int, stream: int = 0) -> None:
        """Samples [t0, t1) of every channel, host -> device, one async 2-D
        copy on `stream` (a cudaStream_t; 0 = the context stream)."""
        check(lib().dd_upload_block_range(self.handle, C.c_void_p(h_block), h_pitch,
                                          C.c_void_p(d_block), d_pitch, channels, t0, t1,
                                          C.c_void_p(stream)))

    def plan(self, d_shifts: int, channels: int, num_dms: int, samples_per_second: int,
             num_samples: int, in_pitch: int, cfg: Optional[KernelConfig] = None,
             dm_tile_depth: int = 1, staging: str = "auto",
             limits: KernelLimits = KernelLimits(), gpu_tiling: bool = False,
             stage_channels: int = 0, high_occupancy: bool = False, flags: int = 0) -> "Plan":
        """gpu_tiling: tile_time need not divide s (staged families only);
        stage_channels: channels per pipeline stage (0 = plan's choice);
        high_occupancy: TMEM windows' three-CTA build; flags: raw DD_CONFIG_*
        bits OR-ed in (as stored in tuning records)."""
        return Plan(self, d_shifts, channels, num_dms, samples_per_second, num_samples, in_pitch,
                    cfg, dm_tile_depth, staging, limits, gpu_tiling, stage_channels,
                    high_occupancy, flags)


class Plan:
    """dd_plan: a table + config bound to one kernel launch."""

    def __init__(self, ctx: Context, d_shifts, channels, num_dms, s, num_samples, in_pitch,
                 cfg, depth, staging, limits, gpu_tiling=False, stage_channels=0,
                 high_occupancy=False, flags=0):
        self.ctx = ctx
        self.num_dms, self.s, self.channels = num_dms, s, channels
        h = C.c_void_p()
        kc = _cfg(cfg, depth, staging, gpu_tiling, stage_channels,
                  high_occupancy) if cfg is not None else None
        if kc is not None:
            kc.flags |= flags
        check(lib().dd_plan_create(ctx.handle, C.c_void_p(d_shifts), channels, num_dms, s,
                                   num_samples, in_pitch, C.byref(kc) if kc is not None else None,
                                   C.byref(limits.c()), C.byref(h)))
        self.handle = h

    def close(self) -> None:
        if self.handle:
            lib().dd_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = N.dd_plan_info()
        check(lib().dd_plan_get_info(self.handle, C.byref(i)))
        d = {f: getattr(i, f) for f, _ in N.dd_plan_info._fields_}
        d["family"] = N.STAGING_NAME.get(d["family"], d["family"])
        return d

    def execute(self, d_in: int, d_out: int, out_pitch: Optional[int] = None) -> None:
        check(lib().dd_plan_execute(self.handle, C.c_void_p(d_in), C.c_void_p(d_out),
                                    out_pitch or self.s))

    def execute_channels(self, d_in: int, d_out: int, ch_begin: int, ch_end: int,
                         accumulate: bool, out_pitch: Optional[int] = None) -> None:
        """Channels [ch_begin, ch_end) only; accumulate continues from d_out."""
        check(lib().dd_plan_execute_channels(self.handle, C.c_void_p(d_in), C.c_void_p(d_out),
                                             out_pitch or self.s, ch_begin, ch_end,
                                             int(accumulate)))

    def execute_beams(self, beams: int, d_in: int, in_beam_stride: int, d_out: int,
                      out_beam_stride: int, out_pitch: Optional[int] = None) -> None:
        """`beams` independent beams in one launch (strides in floats)."""
        check(lib().dd_plan_execute_beams(self.handle, beams, C.c_void_p(d_in), in_beam_stride,
                                          C.c_void_p(d_out), out_pitch or self.s,
                                          out_beam_stride))

    def time(self, d_in: int, d_out: int, warmup: int = 1, repeats: int = 10,
             out_pitch: Optional[int] = None, flush_l2: bool = False) -> List[float]:
        """CUDA-event time of each of `repeats` runs after `warmup` untimed
        ones; flush_l2 evicts L2 before every timed run (outside the events)."""
        runs = (C.c_double * max(repeats, 1))()
        check(lib().dd_plan_time_ex(self.handle, C.c_void_p(d_in), C.c_void_p(d_out),
                                    out_pitch or self.s, warmup, repeats, int(flush_l2), runs))
        return list(runs[:repeats])


_contexts = {}


def context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


def device_count() -> int:
    n = C.c_int()
    st = lib().dd_device_count(C.byref(n))
    return n.value if st == N.DD_OK else 0


# ----------------------------------------------------------------- tuner --
@dataclass
class TuningRecord:
    """reference tuner.hpp:17-23 plus the GPU knobs."""

    config: KernelConfig
    runs: List[float] = field(default_factory=list)
    mean_time: float = 0.0
    gflops: float = 0.0
    timer_warning: bool = False
    dm_tile_depth: int = 1
    staging: str = "auto"
    family: str = ""
    flags: int = 0  # DD_CONFIG_* (GPU tiling, channels per stage)

    @property
    def stage_channels(self) -> int:
        return (self.flags & N.DD_CONFIG_CPS_MASK) >> N.DD_CONFIG_CPS_SHIFT

    def c(self) -> N.dd_tuning_record:
        r = N.dd_tuning_record()
        r.config = _cfg(self.config, self.dm_tile_depth, self.staging)
        r.config.flags = self.flags
        r.mean_time = self.mean_time
        r.gflops = self.gflops
        return r


@dataclass
class TuningStats:
    mean_gflops: float = 0.0
    stddev_gflops: float = 0.0
    snr_optimum: Optional[float] = None
    chebyshev_bound: Optional[float] = None
    degenerate: bool = False


@dataclass
class TuningResult:
    """reference tuner.hpp:37-55"""

    setup: ObservationSetup
    num_dms: int
    zero_dm: bool
    limits: KernelLimits
    repeats: int
    seed: int
    records: List[TuningRecord]
    best_index: int
    stats: TuningStats
    realtime_threshold_gflops: float
    realtime_pass: bool
    rng_id: str = "mt19937_64/box-muller"
    clock_resolution_s: float = 0.5e-6

    def best(self) -> TuningRecord:
        return self.records[self.best_index]


def enumerate_configs(num_dms: int, samples_per_second: int,
                      limits: KernelLimits = KernelLimits()) -> List[KernelConfig]:
    """reference tuner.cpp:103-134"""
    n = C.c_uint64()
    check(lib().dd_enumerate_configs(num_dms, samples_per_second, C.byref(limits.c()), None, 0,
                                     C.byref(n)))
    buf = (N.dd_config * max(n.value, 1))()
    check(lib().dd_enumerate_configs(num_dms, samples_per_second, C.byref(limits.c()), buf,
                                     n.value, C.byref(n)))
    return [KernelConfig(b.items_time, b.items_dm, b.work_time, b.work_dm) for b in buf[:n.value]]


def enumerate_gpu_configs(setup: ObservationSetup, num_dms: int,
                          limits: KernelLimits = KernelLimits(), device: int = 0):
    """The GPU tuning space: [(KernelConfig, dm_tile_depth, staging)]."""
    ctx = context(device)
    n = C.c_uint64()
    check(lib().dd_enumerate_gpu_configs(ctx.handle, C.byref(setup.c()), num_dms,
                                         C.byref(limits.c()), None, 0, C.byref(n)))
    buf = (N.dd_config * max(n.value, 1))()
    check(lib().dd_enumerate_gpu_configs(ctx.handle, C.byref(setup.c()), num_dms,
                                         C.byref(limits.c()), buf, n.value, C.byref(n)))
    return [(KernelConfig(b.items_time, b.items_dm, b.work_time, b.work_dm), b.dm_tile_depth,
             N.STAGING_NAME[b.staging], b.flags) for b in buf[:n.value]]


def select_best(records: Sequence[TuningRecord]) -> int:
    """reference tuner.cpp:172-179 (ties: fewer block items, then config order)."""
    if not records:
        raise ValueError("no records to select from")
    arr = (N.dd_tuning_record * len(records))(*[r.c() for r in records])
    b = C.c_uint64()
    check(lib().dd_select_best(arr, len(records), C.byref(b)))
    return b.value


def compute_stats(records: Sequence[TuningRecord], best_index: int) -> TuningStats:
    """reference tuner.cpp:181-206"""
    if not records:
        raise ValueError("no records to summarize")
    arr = (N.dd_tuning_record * len(records))(*[r.c() for r in records])
    s = N.dd_tuning_summary()
    check(lib().dd_compute_stats(arr, len(records), best_index, C.byref(s)))
    return _stats(s)


def _stats(s) -> TuningStats:
    deg = bool(s.degenerate)
    return TuningStats(s.mean_gflops, s.stddev_gflops, None if deg else s.snr_optimum,
                       None if deg else s.chebyshev_bound, deg)


def _sweep(setup, num_dms, limits, repeats, seed, zero, full_space, max_configs, device,
           flush_l2=True):
    ctx = context(device)
    opt = N.dd_tune_options(limits.c(), repeats, int(zero), seed, int(full_space), max_configs,
                            int(flush_l2), 0)
    n = C.c_uint64()
    if full_space:
        check(lib().dd_enumerate_configs(num_dms, setup.samples_per_second, C.byref(limits.c()),
                                         None, 0, C.byref(n)))
    else:
        check(lib().dd_enumerate_gpu_configs(ctx.handle, C.byref(setup.c()), num_dms,
                                             C.byref(limits.c()), None, 0, C.byref(n)))
    if max_configs:
        n.value = min(n.value, max_configs)
    recs = (N.dd_tuning_record * max(n.value, 1))()
    runs = (C.c_double * max(n.value * repeats, 1))()
    opt.runs = C.cast(runs, C.POINTER(C.c_double))
    summ = N.dd_tuning_summary()
    check(lib().dd_tune(ctx.handle, C.byref(setup.c()), num_dms, C.byref(opt), recs, n.value,
                        C.byref(summ)))
    out = []
    for i, r in enumerate(recs[:summ.count]):
        k = r.config
        out.append(TuningRecord(KernelConfig(k.items_time, k.items_dm, k.work_time, k.work_dm),
                                list(runs[i * repeats:(i + 1) * repeats]), r.mean_time,
                                r.gflops, bool(r.timer_warning),
                                k.dm_tile_depth, N.STAGING_NAME[k.staging],
                                N.STAGING_NAME.get(r.family, ""), k.flags))
    return TuningResult(setup, num_dms, zero, limits, repeats, seed, out, summ.best_index,
                        _stats(summ), summ.realtime_threshold_gflops, bool(summ.realtime_pass))


def tune(setup: ObservationSetup, num_dms: int, limits: KernelLimits = KernelLimits(),
         repeats: int = 10, seed: int = 1, full_reference_space: bool = False,
         max_configs: int = 0, device: int = 0, flush_l2: bool = True) -> TuningResult:
    """reference tuner.cpp:208-211 on the device (CUDA-event timing; L2
    flushed before every timed run unless flush_l2=False; every run kept in
    record.runs like the reference's runs_s)."""
    return _sweep(setup, num_dms, limits, repeats, seed, False, full_reference_space,
                  max_configs, device, flush_l2)


def zero_dm_experiment(setup: ObservationSetup, num_dms: int, limits: KernelLimits = KernelLimits(),
                       repeats: int = 10, seed: int = 1, full_reference_space: bool = False,
                       max_configs: int = 0, device: int = 0,
                       flush_l2: bool = True) -> TuningResult:
    """reference tuner.cpp:213-216"""
    return _sweep(setup, num_dms, limits, repeats, seed, True, full_reference_space,
                  max_configs, device, flush_l2)


def schedule_set(channels: int, samples_per_second: int, num_dms: int,
                 record: Optional["TuningRecord"]) -> None:
    """Register the schedule the one-shot entry points (dedisperse_tiled with
    staging "auto") run for this instance -- typically a tuning result's
    best record; None forgets it (dd_schedule_set)."""
    if record is None:
        check(lib().dd_schedule_set(channels, samples_per_second, num_dms, None))
        return
    kc = _cfg(record.config, record.dm_tile_depth, record.staging)
    kc.flags = record.flags
    check(lib().dd_schedule_set(channels, samples_per_second, num_dms, C.byref(kc)))


def schedule_get(channels: int, samples_per_second: int, num_dms: int):
    """(KernelConfig, dm_tile_depth, staging, flags, builtin) of the
    instance's tuned schedule, or None (dd_schedule_get)."""
    kc, b = N.dd_config(), C.c_int()
    if lib().dd_schedule_get(channels, samples_per_second, num_dms, C.byref(kc),
                             C.byref(b)) != N.DD_OK:
        return None
    return (KernelConfig(kc.items_time, kc.items_dm, kc.work_time, kc.work_dm), kc.dm_tile_depth,
            N.STAGING_NAME[kc.staging], kc.flags, bool(b.value))


def last_run_config(device: int = 0):
    """What the last one-shot call on this device's context ran:
    (KernelConfig, dm_tile_depth, staging, flags, family)."""
    kc, fam = N.dd_config(), C.c_uint32()
    check(lib().dd_last_run_config(context(device).handle, C.byref(kc), C.byref(fam)))
    return (KernelConfig(kc.items_time, kc.items_dm, kc.work_time, kc.work_dm), kc.dm_tile_depth,
            N.STAGING_NAME[kc.staging], kc.flags, N.STAGING_NAME.get(fam.value, fam.value))


def fingerprint(a) -> str:
    """FNV-1a 64 of an array's raw bytes (dd_fingerprint), the hash the
    golden fixtures use; a host numpy array or anything with .numpy()."""
    if hasattr(a, "numpy"):
        a = a.numpy()
    a = np.ascontiguousarray(a)
    h = C.c_uint64()
    check(lib().dd_fingerprint(a.ctypes.data, a.nbytes, C.byref(h)))
    return "%016x" % h.value


@dataclass
class FixedConfigReport:
    config: tuple
    total_gflops: float
    fixed_gflops: List[float]
    speedup_over_fixed: List[float]


def best_fixed_config(results: Sequence[TuningResult]) -> FixedConfigReport:
    """reference tuner.cpp:218-261 (identity = 4-tuple + GPU knobs)."""
    if not results:
        raise ValueError("no tuning results given")
    first = results[0].setup
    for r in results:
        if (r.setup.name != first.name or r.setup.samples_per_second != first.samples_per_second
                or r.setup.channels != first.channels):
            raise ValueError("tuning results mix different setups")
        if not r.records:
            raise ValueError("a tuning result holds no records")
    by = {}
    for i, r in enumerate(results):
        for rec in r.records:
            key = (rec.config, rec.dm_tile_depth, rec.staging, rec.flags)
            v = by.setdefault(key, [])
            if len(v) == i:
                v.append(rec.gflops)
    best = None
    for key in sorted(by, key=lambda k: (k[0], k[1], k[2], k[3])):
        v = by[key]
        if len(v) != len(results):
            continue
        tot = sum(v)
        if best is None or tot > best[1]:
            best = (key, tot, v)
    if best is None:
        raise ValueError("no configuration is valid in every instance")
    key, tot, v = best
    return FixedConfigReport(key, tot, list(v),
                             [r.best().gflops / g for r, g in zip(results, v)])


def default_instances() -> List[int]:
    """reference tuner.cpp:292-296"""
    return [2 ** k for k in range(1, 13)]


# -------------------------------------------------- analysis (metric defs) --
def realtime_threshold_gflops(setup: ObservationSetup, num_dms: int) -> float:
    """reference analysis.cpp:40-45"""
    setup.validate()
    if num_dms == 0:
        raise ValueError("need at least one trial DM")
    return num_dms * setup.samples_per_second * setup.channels / 1e9


def ai_bounds(num_dms: int, samples_per_second: int, channels: int):
    """reference analysis.cpp:11-21 -> (no_reuse, reuse_bound) flop/byte."""
    if not (num_dms and samples_per_second and channels):
        raise ValueError("instance dimensions must all be positive")
    return 0.25, 1.0 / (4.0 * (1.0 / num_dms + 1.0 / samples_per_second + 1.0 / channels))


def algorithmic_bytes(num_dms: int, samples_per_second: int, channels: int) -> int:
    """Eq. 2 no-reuse traffic 4*(d*s*c + d*s + d*c)."""
    d, s, c = num_dms, samples_per_second, channels
    return 4 * (d * s * c + d * s + d * c)


def roofline_gflops(num_dms: int, samples_per_second: int, channels: int, hbm_gbs: float) -> float:
    d, s, c = num_dms, samples_per_second, channels
    return d * s * c / (algorithmic_bytes(d, s, c) / (hbm_gbs * 1e9)) / 1e9


@dataclass(frozen=True)
class MemoryTraffic:
    """reference analysis.hpp:26-30 (elements of 4 bytes)."""

    staged_loads: int
    output_writes: int
    delay_reads: int


def kernel_traffic(table: DelayTable, cfg: KernelConfig, num_dms: int,
                   samples_per_second: int, flags: int = 0) -> MemoryTraffic:
    """reference analysis.cpp:23-31: count_loads' staged loads + one write
    per output + one read per table entry."""
    loads = count_loads(table, cfg, num_dms, samples_per_second, flags)
    return MemoryTraffic(loads.staged_loads, num_dms * samples_per_second,
                         num_dms * table.setup.channels)


def measured_ai(flops: int, traffic: MemoryTraffic) -> float:
    """reference analysis.cpp:33-38"""
    elements = traffic.staged_loads + traffic.output_writes + traffic.delay_reads
    if elements == 0:
        raise ValueError("no memory traffic to divide by")
    return float(flops) / (4.0 * float(elements))


class NotRealTimeError(RuntimeError):
    """reference errors.hpp not_real_time_error"""


@dataclass(frozen=True)
class DeploymentPlan:
    beams_per_device: int
    devices: int


def deployment_sizing(setup: ObservationSetup, num_dms: int, beams: int,
                      measured_time_per_pass: float) -> DeploymentPlan:
    """reference analysis.cpp:47-65"""
    setup.validate()
    if num_dms == 0:
        raise ValueError("need at least one trial DM")
    if beams == 0:
        raise ValueError("need at least one beam")
    t = measured_time_per_pass
    if not math.isfinite(t) or t <= 0.0:
        raise ValueError("pass time must be a positive number of seconds")
    if t >= 1.0:
        raise NotRealTimeError(f"one pass takes {t} s; a device cannot keep up with even a "
                               "single beam")
    per = int(1.0 / t)
    return DeploymentPlan(per, (beams + per - 1) // per)


@dataclass(frozen=True)
class RooflineVerdict:
    memory_bound: bool
    ridge_flop_per_byte: float
    attainable_gflops: float


def classify_roofline(ai_flop_per_byte: float, peak_gflops: float,
                      peak_gbs: float) -> RooflineVerdict:
    """reference analysis.cpp:79-93"""
    if not math.isfinite(ai_flop_per_byte) or ai_flop_per_byte <= 0.0:
        raise ValueError("arithmetic intensity must be positive")
    if (not math.isfinite(peak_gflops) or peak_gflops <= 0.0 or not math.isfinite(peak_gbs)
            or peak_gbs <= 0.0):
        raise ValueError("device peaks must be positive")
    ridge = peak_gflops / peak_gbs
    return RooflineVerdict(ai_flop_per_byte < ridge, ridge,
                           min(peak_gflops, ai_flop_per_byte * peak_gbs))


@dataclass(frozen=True)
class HistogramBin:
    lo: float
    hi: float
    count: int


def make_histogram(result: TuningResult, bins: int) -> List[HistogramBin]:
    """reference tuner.cpp:263-290: equal-width gflops bins over [min, max];
    the maximum lands in the last bin, a flat population in the first."""
    if bins == 0:
        raise ValueError("need at least one histogram bin")
    if not result.records:
        raise ValueError("no records to bin")
    g = [r.gflops for r in result.records]
    lo, hi = min(g), max(g)
    width = (hi - lo) / bins
    edges = [(lo + width * i, hi if i + 1 == bins else lo + width * (i + 1)) for i in range(bins)]
    counts = [0] * bins
    for x in g:
        counts[min(int((x - lo) / width), bins - 1) if width > 0.0 else 0] += 1
    return [HistogramBin(a, b, n) for (a, b), n in zip(edges, counts)]


# ------------------------------------------------ tuning-result documents --
TUNING_SCHEMA = "dedisp-tuning-result/1"


def tuning_result_to_dict(result: TuningResult, threads: int = 1) -> dict:
    """The reference's tuning-result document (report_io.cpp:58-102: same
    keys, same order, schema "dedisp-tuning-result/1") so its `analyze`
    subcommand and tuning_result_from_json read GPU results unchanged.  The
    GPU knobs of each record ride in an extra "b200" object, which the
    reference parser ignores; `threads` is the host-thread field (1: the
    device sweep is sequential)."""
    s = result.setup
    recs = []
    for r in result.records:
        k = r.config
        recs.append({"items_time": k.items_time, "items_dm": k.items_dm,
                     "work_time": k.work_time, "work_dm": k.work_dm,
                     "runs_s": list(r.runs), "mean_time_s": r.mean_time, "gflops": r.gflops,
                     "timer_warning": r.timer_warning,
                     "b200": {"dm_tile_depth": r.dm_tile_depth, "staging": r.staging,
                              "family": r.family, "flags": r.flags}})
    st = result.stats
    return {
        "schema": TUNING_SCHEMA,
        "setup": {"name": s.name, "samples_per_second": s.samples_per_second,
                  "channels": s.channels, "f_min_mhz": s.f_min,
                  "channel_width_mhz": s.channel_width, "dm_first": s.dm_first,
                  "dm_step": s.dm_step},
        "num_dms": result.num_dms,
        "zero_dm": result.zero_dm,
        "limits": {"max_block_items": result.limits.max_block_items,
                   "max_accumulators": result.limits.max_accumulators},
        "repeats": result.repeats,
        "seed": result.seed,
        "environment": {"threads": threads, "rng": result.rng_id,
                        "clock_resolution_s": result.clock_resolution_s},
        "records": recs,
        "best_index": result.best_index,
        "stats": {"mean_gflops": st.mean_gflops, "stddev_gflops": st.stddev_gflops,
                  "snr_optimum": st.snr_optimum, "chebyshev_bound": st.chebyshev_bound,
                  "degenerate": st.degenerate},
        "realtime": {"threshold_gflops": result.realtime_threshold_gflops,
                     "pass": result.realtime_pass},
    }


def tuning_result_to_json(result: TuningResult, threads: int = 1) -> str:
    return json.dumps(tuning_result_to_dict(result, threads), indent=2) + "\n"


class FormatError(ValueError):
    """reference errors.hpp format_error"""


def tuning_result_from_json(text: str) -> TuningResult:
    """reference report_io.cpp:104-156: every key it requires is required
    here; a document without "b200" record objects (the CPU reference's own)
    loads with default GPU knobs."""
    try:
        doc = json.loads(text)
        if doc["schema"] != TUNING_SCHEMA:
            raise FormatError(f"unrecognized schema '{doc['schema']}'")
        s = doc["setup"]
        setup = ObservationSetup(s["name"], int(s["samples_per_second"]), int(s["channels"]),
                                 float(s["f_min_mhz"]), float(s["channel_width_mhz"]),
                                 float(s["dm_first"]), float(s["dm_step"]))
        recs = []
        for n in doc["records"]:
            x = n.get("b200", {})
            recs.append(TuningRecord(KernelConfig(int(n["items_time"]), int(n["items_dm"]),
                                                  int(n["work_time"]), int(n["work_dm"])),
                                     [float(v) for v in n["runs_s"]], float(n["mean_time_s"]),
                                     float(n["gflops"]), bool(n["timer_warning"]),
                                     int(x.get("dm_tile_depth", 1)), x.get("staging", "auto"),
                                     x.get("family", ""), int(x.get("flags", 0))))
        best = int(doc["best_index"])
        if not recs or best >= len(recs):
            raise FormatError("best_index does not point into records")
        st = doc["stats"]
        stats = TuningStats(float(st["mean_gflops"]), float(st["stddev_gflops"]),
                            st["snr_optimum"], st["chebyshev_bound"], bool(st["degenerate"]))
        env = doc["environment"]
        res = TuningResult(setup, int(doc["num_dms"]), bool(doc["zero_dm"]),
                           KernelLimits(int(doc["limits"]["max_block_items"]),
                                        int(doc["limits"]["max_accumulators"])),
                           int(doc["repeats"]), int(doc["seed"]), recs, best, stats,
                           float(doc["realtime"]["threshold_gflops"]),
                           bool(doc["realtime"]["pass"]), env["rng"],
                           float(env["clock_resolution_s"]))
        int(env["threads"])
        return res
    except FormatError:
        raise
    except (ValueError, KeyError, TypeError, AttributeError) as e:
        raise FormatError(f"bad tuning-result document: {e!r}") from None


def tuning_result_to_csv(result: TuningResult) -> str:
    """reference report_io.cpp:166-176"""
    rows = ["items_time,items_dm,work_time,work_dm,mean_time_s,gflops"]
    for r in result.records:
        k = r.config
        rows.append(f"{k.items_time},{k.items_dm},{k.work_time},{k.work_dm},"
                    f"{r.mean_time:.17g},{r.gflops:.17g}")
    return "\n".join(rows) + "\n"
