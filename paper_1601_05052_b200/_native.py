"""ctypes binding of the C-ABI (include/dedisp_b200.h).

The library is the in-tree ``libdedisp_b200.so`` built by
``paper_1601_05052_b200.build``.  There is no fallback: if the library is
missing or has no CUDA device, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# DDB_LIB: load another build of the same library (A/B kernel timing with
# tools/time_configs.py); it must export every symbol below, no fallback.
LIB_PATH = os.environ.get("DDB_LIB") or os.path.join(PKG, "libdedisp_b200.so")

DD_OK, DD_ERR_INVALID_ARGUMENT, DD_ERR_CAPACITY, DD_ERR_CUDA, DD_ERR_NO_DEVICE, DD_ERR_INTERNAL = range(6)
STAGING = {"auto": 0, "smem": 1, "direct": 2, "regwin": 3, "tmem": 4, "rect": 5}
STAGING_NAME = {v: k for k, v in STAGING.items()}
DD_CONFIG_GPU_TILING = 0x1
DD_CONFIG_HIGH_OCCUPANCY = 0x2
DD_CONFIG_TIME_MAJOR = 0x8
DD_CONFIG_PACKED_STAGES = 0x10
DD_CONFIG_WIDE_STAGES = 0x20
DD_CONFIG_CPS_SHIFT = 8
DD_CONFIG_CPS_MASK = 0xF << DD_CONFIG_CPS_SHIFT
DD_CONFIG_NSTAGE_SHIFT = 12
DD_CONFIG_NSTAGE_MASK = 0xF << DD_CONFIG_NSTAGE_SHIFT


class CapacityError(RuntimeError):
    """dedisp::capacity_error (reference errors.hpp:10-13)."""


class DeviceError(RuntimeError):
    """CUDA / device failure (dedisp::device_error)."""


class dd_setup(C.Structure):
    _fields_ = [("samples_per_second", C.c_uint32), ("channels", C.c_uint32),
                ("f_min", C.c_double), ("channel_width", C.c_double),
                ("dm_first", C.c_double), ("dm_step", C.c_double)]


class dd_config(C.Structure):
    _fields_ = [("items_time", C.c_uint32), ("items_dm", C.c_uint32),
                ("work_time", C.c_uint32), ("work_dm", C.c_uint32),
                ("dm_tile_depth", C.c_uint32), ("staging", C.c_uint32),
                ("flags", C.c_uint32)]

    def tuple(self):
        return (self.items_time, self.items_dm, self.work_time, self.work_dm,
                self.dm_tile_depth, self.staging, self.flags)


class dd_limits(C.Structure):
    _fields_ = [("max_block_items", C.c_uint32), ("max_accumulators", C.c_uint32)]


class dd_plan_info(C.Structure):
    _fields_ = [("family", C.c_uint32), ("max_span", C.c_uint32), ("max_delay", C.c_uint32),
                ("grid_x", C.c_uint32), ("grid_y", C.c_uint32), ("block_threads", C.c_uint32),
                ("smem_bytes", C.c_uint32), ("channels_per_stage", C.c_uint32),
                ("stages", C.c_uint32), ("kernel_launches", C.c_uint32),
                ("staged_bytes", C.c_uint64), ("registers", C.c_uint32),
                ("ctas_per_sm", C.c_uint32), ("time_major", C.c_uint32),
                ("packed_stages", C.c_uint32)]


class dd_tune_options(C.Structure):
    _fields_ = [("limits", dd_limits), ("repeats", C.c_uint32), ("zero_dm", C.c_uint32),
                ("seed", C.c_uint64), ("space", C.c_uint32), ("max_configs", C.c_uint32),
                ("flush_l2", C.c_uint32), ("reserved", C.c_uint32),
                ("runs", C.POINTER(C.c_double))]


class dd_tuning_record(C.Structure):
    _fields_ = [("config", dd_config), ("mean_time", C.c_double), ("min_time", C.c_double),
                ("max_time", C.c_double), ("gflops", C.c_double),
                ("timer_warning", C.c_uint32), ("family", C.c_uint32)]


class dd_tuning_summary(C.Structure):
    _fields_ = [("count", C.c_uint64), ("best_index", C.c_uint64), ("mean_gflops", C.c_double),
                ("stddev_gflops", C.c_double), ("snr_optimum", C.c_double),
                ("chebyshev_bound", C.c_double), ("degenerate", C.c_uint32),
                ("realtime_pass", C.c_uint32), ("realtime_threshold_gflops", C.c_double),
                ("clock_resolution_s", C.c_double)]


P = C.c_void_p
u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
pu32, pu64, pf32, pdbl = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_float), C.POINTER(C.c_double)

# name -> (restype, argtypes); mirrors include/dedisp_b200.h exactly.
SIGNATURES = {
    "dd_last_error": (C.c_char_p, []),
    "dd_abi_version": (C.c_int, []),
    "dd_device_count": (i32, [C.POINTER(C.c_int)]),
    "dd_context_create": (i32, [C.c_int, C.POINTER(P)]),
    "dd_context_destroy": (i32, [P]),
    "dd_context_set_stream": (i32, [P, P]),
    "dd_context_stream": (P, [P]),
    "dd_context_synchronize": (i32, [P]),
    "dd_context_device_info": (i32, [P, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "dd_device_malloc": (i32, [P, u64, C.POINTER(P)]),
    "dd_device_free": (i32, [P, P]),
    "dd_host_malloc": (i32, [u64, C.POINTER(P)]),
    "dd_host_free": (i32, [P]),
    "dd_copy_h2d": (i32, [P, P, P, u64]),
    "dd_copy_d2h": (i32, [P, P, P, u64]),
    "dd_upload_filterbank": (i32, [P, P, u64, P, u32, u64]),
    "dd_setup_validate": (i32, [C.POINTER(dd_setup)]),
    "dd_delay_seconds": (i32, [C.c_double, C.c_double, C.c_double, pdbl]),
    "dd_instance_sizing": (i32, [C.POINTER(dd_setup), u32, pu64, pu64, pu32]),
    "dd_delay_table_device": (i32, [P, C.POINTER(dd_setup), u32, u32, C.c_int, P, pu32]),
    "dd_build_delay_table": (i32, [P, C.POINTER(dd_setup), u32, u64, C.c_int, P, pu32]),
    "dd_config_valid": (C.c_int, [C.POINTER(dd_config), u32, u32, C.POINTER(dd_limits)]),
    "dd_validate_config": (i32, [C.POINTER(dd_config), u32, u32, C.POINTER(dd_limits)]),
    "dd_config_family": (i32, [P, C.POINTER(dd_config), u32, u32, u32, u32, pu32]),
    "dd_count_loads": (i32, [P, u32, u32, u32, C.POINTER(dd_config), pu64, pu64]),
    "dd_plan_create": (i32, [P, P, u32, u32, u32, u64, u64, C.POINTER(dd_config),
                             C.POINTER(dd_limits), C.POINTER(P)]),
    "dd_plan_destroy": (i32, [P]),
    "dd_plan_get_info": (i32, [P, C.POINTER(dd_plan_info)]),
    "dd_plan_execute": (i32, [P, P, P, u64]),
    "dd_plan_time": (i32, [P, P, P, u64, u32, u32, pdbl]),
    "dd_plan_time_ex": (i32, [P, P, P, u64, u32, u32, C.c_int, pdbl]),
    "dd_fingerprint": (i32, [P, u64, pu64]),
    "dd_debug_violations": (i32, [pu64, C.POINTER(C.c_int), C.c_int]),
    "dd_schedule_set": (i32, [u32, u32, u32, C.POINTER(dd_config)]),
    "dd_schedule_get": (i32, [u32, u32, u32, C.POINTER(dd_config), C.POINTER(C.c_int)]),
    "dd_last_run_config": (i32, [P, C.POINTER(dd_config), pu32]),
    "dd_block_stream_create": (i32, [P, C.POINTER(dd_setup), u32, C.POINTER(dd_config),
                                     C.POINTER(P)]),
    "dd_block_stream_push": (i32, [P, P, P, C.POINTER(C.c_int)]),
    "dd_block_stream_info": (i32, [P, pu64, pu64, pu64, pu64, C.POINTER(P)]),
    "dd_block_stream_destroy": (i32, [P]),
    "dd_plan_execute_channels": (i32, [P, P, P, u64, u32, u32, C.c_int]),
    "dd_plan_execute_beams": (i32, [P, u32, P, u64, P, u64, u64]),
    "dd_dedisperse_device": (i32, [P, P, u32, u64, u64, P, u32, u32, C.POINTER(dd_config),
                                   C.POINTER(dd_limits), P]),
    "dd_dedisperse": (i32, [P, P, u32, u64, P, u32, u32, C.POINTER(dd_config),
                            C.POINTER(dd_limits), P]),
    "dd_noise_filterbank": (i32, [u32, u64, C.c_float, u64, C.c_int, P]),
    "dd_sigproc_to_filterbank": (i32, [P, P, u32, u64, P, u64, C.POINTER(C.c_int64)]),
    "dd_upload_block_range": (i32, [P, P, u64, P, u64, u32, u64, u64, P]),
    "dd_enumerate_configs": (i32, [u32, u32, C.POINTER(dd_limits), C.POINTER(dd_config), u64, pu64]),
    "dd_enumerate_gpu_configs": (i32, [P, C.POINTER(dd_setup), u32, C.POINTER(dd_limits),
                                       C.POINTER(dd_config), u64, pu64]),
    "dd_tune": (i32, [P, C.POINTER(dd_setup), u32, C.POINTER(dd_tune_options),
                      C.POINTER(dd_tuning_record), u64, C.POINTER(dd_tuning_summary)]),
    "dd_select_best": (i32, [C.POINTER(dd_tuning_record), u64, pu64]),
    "dd_compute_stats": (i32, [C.POINTER(dd_tuning_record), u64, u64, C.POINTER(dd_tuning_summary)]),
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load the native library; raise (never fall back) when it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1601_05052_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int) -> None:
    if status == DD_OK:
        return
    msg = (lib().dd_last_error() or b"").decode()
    if status == DD_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == DD_ERR_CAPACITY:
        raise CapacityError(msg)
    raise DeviceError(msg or f"status {status}")
