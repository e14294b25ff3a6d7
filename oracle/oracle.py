"""ctypes face of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_1601_05052_b200) never does: it fails loudly when its CUDA library is
missing instead of falling back here.

Two libraries are wrapped:

* ``liboracle.so``     -- plain-C restatement of the reference hot path
  (oracle/dedisp_oracle.c, every function cites the reference file:line it
  follows).  Always available (gcc is on the GPU box too).
* ``_ref/libdedisp_ref.so`` -- the unmodified reference core compiled from
  /root/reference by oracle/Makefile (built in the dev container; the .so
  travels to the GPU box, /root/reference does not).  Optional.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LOCK = threading.Lock()
_LIB = None
_REF = None


class SetupC(C.Structure):
    _fields_ = [
        ("samples_per_second", C.c_uint32),
        ("channels", C.c_uint32),
        ("f_min", C.c_double),
        ("channel_width", C.c_double),
        ("dm_first", C.c_double),
        ("dm_step", C.c_double),
    ]


class ConfigC(C.Structure):
    _fields_ = [
        ("items_time", C.c_uint32),
        ("items_dm", C.c_uint32),
        ("work_time", C.c_uint32),
        ("work_dm", C.c_uint32),
    ]


@dataclass(frozen=True)
class Setup:
    """Mirror of ObservationSetup (reference setup.hpp:14-33)."""

    name: str
    samples_per_second: int
    channels: int
    f_min: float
    channel_width: float
    dm_first: float
    dm_step: float

    def c(self) -> SetupC:
        return SetupC(self.samples_per_second, self.channels, self.f_min,
                      self.channel_width, self.dm_first, self.dm_step)


# Built-in setups, reference setup.cpp:139-147.
APERTIF = Setup("Apertif", 20000, 1024, 1420.0, 0.29, 0.0, 0.25)
LOFAR = Setup("LOFAR", 200000, 32, 138.0, 0.19, 0.0, 0.25)


def _build(target: str) -> None:
    subprocess.run(["make", "-s", "-C", HERE, target], check=True,
                   stdout=subprocess.DEVNULL)


def lib() -> C.CDLL:
    """The C restatement; compiled on first use if absent."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            path = os.path.join(HERE, "liboracle.so")
            src = os.path.join(HERE, "dedisp_oracle.c")
            if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
                _build("oracle")
            L = C.CDLL(path)
            u32p = C.POINTER(C.c_uint32)
            u64p = C.POINTER(C.c_uint64)
            f32p = C.POINTER(C.c_float)
            L.or_fnv1a.restype = C.c_uint64
            L.or_fnv1a.argtypes = [C.c_void_p, C.c_uint64]
            L.or_delay_seconds.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
            L.or_build_delay_table.argtypes = [C.POINTER(SetupC), C.c_uint32, C.c_uint64, C.c_int,
                                               u32p, u32p]
            L.or_instance_sizing.argtypes = [C.POINTER(SetupC), C.c_uint32, u64p, u64p, u32p]
            L.or_noise_filterbank.argtypes = [C.c_uint32, C.c_uint64, C.c_float, C.c_uint64, f32p]
            L.or_config_valid.argtypes = [C.POINTER(ConfigC), C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint32]
            L.or_dedisperse_reference.argtypes = [f32p, C.c_uint32, C.c_uint64, u32p, C.c_uint32,
                                                  C.c_uint32, f32p]
            L.or_dedisperse_tiled.argtypes = [f32p, C.c_uint32, C.c_uint64, u32p, C.c_uint32,
                                              C.c_uint32, C.POINTER(ConfigC), C.c_int, f32p, u64p]
            L.or_count_loads.argtypes = [u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.POINTER(ConfigC), u64p, u64p]
            L.or_enumerate_configs.restype = C.c_uint64
            L.or_enumerate_configs.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.POINTER(ConfigC), C.c_uint64]
            _LIB = L
    return _LIB


def ref_lib():
    """The reference core itself (oracle/_ref), or None when not built."""
    global _REF
    with _LOCK:
        if _REF is None:
            path = os.path.join(HERE, "_ref", "libdedisp_ref.so")
            if not os.path.exists(path):
                if os.path.isdir("/root/reference/proj/core/src"):
                    _build("ref")
                else:
                    return None
            L = C.CDLL(path)
            u32p = C.POINTER(C.c_uint32)
            u64p = C.POINTER(C.c_uint64)
            f32p = C.POINTER(C.c_float)
            sp = C.POINTER(SetupC)
            kp = C.POINTER(ConfigC)
            L.ref_build_delay_table.argtypes = [sp, C.c_uint32, C.c_uint64, C.c_int, u32p, u32p]
            L.ref_instance_sizing.argtypes = [sp, C.c_uint32, u64p, u64p, u32p]
            L.ref_noise_filterbank.argtypes = [sp, C.c_uint32, C.c_float, C.c_uint64, f32p]
            L.ref_dedisperse_reference.argtypes = [sp, f32p, C.c_uint64, u32p, C.c_uint32, f32p]
            L.ref_dedisperse_tiled.argtypes = [sp, f32p, C.c_uint64, u32p, C.c_uint32, kp,
                                               C.c_int, f32p]
            L.ref_count_loads.argtypes = [sp, u32p, C.c_uint32, kp, u64p, u64p]
            L.ref_enumerate_configs.restype = C.c_int64
            L.ref_enumerate_configs.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                                kp, C.c_uint64]
            L.ref_job_create.restype = C.c_void_p
            L.ref_job_create.argtypes = [sp, f32p, C.c_uint64, u32p, C.c_uint32, C.c_int]
            L.ref_job_threads.argtypes = [C.c_void_p]
            L.ref_job_run_tiled.argtypes = [C.c_void_p, kp]
            L.ref_job_run_reference.argtypes = [C.c_void_p]
            L.ref_job_output.restype = f32p
            L.ref_job_output.argtypes = [C.c_void_p]
            L.ref_job_destroy.argtypes = [C.c_void_p]
            L.ref_parse_sigproc.argtypes = [C.c_char_p, C.c_uint64, u32p, u64p, f32p, u64p,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double), u32p]
            if hasattr(L, "ref_tuning_roundtrip"):
                L.ref_tuning_roundtrip.argtypes = [C.c_char_p, u32p, u64p, u32p,
                                                   C.POINTER(C.c_double), u32p, C.c_char_p,
                                                   C.c_uint64, u64p]
            _REF = L
    return _REF


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check(rc: int, what: str) -> None:
    if rc == 1:
        raise ValueError(f"oracle {what}: invalid argument")
    if rc == 2:
        raise MemoryError(f"oracle {what}: capacity")
    if rc != 0:
        raise RuntimeError(f"oracle {what}: error {rc}")


def fnv1a(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % lib().or_fnv1a(a.ctypes.data, a.nbytes)


def delay_seconds(dm: float, f_ch: float, f_hi: float) -> float:
    out = C.c_double()
    _check(lib().or_delay_seconds(dm, f_ch, f_hi, C.byref(out)), "delay_seconds")
    return out.value


def delay_table(setup: Setup, num_dms: int, zero: bool = False, cap: int = 1 << 30):
    """(shifts uint32 [num_dms, channels], max_delay) -- setup.cpp:86-110."""
    sh = np.empty((num_dms, setup.channels), np.uint32)
    md = C.c_uint32()
    _check(lib().or_build_delay_table(C.byref(setup.c()), num_dms, cap, int(zero),
                                      _p(sh, C.c_uint32), C.byref(md)), "delay_table")
    return sh, md.value


def instance_sizing(setup: Setup, num_dms: int):
    """(num_samples, flop, max_delay) -- setup.cpp:112-137."""
    t, f, m = C.c_uint64(), C.c_uint64(), C.c_uint32()
    _check(lib().or_instance_sizing(C.byref(setup.c()), num_dms, C.byref(t), C.byref(f),
                                    C.byref(m)), "instance_sizing")
    return t.value, f.value, m.value


def noise(channels: int, t: int, sigma: float = 1.0, seed: int = 1) -> np.ndarray:
    """float32 [channels, t] -- filterbank.cpp:60-80."""
    out = np.empty((channels, t), np.float32)
    _check(lib().or_noise_filterbank(channels, t, sigma, seed, _p(out, C.c_float)), "noise")
    return out


def dedisperse_reference(fb: np.ndarray, shifts: np.ndarray, s: int) -> np.ndarray:
    """float32 [d, s] -- kernels.cpp:83-108."""
    fb = np.ascontiguousarray(fb, np.float32)
    shifts = np.ascontiguousarray(shifts, np.uint32)
    c, t = fb.shape
    d = shifts.shape[0]
    out = np.empty((d, s), np.float32)
    _check(lib().or_dedisperse_reference(_p(fb, C.c_float), c, t, _p(shifts, C.c_uint32), d, s,
                                         _p(out, C.c_float)), "dedisperse_reference")
    return out


def dedisperse_tiled(fb: np.ndarray, shifts: np.ndarray, s: int, cfg, threads: int = 0):
    """float32 [d, s] via the tiled restatement (kernels.cpp:117-206)."""
    fb = np.ascontiguousarray(fb, np.float32)
    shifts = np.ascontiguousarray(shifts, np.uint32)
    c, t = fb.shape
    d = shifts.shape[0]
    out = np.empty((d, s), np.float32)
    threads = threads or os.cpu_count() or 1
    staged = C.c_uint64()
    _check(lib().or_dedisperse_tiled(_p(fb, C.c_float), c, t, _p(shifts, C.c_uint32), d, s,
                                     C.byref(ConfigC(*cfg)), threads, _p(out, C.c_float),
                                     C.byref(staged)), "dedisperse_tiled")
    return out


def config_valid(cfg, num_dms: int, s: int, max_block_items=1024, max_accumulators=256) -> bool:
    return bool(lib().or_config_valid(C.byref(ConfigC(*cfg)), num_dms, s, max_block_items,
                                      max_accumulators))


def count_loads(shifts: np.ndarray, s: int, cfg):
    shifts = np.ascontiguousarray(shifts, np.uint32)
    d, c = shifts.shape
    st, idl = C.c_uint64(), C.c_uint64()
    _check(lib().or_count_loads(_p(shifts, C.c_uint32), c, d, s, C.byref(ConfigC(*cfg)),
                                C.byref(st), C.byref(idl)), "count_loads")
    return st.value, idl.value


def enumerate_configs(num_dms: int, s: int, max_block_items=1024, max_accumulators=256):
    L = lib()
    n = L.or_enumerate_configs(num_dms, s, max_block_items, max_accumulators, None, 0)
    buf = (ConfigC * max(n, 1))()
    L.or_enumerate_configs(num_dms, s, max_block_items, max_accumulators, buf, n)
    return [(b.items_time, b.items_dm, b.work_time, b.work_dm) for b in buf[:n]]


# ------------------------------------------- reference I/O (oracle/_ref) --
def sigproc_bytes(data: np.ndarray, rate: int, fch1: float, foff: float) -> bytes:
    """A SIGPROC stream in the reference's subset (sigproc.cpp:201-250 writes
    the same layout): length-prefixed keywords, little-endian values, payload
    float32 time-major [samples][channels] with channel 0 the highest."""
    import struct
    kw = lambda k: struct.pack("<I", len(k)) + k.encode()
    t, c = data.shape
    head = (kw("HEADER_START") + kw("nchans") + struct.pack("<i", c) + kw("tsamp") +
            struct.pack("<d", 1.0 / rate) + kw("fch1") + struct.pack("<d", fch1) + kw("foff") +
            struct.pack("<d", foff) + kw("nbits") + struct.pack("<i", 32) + kw("nifs") +
            struct.pack("<i", 1) + kw("HEADER_END"))
    return head + np.ascontiguousarray(data, np.float32).tobytes()


def ref_parse_sigproc(stream: bytes):
    """The reference's parse_sigproc (sigproc.cpp:83-191) on a byte stream:
    (channel-major data lowest first, (f_min, channel_width, rate)) or, on
    format_error, (None, byte_offset)."""
    R = ref_lib()
    if R is None:
        raise RuntimeError("oracle/_ref is not built")
    ch, ns, bad = C.c_uint32(), C.c_uint64(), C.c_uint64()
    fm, cw, rate = C.c_double(), C.c_double(), C.c_uint32()
    st = R.ref_parse_sigproc(stream, len(stream), C.byref(ch), C.byref(ns), None, C.byref(bad),
                             C.byref(fm), C.byref(cw), C.byref(rate))
    if st == 4:
        return None, bad.value
    assert st == 0, st
    out = np.empty((ch.value, ns.value), np.float32)
    assert R.ref_parse_sigproc(stream, len(stream), C.byref(ch), C.byref(ns), _p(out, C.c_float),
                               C.byref(bad), C.byref(fm), C.byref(cw), C.byref(rate)) == 0
    return out, (fm.value, cw.value, rate.value)


def ref_tuning_roundtrip(text: str):
    """The reference's tuning_result_from_json then tuning_result_to_json
    (report_io.cpp:58-157): a summary of what it read and its own document,
    or None when oracle/_ref was built without a json.hpp."""
    R = ref_lib()
    if R is None or not hasattr(R, "ref_tuning_roundtrip"):
        return None
    n, best, dms, need = C.c_uint32(), C.c_uint64(), C.c_uint32(), C.c_uint64()
    cfg, g = (C.c_uint32 * 4)(), C.c_double()
    enc = text.encode()
    st = R.ref_tuning_roundtrip(enc, C.byref(n), C.byref(best), cfg, C.byref(g), C.byref(dms),
                                None, 0, C.byref(need))
    if st == 4:
        raise ValueError("reference rejected the document (format_error)")
    assert st == 0, st
    buf = C.create_string_buffer(need.value + 1)
    R.ref_tuning_roundtrip(enc, C.byref(n), C.byref(best), cfg, C.byref(g), C.byref(dms), buf,
                           need.value + 1, C.byref(need))
    return {"records": n.value, "best_index": best.value, "best_config": tuple(cfg),
            "best_gflops": g.value, "num_dms": dms.value, "json": buf.value.decode()}
