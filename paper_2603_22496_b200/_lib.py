"""ctypes binding of libkkb.so (include/kkb.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback:
if the library or a CUDA device is missing, every product entry point
raises ``DeviceError`` instead of computing something else.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# KKB_LIB selects an alternative in-tree build (tuning variants under variants/)
_DEFAULT_LIB_PATH = os.path.join(_HERE, "libkkb.so")
LIB_PATH = os.environ.get("KKB_LIB") or _DEFAULT_LIB_PATH

P = ctypes.c_void_p
I = ctypes.c_int
LL = ctypes.c_longlong
D = ctypes.c_double
F = ctypes.c_float

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "kkb_version": [],
    "kkb_last_error": [],
    "kkb_device_info": [P, P, P],
    "kkb_launch_count": [],
    "kkb_take_device_error": [P],
    "kkb_build_kk_luts": [D, D, I, D, D, I, P, P, I, P, P, I, D, P, P, P, P, P],
    "kkb_kk": [P, I, I, I, P, P, P, P, I, I, P, D, D, I, P, I, I, LL, LL, P, P, P],
    "kkb_kk_plan_create": [P, P, P, P, I, I, I, I, I, P, D, D, I, P, P],
    "kkb_kk_plan_run": [P, P, I, LL, P, I, LL, P, P, P],
    "kkb_kk_plan_run_ex": [P, P, I, LL, P, I, LL, P, P, I, P],
    "kkb_kk_plan_run_strided": [P, P, I, LL, LL, P, I, LL, P, P, I, P],
    "kkb_kk_plan_run_scatter": [P, P, I, LL, P, I, LL, I, LL, P],
    "kkb_kk_plan_run_sets": [P, P, I, LL, I, P, P, I, LL, LL, P, P, I, P],
    "kkb_kk_plan_window": [P],
    "kkb_kk_last_instance": [],
    "kkb_kk_plan_window_check": [P],
    "kkb_kk_plan_tc_ksteps": [P],
    "kkb_decomposer_run_stage": [P, I, P, I, P, P],
    "kkb_decomposer_run_planes": [P, P, I, P, P, P, P, P],
    "kkb_kk_plan_run_planes": [P, P, P, P, P, I, P, I, LL, P, P, I, P],
    "kkb_tc_planes_bytes": [I, I, I],
    "kkb_analytic_signal_stage": [I, P, LL, I, P, P, P],
    "kkb_kk_plan_destroy": [P],
    "kkb_kk_taps": [P, P, P, P, I, I, I, I, I, D, D, I, P, P],
    "kkb_das": [P, I, I, I, P, P, P, I, P, P, P, P, P, D, P, D, D, I, I, I, P, I, P],
    "kkb_analytic_signal": [P, LL, I, P, P],
    "kkb_shear_and_sum": [P, I, I, I, P, P, I, D, D, P, P],
    "kkb_shear_plan_create": [P, P, I, I, I, D, D, P],
    "kkb_shear_plan_run": [P, P, I, P, P],
    "kkb_shear_plan_destroy": [P],
    "kkb_decomposer_create": [I, I, I, P, P, I, D, D, I, P],
    "kkb_decomposer_run": [P, P, I, P, P],
    "kkb_decomposer_run_i16": [P, P, I, P, P],
    "kkb_decomposer_run_scatter": [P, P, I, I, P, I, LL, LL, P],
    "kkb_decomposer_set_pipeline": [P, I, I],
    "kkb_decomposer_symmetric_classes": [P],
    "kkb_decomposer_set_contraction": [P, I],
    "kkb_decomposer_contraction": [P],
    "kkb_decomposer_set_fused": [P, I],
    "kkb_decomposer_fused": [P],
    "kkb_decomposer_set_ring": [P, I, I],
    "kkb_decomposer_ring_error": [P, P],
    "kkb_decomposer_workspace_bytes": [P],
    "kkb_decomposer_destroy": [P],
    "kkb_log_compress": [P, P, I, LL, F, P, P],
    "kkb_compound": [P, I, LL, I, P, P],
    "kkb_render_traces": [P, I, I, I, P, P, P, LL, P, P, P, D, D, D, P, I, D, I, P],
    "kkb_kkrf_read_header": [ctypes.c_char_p, P],
    "kkb_kkrf_read_bytes": [ctypes.c_char_p, LL, LL, P, I, P],
    "kkb_kkrf_read_ensemble": [P, P, I, LL, P, I, P],
    "kkb_kkrf_write": [ctypes.c_char_p, P, P, P, P, LL, I, P],
    "kkb_max_f64": [P, LL, P, P],
    "kkb_gamma_match": [P, P, LL, D, D, D, P, P, P],
    "kkb_last_read_sample_max": [P, I, P, I, P, P, I, P, P, I, P, P],
    "kkb_ipc_alloc": [LL, P],
    "kkb_ipc_free": [P],
    "kkb_ipc_get_handle": [P, P],
    "kkb_ipc_open_handle": [P, P],
    "kkb_ipc_close_handle": [P],
}
_RESTYPES = {
    "kkb_kk_plan_tc_ksteps": LL,
    "kkb_tc_planes_bytes": LL,
    "kkb_version": ctypes.c_char_p,
    "kkb_last_error": ctypes.c_char_p,
    "kkb_launch_count": LL,
    "kkb_decomposer_workspace_bytes": LL,
}


class KKRFHeader(ctypes.Structure):
    """kkb_kkrf_header (include/kkb.h), natural C alignment."""

    _fields_ = [
        ("magic", ctypes.c_char * 4),
        ("version", ctypes.c_uint16),
        ("kind", ctypes.c_uint8),
        ("num_transmits", ctypes.c_uint32),
        ("num_channels", ctypes.c_uint32),
        ("num_samples", ctypes.c_uint32),
        ("sampling_frequency", ctypes.c_double),
        ("center_frequency", ctypes.c_double),
        ("sound_speed", ctypes.c_double),
        ("pitch", ctypes.c_double),
        ("start_time", ctypes.c_double),
        ("head_bytes", ctypes.c_longlong),
        ("file_bytes", ctypes.c_longlong),
    ]


KKB_OUT_C64 = 0
KKB_RUN_ACCUMULATE_INTENSITY = 1
KKB_MAX_DST = 8  # destinations of kkb_kk_plan_run_scatter
KKB_MAX_SETS = 8  # receive sets of kkb_kk_plan_run_sets
KKB_OUT_C128 = 1
KKB_DEVERR_KK_WINDOW = 1
KKB_CONTRACT_FMA, KKB_CONTRACT_TENSOR = 0, 1
# K5 instances (kkb_kk_last_instance)
KKB_KK_INST_DIRECT, KKB_KK_INST_SMALL, KKB_KK_INST_MID, KKB_KK_INST_BIG, KKB_KK_INST_BIG_FR, KKB_KK_INST_TC = range(6)
KKB_KK_INST_SETS = 16
KKB_KK_INST_NAMES = {0: "direct", 1: "small", 2: "mid", 3: "big", 4: "big_fr", 5: "tc"}

_lib = None


def load() -> ctypes.CDLL:
    """Load libkkb.so once; raise DeviceError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
            "this package has no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    variant = LIB_PATH != _DEFAULT_LIB_PATH  # tuning builds may predate newer entry points
    for name, args in SIGNATURES.items():
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, I)
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and map failures to exceptions."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st != 0:
        raise_for_status(st, name, lib.kkb_last_error().decode(errors="replace"))


def last_error() -> str:
    return load().kkb_last_error().decode(errors="replace")


def launch_count() -> int:
    """Kernel launches issued by libkkb in this process so far."""
    return int(load().kkb_launch_count())


def last_instance() -> int:
    """K5 instance the last gather launch of this process dispatched to
    (KKB_KK_INST_*; or-ed with KKB_KK_INST_SETS for the multi-set form)."""
    return int(load().kkb_kk_last_instance())


def take_device_error() -> int:
    """Read and clear the device-side error word (KKB_DEVERR_* bits)."""
    v = ctypes.c_int(0)
    call("kkb_take_device_error", ctypes.byref(v))
    return int(v.value)


def version() -> str:
    return load().kkb_version().decode()
