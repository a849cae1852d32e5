"""ctypes binding of libwavehop_b200.so (the C ABI in include/wavehop_b200.h).

The library is built in-tree by ``paper_2408_14302_b200.build``.  There is no CPU
fallback: if the shared library is missing or no CUDA device is present, every entry
point raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, EmptySignal, InvalidHop, InvalidScale

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwavehop_b200.so")
# tools only: WH_DIAG_LIB=1 loads the diagnostics build (build.py --diag)
if os.environ.get("WH_DIAG_LIB") == "1":
    LIB_PATH = os.path.join(HERE, "libwavehop_b200_diag.so")

WH_OK = 0
WH_E_INVALID_HOP = 1
WH_E_INVALID_SCALE = 2
WH_E_INVALID_ARG = 3
WH_E_EMPTY_SIGNAL = 4
WH_E_CUDA = 5
WH_E_NO_DEVICE = 6
WH_E_UNSUPPORTED = 7
WH_E_OOM = 8

WAVELETS = {"cmor": 0, "rmor": 1}
OUTPUTS = {"complex": 0, "abs": 1, "power": 2, "log_db": 3, "log1p": 4}
NORMS = {None: 0, "none": 0, "minmax": 1, "render": 2, "render_noflip": 3}
ENGINES = {"auto": 0, "simt": 1, "umma": 2}
ENGINE_NAMES = {v: k for k, v in ENGINES.items()}

# every symbol include/wavehop_b200.h declares: name -> (restype, argtypes)
_i32, _i64, _d, _p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)
SIGNATURES = {
    "wh_abi_version": (ctypes.c_int, []),
    "wh_last_error": (ctypes.c_char_p, []),
    "wh_half_width": (ctypes.c_int, [_d, _d, _d, _pi64]),
    "wh_frame_count": (ctypes.c_int, [_i64, _i64, _pi64]),
    "wh_plan_create": (ctypes.c_int, [ctypes.POINTER(_p), ctypes.c_int, _p, _i32, _d, _d, _d, _i32,
                                      _i64, _i64, _i64, _i32, _i32, _i32]),
    "wh_plan_destroy": (ctypes.c_int, [_p]),
    "wh_plan_frames": (ctypes.c_int, [_p, _pi64]),
    "wh_plan_engine": (ctypes.c_int, [_p, _pi32]),
    "wh_plan_out_bytes": (ctypes.c_int, [_p, _i64, _pi64]),
    "wh_plan_launches": (ctypes.c_int, [_p, _i64, _pi64]),
    "wh_plan_mma_flops": (ctypes.c_int, [_p, _i64, ctypes.POINTER(ctypes.c_double)]),
    "wh_plan_taps": (ctypes.c_int, [_p, _i32, _p, _p, _i64, _pi64]),
    "wh_plan_profile": (ctypes.c_int, [_p, _i32, _p, _i32]),
    "wh_plan_trace": (ctypes.c_int, [_p, _i32, _p, _i32]),
    "wh_execute": (ctypes.c_int, [_p, _p, _i64, _i64, _p, _p]),
    "wh_execute_host": (ctypes.c_int, [_p, _p, _i64, _p]),
    "wh_strided_correlate": (ctypes.c_int, [ctypes.c_int, _p, _i64, _p, _p, _i64, _i64, _i64, _p, _p]),
    "wh_strided_correlate_symmetric": (ctypes.c_int, [ctypes.c_int, _p, _i64, _p, _p, _i64, _i64, _i64,
                                                      _p, _p]),
    "wh_decimate": (ctypes.c_int, [ctypes.c_int, _p, _i64, _i64, _i64, _i64, _i32, _p, _i64, _p]),
    "wh_render_u8": (ctypes.c_int, [ctypes.c_int, _p, _i64, _i64, _i64, _i32, _p, _p]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raise DeviceError if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceError(
                    f"{path} is not built; run `python -m paper_2408_14302_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().wh_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a WH_E_* code onto the reference's exception types (errors.py)."""
    if rc == WH_OK:
        return
    msg = last_error()
    if rc == WH_E_INVALID_HOP:
        raise InvalidHop(msg)
    if rc == WH_E_INVALID_SCALE:
        raise InvalidScale(msg)
    if rc == WH_E_EMPTY_SIGNAL:
        raise EmptySignal(msg)
    if rc == WH_E_INVALID_ARG:
        raise ValueError(msg)
    raise DeviceError(f"libwavehop_b200 error {rc}: {msg}")
