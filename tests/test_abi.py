"""The C-ABI library without a GPU: it builds, loads, exports every symbol the header
declares, and its host-only entry points and error paths behave like the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
from oracle import oracle as O
from paper_2408_14302_b200 import _lib, synth

HEADER = os.path.join(REPO, "include", "wavehop_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(wh_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_functions()
    for must in ("wh_plan_create", "wh_execute", "wh_execute_host", "wh_half_width",
                 "wh_strided_correlate", "wh_strided_correlate_symmetric", "wh_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(built_lib):
    lib = ctypes.CDLL(built_lib)
    for name in declared_functions():
        assert hasattr(lib, name), name
    # and the ctypes binding covers exactly the header
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_abi_version(built_lib):
    assert _lib.load().wh_abi_version() == 2


def test_half_width_matches_oracle(built_lib):
    lib = _lib.load()
    out = ctypes.c_int64()
    for cid in range(1, 6):
        for s in synth.config_scales(cid):
            assert lib.wh_half_width(float(s), 1.5, 6.0, ctypes.byref(out)) == 0
            assert out.value == O.half_width(float(s))
    assert lib.wh_half_width(0.0, 1.5, 6.0, ctypes.byref(out)) == _lib.WH_E_INVALID_SCALE
    assert "scale" in _lib.last_error()
    assert lib.wh_half_width(float("nan"), 1.5, 6.0, ctypes.byref(out)) == _lib.WH_E_INVALID_SCALE


def test_frame_count_and_errors(built_lib):
    lib = _lib.load()
    f = ctypes.c_int64()
    assert lib.wh_frame_count(160000, 128, ctypes.byref(f)) == 0 and f.value == 1250
    assert lib.wh_frame_count(1001, 64, ctypes.byref(f)) == 0 and f.value == 16
    assert lib.wh_frame_count(10, 0, ctypes.byref(f)) == _lib.WH_E_INVALID_HOP
    assert lib.wh_frame_count(0, 4, ctypes.byref(f)) == _lib.WH_E_EMPTY_SIGNAL
    with pytest.raises(Exception) as ei:
        _lib.check(_lib.WH_E_INVALID_HOP)
    assert isinstance(ei.value, _lib.InvalidHop)


def test_plan_validation_precedes_device(built_lib):
    """Argument errors are reported exactly like the reference even without a device."""
    lib = _lib.load()
    h = ctypes.c_void_p()
    sc = np.array([1.0, 2.0])
    p = sc.ctypes.data_as(ctypes.c_void_p)
    args = (1.0, 1.5, 6.0, 0, 64, 1000, 1, 1, 0, 0)
    rc = lib.wh_plan_create(ctypes.byref(h), 0, p, 2, 1.0, 1.5, 6.0, 0, 0, 1000, 1, 1, 0, 0)
    assert rc == _lib.WH_E_INVALID_HOP
    bad = np.array([2.0, 1.0])
    rc = lib.wh_plan_create(ctypes.byref(h), 0, bad.ctypes.data_as(ctypes.c_void_p), 2, *args)
    assert rc == _lib.WH_E_INVALID_ARG
    neg = np.array([-1.0, 1.0])
    rc = lib.wh_plan_create(ctypes.byref(h), 0, neg.ctypes.data_as(ctypes.c_void_p), 2, *args)
    assert rc == _lib.WH_E_INVALID_SCALE
    rc = lib.wh_plan_create(ctypes.byref(h), 0, p, 2, 1.0, 1.5, 2.0, 0, 64, 1000, 1, 1, 0, 0)
    assert rc == _lib.WH_E_INVALID_ARG  # support_radius < 3 (wavelet.py:52)
    rc = lib.wh_plan_create(ctypes.byref(h), 0, p, 2, 1.0, 1.5, 6.0, 0, 64, 0, 1, 1, 0, 0)
    assert rc == _lib.WH_E_EMPTY_SIGNAL
    rc = lib.wh_plan_create(ctypes.byref(h), 0, p, 2, 1.0, 1.5, 6.0, 0, 64, 1000, 1, 0, 1, 0)
    assert rc == _lib.WH_E_INVALID_ARG  # min-max needs a real output


def test_no_cpu_fallback_without_device(built_lib):
    """With no CUDA device visible the product path fails loudly (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2408_14302_b200 as wh

    with pytest.raises(wh.DeviceError):
        wh.cwth_batch(np.zeros((1, 100), np.float32), [1.0, 2.0], hop=4)
    sig = wh.SignalBuffer(np.zeros(64), 16000.0)
    with pytest.raises(wh.DeviceError):
        wh.cwth_strided(sig, wh.ScaleGrid([1.0]), hop=8)
    # validation still happens first, on the host, with the reference's exception types
    with pytest.raises(wh.InvalidHop):
        wh.cwth_strided(sig, wh.ScaleGrid([1.0]), hop=0)
    with pytest.raises(wh.InvalidScale):
        wh.sample_wavelet(wh.MorletParams(), 0.0)


def test_package_never_imports_oracle():
    """The product package does not reference oracle/ anywhere (task ③)."""
    pkg = os.path.join(REPO, "paper_2408_14302_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "libwh_oracle" not in text, f
