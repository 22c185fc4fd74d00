"""The C-ABI boundary: the product library loads, exports every symbol of
include/kifmm.h, maps errors onto the reference taxonomy, and has no CPU
fallback (GPU entry points fail loudly without a device)."""
import ctypes as C
import os
import re

import pytest

from conftest import gpu_available
from paper_2303_08394_b200 import DeviceError, InvalidArgument, _lib, fmm, generators, host

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kifmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kifmm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    names = _declared()
    assert len(names) >= 30
    lib = C.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/kifmm.h but not exported"
    assert set(names) == set(_lib.EXPORTED)


def test_no_torch_types_in_header():
    src = open(os.path.join(ROOT, "include", "kifmm.h")).read()
    assert "at::" not in src and "torch::" not in src
    assert 'extern "C"' in src


def test_status_mapping():
    with pytest.raises(InvalidArgument):
        host.encode((4, 0, 0), 2)
    assert "anchor" in _lib.last_error()


def test_version():
    assert b"sm_100a" in _lib.lib.kifmm_version()


def test_oracle_not_imported_by_product():
    import sys
    pkg = os.path.join(ROOT, "paper_2303_08394_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt, f
    assert "oracle" not in [m.split(".")[0] for m in sys.modules if m.startswith("paper_2303_08394_b200.")]


@pytest.mark.skipif(gpu_available(), reason="checks the no-device failure mode")
def test_gpu_plan_fails_loudly_without_device():
    pos, q = generators.sample("uniform-cube", 500, seed=0)
    with pytest.raises(DeviceError):
        fmm.Fmm(pos, fmm.FmmConfig(p=3, n_crit=20))


def test_null_plan_arguments_rejected():
    """Every evaluate entry point validates its arguments before touching a device (no CUDA needed):
    a null plan is KIFMM_E_INVALID_ARGUMENT, raised as the reference's InvalidArgument class."""
    import ctypes as C

    from paper_2303_08394_b200._lib import check, lib
    from paper_2303_08394_b200.errors import InvalidArgument

    buf = (C.c_float * 4)()
    ptrs = (C.c_void_p * 1)(C.cast(buf, C.c_void_p))
    pp = C.cast(ptrs, C.POINTER(C.c_void_p))
    with pytest.raises(InvalidArgument):
        check(lib.kifmm_gpu_evaluate(None, buf, buf, None, 1, None), "evaluate")
    with pytest.raises(InvalidArgument):
        check(lib.kifmm_gpu_evaluate_many(None, 1, pp, pp, None, 1), "evaluate_many")
    with pytest.raises(InvalidArgument):
        check(lib.kifmm_gpu_evaluate_device(None, buf, buf, None, 1, None), "evaluate_device")
