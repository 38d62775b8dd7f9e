"""CPU-side checks of the product boundary: the C-ABI library builds for sm_100a, loads without
a GPU, exports every symbol include/mobi_b200.h declares, and fails loudly (no CPU fallback)
when no device is present.  Host-side helpers mirror the reference's error behaviour."""
import re
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2602_20191_b200 import _lib
    _lib.build()
    return _lib.lib()


def header_symbols():
    text = (ROOT / "include" / "mobi_b200.h").read_text()
    return sorted(set(re.findall(r"MOBI_API\s+(?:int|const char\*)\s+(mobi_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ("mobi_layer_create", "mobi_forward", "mobi_forward_masked", "mobi_route", "mobi_score",
              "mobi_permute_by_slice", "mobi_calibrate_threshold", "mobi_forward_host", "mobi_decompose"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2602_20191_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (mobi_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    for s in header_symbols():
        assert hasattr(lib, s)
    assert b"sm_100a" in lib.mobi_version()


def test_library_is_sm100a_only():
    from paper_2602_20191_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ptx = subprocess.run(["cuobjdump", "--list-ptx", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "compute_100." not in ptx.replace("compute_100a", "")


def test_tcgen05_and_tma_in_sass():
    from paper_2602_20191_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "no tcgen05.mma in the GEMM"
    assert "UTMALDG" in sass, "no TMA loads"
    assert "STTM" in sass and "LDTM" in sass, "no TMEM traffic"


def test_no_device_fails_loudly(lib):
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_20191_b200 import MobiError, MobiLayer
    import numpy as np
    with pytest.raises(MobiError):
        MobiLayer.from_stack(np.zeros((4, 8, 8), np.uint8), [2] * 4, np.ones(8), np.zeros(8), 8,
                             np.zeros((8, 2)), np.zeros(2), np.zeros((2, 3)), np.zeros(3))


def test_ratio_from_target_bits_mirror(orc):
    from paper_2602_20191_b200 import ratio_from_target_bits
    for t in (2.0, 2.5, 3.0, 4.0, 8.0):
        assert ratio_from_target_bits(t, [2, 2, 2, 2]) == orc.ratio_from_target_bits(t, [2, 2, 2, 2])
    with pytest.raises(ValueError, match="outside"):
        ratio_from_target_bits(1.5, [2, 2, 2, 2])


def test_joint_step_validates_like_the_reference(lib):
    """mobi_joint_step rejects bad schedules / slice layouts before touching a device (the reference's
    MOBI_CHECKs in schedule_value / gate_soft, trainer.hpp:52-56, router.hpp:79-81)."""
    import ctypes as C
    import numpy as np
    from paper_2602_20191_b200.layer import BudgetSchedule, _JointScalars
    sb = np.array([2, 2, 2, 2], np.int32)
    g = np.zeros(4)
    res = _JointScalars()
    dummy = C.c_void_p(16)  # never dereferenced: validation fails first
    for sched, t, bits, msg in [(BudgetSchedule(8, 3, 10, 0, 1e-3), 0, sb, b"outside [1,10]"),
                                (BudgetSchedule(8, 3, 10, 0, 1e-3), 11, sb, b"outside [1,10]"),
                                (BudgetSchedule(8, 0, 10, 3, 1e-3), 2, sb, b"exponential"),
                                (BudgetSchedule(8, 3, 10, 0, 1e-3), 2, np.array([4, 4, 2], np.int32), b"exceed"),
                                (BudgetSchedule(8, 3, 10, 0, 1e-3), 2, np.array([8], np.int32), b"slices")]:
        rc = lib.mobi_joint_step(dummy, 4, 8, 8, bits.ctypes.data, bits.size, g.ctypes.data, g.ctypes.data, dummy,
                                 dummy, dummy, dummy, 2, dummy, dummy, 3, C.byref(sched), t, 0, None, C.byref(res),
                                 None, None, None, None, None, None, None)
        assert rc == 1 and msg in lib.mobi_last_error(), (rc, lib.mobi_last_error())
