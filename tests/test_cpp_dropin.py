"""The reference's own C++ hot-path calls side by side with the C++ drop-in shim
(include/mobi_b200.hpp over the C ABI): tests/cpp/dropin_test.cpp."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "tests" / "cpp" / "bin" / "dropin_test"


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not BIN.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=False)
    if not BIN.exists():
        pytest.skip("drop-in test binary not built (needs the reference headers at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr
