"""The C++ drop-in check: tests/cpp/overlay_test (the reference's own headers compiled in place next
to the device path reached through include/adfem_b200/adfem.hpp with the reference's types).
Every PASS/FAIL line names the reference test it mirrors; see tests/cpp/overlay_test.cpp."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "overlay_test")


@pytest.mark.skipif(not os.path.exists(EXE), reason="overlay_test not built (needs the reference headers at build time)")
def test_cpp_overlay_against_reference():
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout
