"""Pins the test shims (tests/cpp/shim: a minimal GoogleTest and Eigen, both absent from the image):
the reference's unit suite (proj/tests, compiled in place) built with them against the UNMODIFIED
reference headers must pass on the CPU, 160 / 160. The same sources and shims, built against the
drop-in header tree, are the GPU suite (test_gpu_ref_suite.py)."""
import os
import re
import subprocess

import pytest

EXE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "ref_suite_cpu")


@pytest.mark.skipif(not os.path.exists(EXE), reason="ref_suite_cpu not built (needs the reference tree)")
def test_reference_suite_with_shims_on_cpu():
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    m = re.search(r"\[==========\] (\d+) tests ran\.\n\[  PASSED  \] (\d+) tests\.", p.stdout)
    assert m and int(m.group(1)) == 160 and int(m.group(2)) == 160 and p.returncode == 0, p.stdout[-4000:]
