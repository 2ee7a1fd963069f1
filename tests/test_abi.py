"""CPU tests of the C-ABI library: it builds for sm_100a, loads, exports every symbol include/afem.h
declares, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "afem.h")
HEADERS = [HEADER, os.path.join(ROOT, "include", "afem_testing.h")]


def declared_symbols(headers=(HEADER,)):
    src = "".join(open(h).read() for h in headers)
    return sorted(set(re.findall(r"^(?:afem_status|const char\*|int32_t)\s+(afem_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2604_22087_b200", "csrc"), "-j8"], check=True,
                   stdout=subprocess.DEVNULL)
    import paper_2604_22087_b200 as afem
    return afem.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["afem_residual", "afem_jacobian", "afem_op_apply", "afem_solve", "afem_solve_bvp",
                 "afem_buffer_handoff", "afem_pattern", "afem_op_create_mf"]:
        assert must in syms
    assert len(syms) >= 50


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols(HEADERS) if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.afem_abi_version() == 1


def test_library_is_sm100a_only(lib):
    import paper_2604_22087_b200 as afem
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", afem.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_fibre_generator_matches_oracle(lib):
    import numpy as np

    import paper_2604_22087_b200 as afem
    from oracle.pyoracle import Oracle
    assert np.array_equal(afem.fibres(12345, 40), Oracle("restate").fibres(12345, 40))


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_22087_b200 as afem
    with pytest.raises(afem.AfemError):
        afem.Context(0)
