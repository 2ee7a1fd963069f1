"""tools/afem_bench — the GPU-backed bench CLI (the reference's `bench` subcommands, bench.hpp:189-406,
emitting the reference CSV schema) and its `verify` suite (verify.hpp:62-308 through the ABI)."""
import os
import subprocess

import pytest

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "build", "afem_bench")
HEADER = "experiment,dof,method,pc,operator,converged,iters,time_s,final_rres"

needs_exe = pytest.mark.skipif(not os.path.exists(EXE), reason="tools/build/afem_bench not built")


def run(*args, timeout=900):
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=timeout)


@needs_exe
def test_usage_errors_exit_2():
    """Exit codes follow bench_main.cpp:76-114 (2 = usage / configuration error); no GPU needed."""
    assert run().returncode == 2
    assert run("nope").returncode == 2
    assert run("spmv", "--materials", "rubber").returncode == 2
    assert run("spmv", "--dim", "4").returncode == 2


@needs_exe
@pytest.mark.gpu
@pytest.mark.parametrize("dim", ["2", "3"])
def test_verify_suite_passes(dim):
    p = run("verify", "--dim", dim)
    print(p.stdout, p.stderr)
    assert p.returncode == 0, p.stdout + p.stderr
    names = [ln.split()[0] for ln in p.stdout.splitlines()[1:]]
    assert names == ["fd_vs_tangent", "dense_equivalence", "operator_equivalence", "patch_test", "mms_convergence"]


@needs_exe
@pytest.mark.gpu
def test_csv_schema_and_rows():
    p = run("solvers", "--levels", "2", "--reps", "1", "--rtol", "1e-10", "--max-iter", "20000")
    assert p.returncode == 0, p.stderr
    lines = p.stdout.splitlines()
    assert lines[0].startswith("# afem_bench") and lines[1] == HEADER
    rows = [ln.split(",") for ln in lines[2:]]
    assert len(rows) == 2 * 9  # 2 meshes x {CG, GMRES, BICGSTAB} x {NONE, JACOBI, ILU0}
    assert {r[2] for r in rows} == {"CG", "GMRES", "BICGSTAB"} and {r[3] for r in rows} == {"NONE", "JACOBI", "ILU0"}
    cg_jacobi = [r for r in rows if r[2] == "CG" and r[3] == "JACOBI"]
    assert all(r[5] == "1" and float(r[8]) <= 1e-10 for r in cg_jacobi)
    p = run("newton", "--levels", "1", "--reps", "1")
    rows = [ln.split(",") for ln in p.stdout.splitlines()[2:]]
    assert p.returncode == 0 and [r[4] for r in rows] == ["EXPLICIT", "MATRIX_FREE"]
    assert all(r[5] == "1" for r in rows) and rows[0][6] == rows[1][6]  # same Newton count both kinds
    p = run("direct", "--levels", "2", "--reps", "1")
    rows = [ln.split(",") for ln in p.stdout.splitlines()[2:]]
    assert p.returncode == 0 and [r[2] for r in rows] == ["DIRECT_CHOL", "DIRECT_LU"] * 2
    assert all(r[5] == "1" and r[6] == "1" and float(r[8]) <= 1e-10 for r in rows)
    for cmd in ("spmv", "mfapply"):
        p = run(cmd, "--levels", "1", "--reps", "2")
        rows = [ln.split(",") for ln in p.stdout.splitlines()[2:]]
        assert p.returncode == 0 and len(rows) == 2 and all(r[6] == "100" for r in rows)
