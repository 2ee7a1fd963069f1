"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

The reference (/root/reference/proj/include, header-only C++) is compiled in place by
``make -C oracle`` into oracle/_ref/libadfem_ref.so; this script calls it through oracle/pyoracle.py
and stores its outputs as small .npz files. Run in the build container (the GPU box has no
/root/reference): ``python tests/golden/make_golden.py``.

Cases mirror the reference's own fixtures (tests/test_support.hpp:27-39): benchmark_mesh(n) with
r=0.25 at the centre, benchmark_materials (SVK E=1 + linear E=10) and linear_materials(10),
benchmark_bcs(strain), random vectors from a fixed seed.
"""
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.pyoracle import Oracle, build  # noqa: E402

SVK_MIX = [(1, 1.0, 0.3), (0, 10.0, 0.3)]   # test_support.hpp:27-30
LINEAR = [(0, 1.0, 0.3), (0, 10.0, 0.3)]    # test_support.hpp:32-35

CASES = [
    # name, n, materials, strain
    ("q4_n2_svk", 2, SVK_MIX, 0.01),
    ("q4_n5_svk", 5, SVK_MIX, 0.02),
    ("q4_n8_linear", 8, LINEAR, 0.01),
    ("q4_n16_svk", 16, SVK_MIX, 0.01),
]


def make_case(R, name, n, mats, strain):
    coords, conn, phase = R.mesh2d(n, n)
    s = R.system(2, coords, conn, phase, mats, grid=(n, n, 0, 1.0, 1.0, 1.0))
    node, comp, val = R.bcs(2, n, n, 0, 1.0, strain)
    s.set_dirichlet(node, comp, val)
    rp, rows, cols = s.pattern()
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    u = rng.uniform(-0.01, 0.01, s.n)
    for nd, c, v in zip(node, comp, val):
        u[2 * nd + c] = v
    x = rng.uniform(-1.0, 1.0, s.n)
    res = s.residual(u)
    jac = s.jacobian(u)
    diag = s.diagonal(u)
    vals_el, rhs_el = s.eliminate(jac, res, u)
    mf = s.mf_apply(u, x)
    mfd = s.mf_diagonal(u)
    csr = s.csr_apply(vals_el, x)
    b = -rhs_el
    x_cg, rep_cg = s.solve(0, vals_el, b, method=0, precond=1, rtol=1e-10)
    x_gm, rep_gm = s.solve(0, vals_el, b, method=1, precond=1, rtol=1e-12)
    u_bvp, rep_bvp = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12)
    u_mf, rep_mf = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=1)
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"),
        n=n, strain=strain, mats=np.array(mats, np.float64), coords=coords, conn=conn, phase=phase,
        bc_node=node, bc_comp=comp, bc_val=val, row_ptr=rp, rows=rows, cols=cols, u=u, x=x,
        residual=res, jacobian=jac, diagonal=diag, elim_values=vals_el, elim_rhs=rhs_el,
        mf_apply=mf, mf_diagonal=mfd, csr_apply=csr,
        x_cg=x_cg, cg_iterations=rep_cg["iterations"], cg_history=rep_cg["residual_history"],
        x_gmres=x_gm, gmres_iterations=rep_gm["iterations"],
        u_bvp=u_bvp, bvp_iterations=rep_bvp["iterations"], bvp_norms=rep_bvp["residual_norms"],
        u_bvp_mf=u_mf, bvp_mf_iterations=rep_mf["iterations"],
    )
    print(name, "n_dof", s.n, "nnz", len(cols), "cg", rep_cg["iterations"], "newton", rep_bvp["iterations"])


def main():
    build()
    R = Oracle("ref")
    for case in CASES:
        make_case(R, *case)


if __name__ == "__main__":
    main()
