// Device element math (fp64): quad4 / hex8 geometry at the 2x2(x2) Gauss points, constitutive
// laws, and the three per-quadrature-point products the assembly kernels need:
//   residual rows   f_a  = sum_q w detJ  P(F)     : grad N_a            (element.hpp:68-125)
//   JVP rows        df_a = sum_q w detJ  dP[dF]   : grad N_a            (backend.hpp:135-145, Dual<1>)
//   tangent blocks  K_ab = sum_q w detJ  grad N_a . A(F) . grad N_b     (assembly.hpp:144-173, Dual<8>)
// The reference obtains tangents by forward AD through the residual kernel; here they are
// hand-derived closed forms (SVK: K_ab = d_ab gSg + lam (F g_a)(F g_b)^T + mu (FF^T)(g_a.g_b)
// + mu (F g_b)(F g_a)^T; Neo-Hookean and J2 below), checked against the AD oracle to 1e-12
// relative in tests/. Neo-Hookean and J2 are the north star's config-3/4 laws; the reference has
// neither (its material.hpp:13 stops at SVK), so their oracle is the restatement (oracle/).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace afem {

template <int D> struct EL;
template <> struct EL<2> { static constexpr int npe = 4, nq = 4, nd = 8; };
template <> struct EL<3> { static constexpr int npe = 8, nq = 8, nd = 24; };

enum : int { MODEL_LINEAR = 0, MODEL_SVK = 1, MODEL_NEOHOOKE = 2, MODEL_J2 = 3 };

// Quadrature-point history slot (J2): plastic strain tensor [xx, yy, zz, yz, xz, xy], the
// equivalent plastic strain alpha, one pad word -> 64 bytes per qp, nq slots per element.
constexpr int kHist = 8;

// Per-phase material constants, precomputed on the host with the reference's formulas
// (material.hpp:20-21 for lambda/mu; material.hpp:35-38 for the Hooke constants).
struct DMat {
  int model;
  double E, nu;
  double lam, mu;        // Material::lambda(), Material::mu()
  double c11, c12, c33;  // stress_linear constants
  double kappa;          // bulk modulus lam + 2 mu / 3 (Neo-Hookean, J2)
  double sy, hh;         // J2: initial yield stress, linear isotropic hardening modulus
};

constexpr int kMaxMat = 16;

enum : int { ERR_DETJ = 1, ERR_INVERTED = 2, ERR_VALENCE = 4 };

__device__ __forceinline__ double gauss_coord(int bit) {
  return bit ? 0.57735026918962576451 : -0.57735026918962576451;
}

// Gauss point q of the 2x2 rule in the reference's counter-clockwise order
// (element.hpp:42-43); hex8 appends zeta = -g (q<4) then +g.
__device__ __forceinline__ void gauss_point(int q, double& xi, double& eta, double& zeta) {
  const int r = q & 3;
  xi = gauss_coord(r == 1 || r == 2);
  eta = gauss_coord(r >= 2);
  zeta = gauss_coord(q >= 4);
}

// Corner signs (element.hpp:22-23; hex8: the quad ring at z=-1 then z=+1).
__device__ __forceinline__ double corner_sx(int i) { return ((i & 3) == 1 || (i & 3) == 2) ? 1.0 : -1.0; }
__device__ __forceinline__ double corner_sy(int i) { return ((i & 3) >= 2) ? 1.0 : -1.0; }
__device__ __forceinline__ double corner_sz(int i) { return i >= 4 ? 1.0 : -1.0; }

// Physical shape-function gradients g[i][b] = dN_i/dx_b and w*detJ at Gauss point q.
// Returns false when detJ <= 0 (element_internal_force throws invalid_argument, element.hpp:87-88).
template <int D>
__device__ __forceinline__ bool qp_geometry(const double (&xc)[EL<D>::npe][D], int q,
                                            double (&g)[EL<D>::npe][D], double& wdet) {
  constexpr int npe = EL<D>::npe;
  double xi, eta, zeta;
  gauss_point(q, xi, eta, zeta);
  double dn[npe][D];
#pragma unroll
  for (int i = 0; i < npe; ++i) {
    const double sx = corner_sx(i), sy = corner_sy(i);
    if constexpr (D == 2) {
      dn[i][0] = 0.25 * sx * (1.0 + sy * eta);
      dn[i][1] = 0.25 * sy * (1.0 + sx * xi);
    } else {
      const double sz = corner_sz(i);
      dn[i][0] = 0.125 * sx * (1.0 + sy * eta) * (1.0 + sz * zeta);
      dn[i][1] = 0.125 * sy * (1.0 + sx * xi) * (1.0 + sz * zeta);
      dn[i][2] = 0.125 * sz * (1.0 + sx * xi) * (1.0 + sy * eta);
    }
  }
  double J[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < npe; ++i) s += dn[i][a] * xc[i][b];
      J[a][b] = s;
    }
  double Ji[D][D];
  double detJ;
  if constexpr (D == 2) {
    detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double inv = 1.0 / detJ;
    Ji[0][0] = J[1][1] * inv; Ji[0][1] = -J[0][1] * inv;
    Ji[1][0] = -J[1][0] * inv; Ji[1][1] = J[0][0] * inv;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    detJ = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double inv = 1.0 / detJ;
    Ji[0][0] = c00 * inv;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
    Ji[1][0] = c01 * inv;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
    Ji[2][0] = c02 * inv;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
  }
#pragma unroll
  for (int i = 0; i < npe; ++i)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) s += dn[i][a] * Ji[b][a];
      g[i][b] = s;
    }
  wdet = detJ;  // 2x2(x2) Gauss weights are 1
  return detJ > 0.0;
}

// Displacement gradient H[a][b] = sum_i u[D i + a] g[i][b].
template <int D>
__device__ __forceinline__ void grad_u(const double (&ue)[EL<D>::nd], const double (&g)[EL<D>::npe][D],
                                       double (&H)[D][D]) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < EL<D>::npe; ++i) s += ue[D * i + a] * g[i][b];
      H[a][b] = s;
    }
}

template <int D>
__device__ __forceinline__ double det(const double (&F)[D][D]) {
  if constexpr (D == 2) return F[0][0] * F[1][1] - F[0][1] * F[1][0];
  else
    return F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
           F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
}

// Linear elastic stress from the displacement gradient (small strain; plane strain in 2D):
// stress_linear (material.hpp:33-40) and its 3D isotropic twin.
template <int D>
__device__ __forceinline__ void stress_linear(const DMat& m, const double (&H)[D][D], double (&S)[D][D]) {
  if constexpr (D == 2) {
    const double exx = H[0][0], eyy = H[1][1], gxy = H[0][1] + H[1][0];
    S[0][0] = m.c11 * exx + m.c12 * eyy;
    S[1][1] = m.c12 * exx + m.c11 * eyy;
    S[0][1] = S[1][0] = m.c33 * gxy;
  } else {
    const double exx = H[0][0], eyy = H[1][1], ezz = H[2][2];
    S[0][0] = m.c11 * exx + m.c12 * eyy + m.c12 * ezz;
    S[1][1] = m.c12 * exx + m.c11 * eyy + m.c12 * ezz;
    S[2][2] = m.c12 * exx + m.c12 * eyy + m.c11 * ezz;
    S[1][2] = S[2][1] = m.c33 * (H[1][2] + H[2][1]);
    S[0][2] = S[2][0] = m.c33 * (H[0][2] + H[2][0]);
    S[0][1] = S[1][0] = m.c33 * (H[0][1] + H[1][0]);
  }
}

// SVK second Piola-Kirchhoff stress S(F) (material.hpp:49-69). Returns false if det F <= 0.
template <int D>
__device__ __forceinline__ bool stress_svk(const DMat& m, const double (&F)[D][D], double (&S)[D][D]) {
  if (!(det<D>(F) > 0.0)) return false;
  double E[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double c = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) c += F[k][a] * F[k][b];
      E[a][b] = 0.5 * (a == b ? c - 1.0 : c);
    }
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tr += E[a][a];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) S[a][b] = 2.0 * m.mu * E[a][b] + (a == b ? m.lam * tr : 0.0);
  return true;
}

// ---------------------------------------------------------------- Neo-Hookean (model 2)
// Compressible Neo-Hookean in the pow-only form the reference's Dual primitives support
// (dual.hpp:162-177 has sqrt and pow but no log):
//   psi = mu/2 (J^{-2/3} I1 - 3) + kappa/2 (J - 1)^2,   kappa = lam + 2 mu / 3
//   P   = c1 F + (c3 - c2) C,   C = cof F = J F^{-T},  c1 = mu J^{-2/3},
//         c2 = (mu/3) I1 J^{-5/3},  c3 = kappa (J - 1).
// 2D is plane strain: F33 = 1 (I1 gains +1, J and C are the in-plane 2x2 determinant/cofactor).
template <int D>
struct NHQP {
  double F[D][D], C[D][D];
  double J, c1, c2, c3;
};

template <int D>
__device__ __forceinline__ bool nh_state(const DMat& m, const double (&H)[D][D], NHQP<D>& t) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) t.F[a][b] = H[a][b] + (a == b ? 1.0 : 0.0);
  const double (&F)[D][D] = t.F;
  if constexpr (D == 2) {
    t.C[0][0] = F[1][1]; t.C[0][1] = -F[1][0];
    t.C[1][0] = -F[0][1]; t.C[1][1] = F[0][0];
  } else {
    t.C[0][0] = F[1][1] * F[2][2] - F[1][2] * F[2][1];
    t.C[0][1] = F[1][2] * F[2][0] - F[1][0] * F[2][2];
    t.C[0][2] = F[1][0] * F[2][1] - F[1][1] * F[2][0];
    t.C[1][0] = F[0][2] * F[2][1] - F[0][1] * F[2][2];
    t.C[1][1] = F[0][0] * F[2][2] - F[0][2] * F[2][0];
    t.C[1][2] = F[0][1] * F[2][0] - F[0][0] * F[2][1];
    t.C[2][0] = F[0][1] * F[1][2] - F[0][2] * F[1][1];
    t.C[2][1] = F[0][2] * F[1][0] - F[0][0] * F[1][2];
    t.C[2][2] = F[0][0] * F[1][1] - F[0][1] * F[1][0];
  }
  double J = 0.0, I1 = (D == 2) ? 1.0 : 0.0;
#pragma unroll
  for (int b = 0; b < D; ++b) J += F[0][b] * t.C[0][b];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) I1 += F[a][b] * F[a][b];
  t.J = J;
  if (!(J > 0.0)) {
    t.c1 = t.c2 = t.c3 = 0.0;
    return false;
  }
  const double a23 = pow(J, -2.0 / 3.0);
  t.c1 = m.mu * a23;
  t.c2 = (m.mu / 3.0) * I1 * a23 / J;
  t.c3 = m.kappa * (J - 1.0);
  return true;
}

// ---------------------------------------------------------------- J2 plasticity (model 3)
// Small-strain J2 with linear isotropic hardening, radial return (history: plastic strain +
// equivalent plastic strain alpha, committed values read from hq; see history_commit).
//   s_tr = 2 mu dev(eps - eps_p),  q_tr = sqrt(3/2 s_tr:s_tr),  f = q_tr - (sy + hh alpha)
//   f > 0:  da = f / (3 mu + hh),  s = (1 - 3 mu da / q_tr) s_tr,  eps_p += da (3/2) s_tr / q_tr
//   sigma = kappa tr(eps - eps_p) I + s
// Consistent tangent: kappa I(x)I + 2 mu beta I_dev - 2 mu gbar n(x)n, n = s_tr/|s_tr|,
//   beta = 1 - 3 mu da / q_tr, gbar = 3 mu / (3 mu + hh) - 3 mu da / q_tr (elastic: 1, 0).
// 2D is plane strain (eps_zz = 0; the out-of-plane plastic strain is carried in the history).
struct J2QP {
  double sig[3][3];
  double n[3][3];
  double beta, gbar;
  double da, q;
  double ee_tr;  // trace of the elastic trial strain
  double str[3][3];
};

template <int D>
__device__ __forceinline__ void j2_state(const DMat& m, const double (&H)[D][D], const double* hq, J2QP& t) {
  double e[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) e[a][b] = (a < D && b < D) ? 0.5 * (H[a][b] + H[b][a]) : 0.0;
  double ep[6] = {0, 0, 0, 0, 0, 0}, alpha = 0.0;
  if (hq) {
#pragma unroll
    for (int k = 0; k < 6; ++k) ep[k] = hq[k];
    alpha = hq[6];
  }
  e[0][0] -= ep[0]; e[1][1] -= ep[1]; e[2][2] -= ep[2];
  e[1][2] -= ep[3]; e[2][1] -= ep[3];
  e[0][2] -= ep[4]; e[2][0] -= ep[4];
  e[0][1] -= ep[5]; e[1][0] -= ep[5];
  const double tr = e[0][0] + e[1][1] + e[2][2];
  t.ee_tr = tr;
  double ss = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      t.str[a][b] = 2.0 * m.mu * (e[a][b] - (a == b ? tr / 3.0 : 0.0));
      ss += t.str[a][b] * t.str[a][b];
    }
  const double q2 = 1.5 * ss;
  const double sY = m.sy + m.hh * alpha;
  double fac = 1.0;
  t.beta = 1.0; t.gbar = 0.0; t.da = 0.0; t.q = 0.0;
  if (q2 > sY * sY) {
    const double q = sqrt(q2);
    const double da = (q - sY) / (3.0 * m.mu + m.hh);
    fac = 1.0 - 3.0 * m.mu * da / q;
    t.beta = fac;
    t.gbar = 3.0 * m.mu / (3.0 * m.mu + m.hh) - 3.0 * m.mu * da / q;
    t.da = da;
    t.q = q;
  }
  const double inv_norm = (t.da > 0.0) ? 1.0 / sqrt(ss) : 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      t.sig[a][b] = fac * t.str[a][b] + (a == b ? m.kappa * tr : 0.0);
      t.n[a][b] = t.str[a][b] * inv_norm;
    }
}

// Updated history at (H, committed hq) -> out (8 words).
template <int D>
__device__ __forceinline__ void j2_commit(const DMat& m, const double (&H)[D][D], const double* hq, double* out) {
  J2QP t;
  j2_state<D>(m, H, hq, t);
  double h[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) h[k] = hq ? hq[k] : 0.0;
  if (t.da > 0.0) {
    const double f = t.da * 1.5 / t.q;
    h[0] += f * t.str[0][0]; h[1] += f * t.str[1][1]; h[2] += f * t.str[2][2];
    h[3] += f * t.str[1][2]; h[4] += f * t.str[0][2]; h[5] += f * t.str[0][1];
    h[6] += t.da;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) out[k] = h[k];
}

// First Piola-Kirchhoff stress P at displacement gradient H (hq: the qp's committed history,
// J2 only); err |= ERR_INVERTED on det F <= 0.
template <int D>
__device__ __forceinline__ void piola(const DMat& m, const double (&H)[D][D], double (&P)[D][D], int& err,
                                      const double* hq = nullptr) {
  if (m.model == MODEL_LINEAR) {
    stress_linear<D>(m, H, P);
    return;
  }
  if (m.model == MODEL_J2) {
    J2QP t;
    j2_state<D>(m, H, hq, t);
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) P[a][b] = t.sig[a][b];
    return;
  }
  if (m.model == MODEL_NEOHOOKE) {
    NHQP<D> t;
    if (!nh_state<D>(m, H, t)) err |= ERR_INVERTED;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) P[a][b] = t.c1 * t.F[a][b] + (t.c3 - t.c2) * t.C[a][b];
    return;
  }
  double F[D][D], S[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) F[a][b] = H[a][b] + (a == b ? 1.0 : 0.0);
  if (!stress_svk<D>(m, F, S)) err |= ERR_INVERTED;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += F[a][k] * S[k][b];
      P[a][b] = s;
    }
}

// Neo-Hookean directional derivative dP[dF] (see the block form in tangent_block).
template <int D>
__device__ __forceinline__ void nh_jvp(const DMat& m, const NHQP<D>& t, const double (&dF)[D][D], double (&dP)[D][D]) {
  double CdF = 0.0, FdF = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      CdF += t.C[a][b] * dF[a][b];
      FdF += t.F[a][b] * dF[a][b];
    }
  const double iJ = 1.0 / t.J;
  // dC = (1/J) [ (C:dF) C - C dF^T C ]
  double CdFt[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += t.C[a][k] * dF[b][k];
      CdFt[a][b] = s;
    }
  const double dc1 = -(2.0 / 3.0) * t.c1 * CdF * iJ;
  // c2 = (mu/3) I1 a / J with a = J^{-2/3}:  dc2 = (2 mu / 3)(a / J)(F:dF) - (5/3) c2 (C:dF) / J
  const double aJ = t.c1 / m.mu * iJ;  // a / J
  const double dc2v = (2.0 * m.mu / 3.0) * aJ * FdF - (5.0 / 3.0) * t.c2 * CdF * iJ;
  const double dc3 = m.kappa * CdF;
  const double k = t.c3 - t.c2;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int kk = 0; kk < D; ++kk) s += CdFt[a][kk] * t.C[kk][b];
      const double dC = iJ * (CdF * t.C[a][b] - s);
      dP[a][b] = t.c1 * dF[a][b] + dc1 * t.F[a][b] + k * dC + (dc3 - dc2v) * t.C[a][b];
    }
}

// Directional derivative dP[dH] at displacement gradient H (the Dual<1> JVP of backend.hpp:142).
template <int D>
__device__ __forceinline__ void piola_jvp(const DMat& m, const double (&H)[D][D], const double (&dH)[D][D],
                                          double (&dP)[D][D], const double* hq = nullptr) {
  if (m.model == MODEL_LINEAR) {
    stress_linear<D>(m, dH, dP);
    return;
  }
  if (m.model == MODEL_J2) {
    J2QP t;
    j2_state<D>(m, H, hq, t);
    double de[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) de[a][b] = (a < D && b < D) ? 0.5 * (dH[a][b] + dH[b][a]) : 0.0;
    const double tr = de[0][0] + de[1][1] + de[2][2];
    double nde = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) nde += t.n[a][b] * de[a][b];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        dP[a][b] = (a == b ? m.kappa * tr : 0.0) + 2.0 * m.mu * t.beta * (de[a][b] - (a == b ? tr / 3.0 : 0.0)) -
                   2.0 * m.mu * t.gbar * nde * t.n[a][b];
    return;
  }
  if (m.model == MODEL_NEOHOOKE) {
    NHQP<D> t;
    nh_state<D>(m, H, t);
    nh_jvp<D>(m, t, dH, dP);
    return;
  }
  double F[D][D], S[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) F[a][b] = H[a][b] + (a == b ? 1.0 : 0.0);
  stress_svk<D>(m, F, S);
  // dE = sym(F^T dF); dS = lam tr(dE) I + 2 mu dE; dP = dF S + F dS
  double dE[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += F[k][a] * dH[k][b] + dH[k][a] * F[k][b];
      dE[a][b] = 0.5 * s;
    }
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) tr += dE[a][a];
  double dS[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) dS[a][b] = 2.0 * m.mu * dE[a][b] + (a == b ? m.lam * tr : 0.0);
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += dH[a][k] * S[k][b] + F[a][k] * dS[k][b];
      dP[a][b] = s;
    }
}

// Per-quadrature-point tangent context.
//   linear: isotropic block with (lam, mu) = (c12, c33)
//   SVK:    F, S, F F^T
//   NH:     NHQP (F, cof F, J, c1..c3)
//   J2:     isotropic block with (kappa - 2 mu beta / 3, mu beta) plus -2 mu gbar (n g_n)(n g_m)^T
template <int D>
struct TangentQP {
  double F[D][D], S[D][D], FFt[D][D];
  double n[3][3];
  double lam, mu, g2;
  int model;
  bool iso;  // isotropic block form (linear, J2)
  NHQP<D> nh;
  double kappa, mu0;
  double k1, k2, k3;  // Neo-Hookean block coefficients (below), once per Gauss point
};

template <int D>
__device__ __forceinline__ void tangent_qp(const DMat& m, const double (&H)[D][D], TangentQP<D>& t, int& err,
                                           const double* hq = nullptr) {
  t.model = m.model;
  t.iso = m.model == MODEL_LINEAR || m.model == MODEL_J2;
  t.g2 = 0.0;
  if (m.model == MODEL_LINEAR) {
    t.lam = m.c12;
    t.mu = m.c33;
    return;
  }
  if (m.model == MODEL_J2) {
    J2QP j;
    j2_state<D>(m, H, hq, j);
    t.mu = m.mu * j.beta;
    t.lam = m.kappa - 2.0 * t.mu / 3.0;
    t.g2 = 2.0 * m.mu * j.gbar;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t.n[a][b] = j.n[a][b];
    return;
  }
  if (m.model == MODEL_NEOHOOKE) {
    if (!nh_state<D>(m, H, t.nh)) err |= ERR_INVERTED;
    t.kappa = m.kappa;
    t.mu0 = m.mu;
    const double iJ = 1.0 / t.nh.J;  // hoisted out of the per-block work (same expressions, same values)
    t.k1 = (2.0 / 3.0) * t.nh.c1 * iJ;
    t.k2 = (t.nh.c3 - t.nh.c2) * iJ;
    t.k3 = t.kappa + (5.0 / 3.0) * t.nh.c2 * iJ;
    return;
  }
  t.lam = m.lam;
  t.mu = m.mu;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) t.F[a][b] = H[a][b] + (a == b ? 1.0 : 0.0);
  if (!stress_svk<D>(m, t.F, t.S)) err |= ERR_INVERTED;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += t.F[a][k] * t.F[b][k];
      t.FFt[a][b] = s;
    }
}

// Tangent block K[(n,a),(m,b)] contribution at one quadrature point (without w detJ).
template <int D>
__device__ __forceinline__ void tangent_block(const TangentQP<D>& t, const double (&gn)[D], const double (&gm)[D],
                                              double (&blk)[D][D]) {
  double gg = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) gg += gn[k] * gm[k];
  if (t.iso) {
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        blk[a][b] = t.lam * gn[a] * gm[b] + t.mu * gm[a] * gn[b] + (a == b ? t.mu * gg : 0.0);
    if (t.g2 != 0.0) {
      double ngn[D], ngm[D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          s1 += t.n[a][k] * gn[k];
          s2 += t.n[a][k] * gm[k];
        }
        ngn[a] = s1; ngm[a] = s2;
      }
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) blk[a][b] -= t.g2 * ngn[a] * ngm[b];
    }
    return;
  }
  if (t.model == MODEL_NEOHOOKE) {
    // dF = e_b g_m^T contracted with g_n (derivation in DESIGN.md §Constitutive):
    // blk = c1 gg I - (2/3)(c1/J)[(F g_n)(C g_m)^T + (C g_n)(F g_m)^T]
    //       + ((c3 - c2)/J)[(C g_n)(C g_m)^T - (C g_m)(C g_n)^T] + (kappa + (5/3) c2 / J)(C g_n)(C g_m)^T
    const NHQP<D>& h = t.nh;
    double Fgn[D], Fgm[D], Cgn[D], Cgm[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        s1 += h.F[a][k] * gn[k];
        s2 += h.F[a][k] * gm[k];
        s3 += h.C[a][k] * gn[k];
        s4 += h.C[a][k] * gm[k];
      }
      Fgn[a] = s1; Fgm[a] = s2; Cgn[a] = s3; Cgm[a] = s4;
    }
    const double k1 = t.k1, k2 = t.k2, k3 = t.k3;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        blk[a][b] = (a == b ? h.c1 * gg : 0.0) - k1 * (Fgn[a] * Cgm[b] + Cgn[a] * Fgm[b]) +
                    k2 * (Cgn[a] * Cgm[b] - Cgm[a] * Cgn[b]) + k3 * Cgn[a] * Cgm[b];
    return;
  }
  double Fgn[D], Fgm[D], Sgm[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      s1 += t.F[a][k] * gn[k];
      s2 += t.F[a][k] * gm[k];
      s3 += t.S[a][k] * gm[k];
    }
    Fgn[a] = s1; Fgm[a] = s2; Sgm[a] = s3;
  }
  double gSg = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) gSg += gn[k] * Sgm[k];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b)
      blk[a][b] = (a == b ? gSg : 0.0) + t.lam * Fgn[a] * Fgm[b] + t.mu * t.FFt[a][b] * gg + t.mu * Fgm[a] * Fgn[b];
}

}  // namespace afem
