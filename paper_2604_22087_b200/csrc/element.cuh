// Device element math (fp64): quad4 / hex8 geometry at the 2x2(x2) Gauss points, constitutive
// laws, and the three per-quadrature-point products the assembly kernels need:
//   residual rows   f_a  = sum_q w detJ  P(F)     : grad N_a            (element.hpp:68-125)
//   JVP rows        df_a = sum_q w detJ  dP[dF]   : grad N_a            (backend.hpp:135-145, Dual<1>)
//   tangent blocks  K_ab = sum_q w detJ  grad N_a . A(F) . grad N_b     (assembly.hpp:144-173, Dual<8>)
// The reference obtains tangents by forward AD through the residual kernel; here they are
// hand-derived closed forms (SVK: K_ab = d_ab gSg + lam (F g_a)(F g_b)^T + mu (FF^T)(g_a.g_b)
// + mu (F g_b)(F g_a)^T), checked against the AD oracle to 1e-12 relative in tests/.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace afem {

template <int D> struct EL;
template <> struct EL<2> { static constexpr int npe = 4, nq = 4, nd = 8; };
template <> struct EL<3> { static constexpr int npe = 8, nq = 8, nd = 24; };

enum : int { MODEL_LINEAR = 0, MODEL_SVK = 1 };

// Per-phase material constants, precomputed on the host with the reference's formulas
// (material.hpp:20-21 for lambda/mu; material.hpp:35-38 for the Hooke constants).
struct DMat {
  int model;
  double E, nu;
  double lam, mu;        // Material::lambda(), Material::mu()
  double c11, c12, c33;  // stress_linear constants
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

// First Piola-Kirchhoff stress P at displacement gradient H; err |= ERR_INVERTED on det F <= 0.
template <int D>
__device__ __forceinline__ void piola(const DMat& m, const double (&H)[D][D], double (&P)[D][D], int& err) {
  if (m.model == MODEL_LINEAR) {
    stress_linear<D>(m, H, P);
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

// Directional derivative dP[dH] at displacement gradient H (the Dual<1> JVP of backend.hpp:142).
template <int D>
__device__ __forceinline__ void piola_jvp(const DMat& m, const double (&H)[D][D], const double (&dH)[D][D],
                                          double (&dP)[D][D]) {
  if (m.model == MODEL_LINEAR) {
    stress_linear<D>(m, dH, dP);
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

// Per-quadrature-point tangent context: for SVK the deformation gradient F, S and F F^T; for the
// linear law (lam, mu) = (c12, c33) and F = I, S = 0.
template <int D>
struct TangentQP {
  double F[D][D], S[D][D], FFt[D][D];
  double lam, mu;
  bool linear;
};

template <int D>
__device__ __forceinline__ void tangent_qp(const DMat& m, const double (&H)[D][D], TangentQP<D>& t, int& err) {
  t.linear = m.model == MODEL_LINEAR;
  if (t.linear) {
    t.lam = m.c12;
    t.mu = m.c33;
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
  if (t.linear) {
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b)
        blk[a][b] = t.lam * gn[a] * gm[b] + t.mu * gm[a] * gn[b] + (a == b ? t.mu * gg : 0.0);
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
