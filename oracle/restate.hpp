// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path (the parity oracle).
//
// Follows /root/reference/proj/include/adfem/*.hpp function by function; every routine cites the
// reference file:line it restates. The 2D quad4 branch reproduces the reference's floating-point
// expression order exactly (so it is pinned bit-for-bit against oracle/_ref, the reference compiled
// in place). The 3D hex8 branch is the natural twin the reference lacks (north_star configs 2-5):
// same conventions (dof interleave, strict centroid test, (batch, element) scatter order, symmetric
// elimination, AD tangents through Dual<8>, CG/GMRES semantics). Its parity is pinned by this
// restatement plus the property checks in tests/ (patch test, FD-vs-AD, rigid modes), not by a
// reference run.
//
// Never linked by the product. Compiled with -O2 -ffp-contract=off (no FMA contraction), the same
// flags oracle/Makefile uses for the reference build.
#ifndef ORC_RESTATE_HPP
#define ORC_RESTATE_HPP

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <numeric>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors (errors.hpp:10-38)
struct LeaseError : std::logic_error { using std::logic_error::logic_error; };
struct StaleEpochError : std::logic_error { using std::logic_error::logic_error; };
struct CapabilityError : std::logic_error { using std::logic_error::logic_error; };
struct FactorizationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvertedElementError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- dual numbers (dual.hpp:19-177)
template <int L>
struct Dual {
  double v = 0.0;
  std::array<double, L> d{};
  constexpr Dual() = default;
  constexpr Dual(double value) : v(value) {}  // NOLINT
};
template <int L> inline Dual<L> operator+(const Dual<L>& a, const Dual<L>& b) {
  Dual<L> r(a.v + b.v); for (int k = 0; k < L; ++k) r.d[k] = a.d[k] + b.d[k]; return r; }
template <int L> inline Dual<L> operator+(const Dual<L>& a, double b) { Dual<L> r = a; r.v += b; return r; }
template <int L> inline Dual<L> operator+(double a, const Dual<L>& b) { return b + a; }
template <int L> inline Dual<L> operator-(const Dual<L>& a) {
  Dual<L> r(-a.v); for (int k = 0; k < L; ++k) r.d[k] = -a.d[k]; return r; }
template <int L> inline Dual<L> operator-(const Dual<L>& a, const Dual<L>& b) {
  Dual<L> r(a.v - b.v); for (int k = 0; k < L; ++k) r.d[k] = a.d[k] - b.d[k]; return r; }
template <int L> inline Dual<L> operator-(const Dual<L>& a, double b) { Dual<L> r = a; r.v -= b; return r; }
template <int L> inline Dual<L> operator-(double a, const Dual<L>& b) {
  Dual<L> r(a - b.v); for (int k = 0; k < L; ++k) r.d[k] = -b.d[k]; return r; }
template <int L> inline Dual<L> operator*(const Dual<L>& a, const Dual<L>& b) {
  Dual<L> r(a.v * b.v); for (int k = 0; k < L; ++k) r.d[k] = a.d[k] * b.v + a.v * b.d[k]; return r; }
template <int L> inline Dual<L> operator*(const Dual<L>& a, double b) {
  Dual<L> r(a.v * b); for (int k = 0; k < L; ++k) r.d[k] = a.d[k] * b; return r; }
template <int L> inline Dual<L> operator*(double a, const Dual<L>& b) { return b * a; }
template <int L> inline Dual<L> operator/(const Dual<L>& a, const Dual<L>& b) {
  if (b.v == 0.0) throw std::domain_error("dual division by zero-valued denominator");
  const double inv = 1.0 / b.v; Dual<L> r(a.v * inv);
  for (int k = 0; k < L; ++k) r.d[k] = (a.d[k] - r.v * b.d[k]) * inv;
  return r; }
template <int L> inline Dual<L> operator/(const Dual<L>& a, double b) {
  const double inv = 1.0 / b; Dual<L> r(a.v * inv); for (int k = 0; k < L; ++k) r.d[k] = a.d[k] * inv; return r; }
template <int L> inline Dual<L>& operator+=(Dual<L>& a, const Dual<L>& b) { a = a + b; return a; }
// sqrt / pow(x, double) (dual.hpp:162-177): the only transcendental primitives the reference's Dual has.
template <int L> inline Dual<L> sqrt(const Dual<L>& a) {
  const double sv = std::sqrt(a.v);
  Dual<L> r(sv);
  const double g = 0.5 / sv;
  for (int k = 0; k < L; ++k) r.d[k] = g * a.d[k];
  return r;
}
template <int L> inline Dual<L> pow(const Dual<L>& a, double p) {
  Dual<L> r(std::pow(a.v, p));
  const double g = p * std::pow(a.v, p - 1.0);
  for (int k = 0; k < L; ++k) r.d[k] = g * a.d[k];
  return r;
}
inline double sqrt(double x) { return std::sqrt(x); }
inline double pow(double x, double p) { return std::pow(x, p); }
inline double value_of(double x) { return x; }
template <int L> inline double value_of(const Dual<L>& x) { return x.v; }

// ---------------------------------------------------------------- material (material.hpp:13-69)
// NEOHOOKE and J2 are the north star's config-3/4 laws; the reference stops at SVK (material.hpp:13).
enum Model { LINEAR = 0, SVK = 1, NEOHOOKE = 2, J2 = 3 };
constexpr int kHist = 8;  // J2 history words per Gauss point: eps_p [xx,yy,zz,yz,xz,xy], alpha, pad
struct Material {
  int model = LINEAR;
  double E = 1.0, nu = 0.3;
  double sigma_y = 0.0, hardening = 0.0;  // J2 only
  double kappa() const { return lambda() + 2.0 * mu() / 3.0; }
  double lambda() const { return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)); }  // material.hpp:20
  double mu() const { return E / (2.0 * (1.0 + nu)); }                        // material.hpp:21
  void validate() const {                                                     // material.hpp:23-26
    if (!(E > 0.0)) throw std::invalid_argument("material: E must be > 0");
    if (!(nu > -1.0 && nu < 0.5)) throw std::invalid_argument("material: nu must be in (-1, 0.5)");
    if (model < LINEAR || model > J2) throw std::invalid_argument("material: unsupported model");
    if (model == J2 && !(sigma_y > 0.0 && hardening >= 0.0))
      throw std::invalid_argument("material: J2 needs sigma_y > 0 and hardening >= 0");
  }
};

// ---------------------------------------------------------------- element geometry (element.hpp:16-54)
template <int D> struct ET;
template <> struct ET<2> { static constexpr int npe = 4, ndpe = 8, pairs = 64; };
template <> struct ET<3> { static constexpr int npe = 8, ndpe = 24, pairs = 576; };

struct GP { double xi, eta, zeta, w; };

// 2x2 rule in the reference's counter-clockwise order (element.hpp:42-43); 3D = that ring at
// zeta = -g then +g. 3x3 rule row-major (element.hpp:47-50); 3D adds zeta as the outer index.
inline const std::vector<GP>& gauss_rule(int dim, int p) {
  static const double g2 = 0.57735026918962576451, g3 = 0.77459666924148337704;
  static const double w0 = 5.0 / 9.0, w1 = 8.0 / 9.0;
  static const std::vector<GP> r2_2d = {{-g2, -g2, 0, 1.0}, {g2, -g2, 0, 1.0}, {g2, g2, 0, 1.0}, {-g2, g2, 0, 1.0}};
  static const std::vector<GP> r3_2d = {
      {-g3, -g3, 0, w0 * w0}, {0.0, -g3, 0, w1 * w0}, {g3, -g3, 0, w0 * w0},
      {-g3, 0.0, 0, w0 * w1}, {0.0, 0.0, 0, w1 * w1}, {g3, 0.0, 0, w0 * w1},
      {-g3, g3, 0, w0 * w0},  {0.0, g3, 0, w1 * w0},  {g3, g3, 0, w0 * w0}};
  static const std::vector<GP> r2_3d = [] {
    std::vector<GP> r;
    for (double z : {-g2, g2}) for (const GP& q : r2_2d) r.push_back({q.xi, q.eta, z, 1.0});
    return r;
  }();
  static const std::vector<GP> r3_3d = [] {
    std::vector<GP> r;
    const double zs[3] = {-g3, 0.0, g3}, ws[3] = {w0, w1, w0};
    for (int k = 0; k < 3; ++k) for (const GP& q : r3_2d) r.push_back({q.xi, q.eta, zs[k], q.w * ws[k]});
    return r;
  }();
  if (p == 2) return dim == 2 ? r2_2d : r2_3d;
  if (p == 3) return dim == 2 ? r3_2d : r3_3d;
  throw std::invalid_argument("gauss_rule: only 2x2 and 3x3 rules are provided");
}

// shape_quad4 (element.hpp:21-31); hex8 corners (-1,-1,-1),(1,-1,-1),(1,1,-1),(-1,1,-1), then z=+1.
inline void shape_grad(int dim, const GP& q, double dn[8][3]) {
  static const double sx[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
  static const double sy[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
  static const double sz[8] = {-1, -1, -1, -1, 1, 1, 1, 1};
  if (dim == 2) {
    for (int i = 0; i < 4; ++i) {
      dn[i][0] = 0.25 * sx[i] * (1.0 + sy[i] * q.eta);
      dn[i][1] = 0.25 * sy[i] * (1.0 + sx[i] * q.xi);
    }
  } else {
    for (int i = 0; i < 8; ++i) {
      dn[i][0] = 0.125 * sx[i] * (1.0 + sy[i] * q.eta) * (1.0 + sz[i] * q.zeta);
      dn[i][1] = 0.125 * sy[i] * (1.0 + sx[i] * q.xi) * (1.0 + sz[i] * q.zeta);
      dn[i][2] = 0.125 * sz[i] * (1.0 + sx[i] * q.xi) * (1.0 + sy[i] * q.eta);
    }
  }
}

// ---------------------------------------------------------------- element kernel (element.hpp:68-125)
// coords: npe*D doubles; u, out: ndpe values.
// Small-strain J2 radial return at one Gauss point (the north star's config-4 law): committed
// history h (kHist words, may be null = virgin), total strain eps (3x3, plane strain in 2D) ->
// stress sig; h_new (may be null) receives the updated history. The yield test is decided on
// values (like the reference's value-only comparisons, dual.hpp:137-160) and sqrt is taken only
// on the plastic branch, so the AD tangent is the consistent tangent.
template <class T>
void j2_stress(const Material& mat, const T (&eps)[3][3], const double* h, T (&sig)[3][3], double* h_new) {
  const double mu = mat.mu(), kappa = mat.kappa();
  double ep[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, alpha = 0.0;
  if (h) {
    ep[0][0] = h[0]; ep[1][1] = h[1]; ep[2][2] = h[2];
    ep[1][2] = ep[2][1] = h[3]; ep[0][2] = ep[2][0] = h[4]; ep[0][1] = ep[1][0] = h[5];
    alpha = h[6];
  }
  T ee[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) ee[a][b] = eps[a][b] - ep[a][b];
  const T tr = ee[0][0] + ee[1][1] + ee[2][2];
  T str[3][3];
  T ss(0.0);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      str[a][b] = 2.0 * mu * (a == b ? ee[a][b] - tr / 3.0 : ee[a][b]);
      ss += str[a][b] * str[a][b];
    }
  const T q2 = 1.5 * ss;
  const double sY = mat.sigma_y + mat.hardening * alpha;
  T fac(1.0);
  double da_v = 0.0, q_v = 0.0;
  if (value_of(q2) > sY * sY) {
    const T q = sqrt(q2);
    const T da = (q - sY) / (3.0 * mu + mat.hardening);
    fac = 1.0 - 3.0 * mu * da / q;
    da_v = value_of(da);
    q_v = value_of(q);
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) sig[a][b] = a == b ? fac * str[a][b] + kappa * tr : fac * str[a][b];
  if (h_new) {
    double hn[kHist];
    for (int k = 0; k < kHist; ++k) hn[k] = h ? h[k] : 0.0;
    if (da_v > 0.0) {
      const double f = da_v * 1.5 / q_v;
      hn[0] += f * value_of(str[0][0]); hn[1] += f * value_of(str[1][1]); hn[2] += f * value_of(str[2][2]);
      hn[3] += f * value_of(str[1][2]); hn[4] += f * value_of(str[0][2]); hn[5] += f * value_of(str[0][1]);
      hn[6] += da_v;
    }
    for (int k = 0; k < kHist; ++k) h_new[k] = hn[k];
  }
}

// hist: the element's committed Gauss-point history (nq * kHist words, J2 only; may be null).
// hist_new: if non-null, receives the updated history (history commit; J2 only).
template <int D, class T>
void element_internal_force(const double* coords, const Material& mat, int gauss_points,
                            const T* u, T* out, const double* hist = nullptr, double* hist_new = nullptr) {
  int qi = -1;
  constexpr int npe = ET<D>::npe, nd = ET<D>::ndpe;
  for (int k = 0; k < nd; ++k) out[k] = T(0.0);
  for (const GP& gp : gauss_rule(D, gauss_points)) {
    ++qi;
    double dn[8][3];
    shape_grad(D, gp, dn);
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < npe; ++i)
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) J[a][b] += dn[i][a] * coords[i * D + b];
    double detJ, Jinv[3][3];
    if constexpr (D == 2) {
      detJ = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      if (!(detJ > 0.0)) throw std::invalid_argument("element_internal_force: non-positive element Jacobian");
      const double inv = 1.0 / detJ;
      Jinv[0][0] = J[1][1] * inv; Jinv[0][1] = -J[0][1] * inv;
      Jinv[1][0] = -J[1][0] * inv; Jinv[1][1] = J[0][0] * inv;
    } else {
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      detJ = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      if (!(detJ > 0.0)) throw std::invalid_argument("element_internal_force: non-positive element Jacobian");
      const double inv = 1.0 / detJ;
      Jinv[0][0] = c00 * inv;
      Jinv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
      Jinv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
      Jinv[1][0] = c01 * inv;
      Jinv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
      Jinv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
      Jinv[2][0] = c02 * inv;
      Jinv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
      Jinv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
    }
    double g[8][3];
    for (int i = 0; i < npe; ++i)
      for (int b = 0; b < D; ++b) {
        if constexpr (D == 2) g[i][b] = dn[i][0] * Jinv[b][0] + dn[i][1] * Jinv[b][1];
        else g[i][b] = dn[i][0] * Jinv[b][0] + dn[i][1] * Jinv[b][1] + dn[i][2] * Jinv[b][2];
      }
    const double wdet = gp.w * detJ;

    if (mat.model == LINEAR) {
      const double c = mat.E / ((1.0 + mat.nu) * (1.0 - 2.0 * mat.nu));  // material.hpp:35-38
      const double c11 = c * (1.0 - mat.nu);
      const double c12 = c * mat.nu;
      const double c33 = c * (1.0 - 2.0 * mat.nu) / 2.0;
      if constexpr (D == 2) {  // element.hpp:95-106 verbatim order
        T exx(0.0), eyy(0.0), gxy(0.0);
        for (int i = 0; i < 4; ++i) {
          exx += u[2 * i] * g[i][0];
          eyy += u[2 * i + 1] * g[i][1];
          gxy += u[2 * i] * g[i][1] + u[2 * i + 1] * g[i][0];
        }
        const T s0 = c11 * exx + c12 * eyy, s1 = c12 * exx + c11 * eyy, s2 = c33 * gxy;
        for (int i = 0; i < 4; ++i) {
          out[2 * i] += wdet * (g[i][0] * s0 + g[i][1] * s2);
          out[2 * i + 1] += wdet * (g[i][1] * s1 + g[i][0] * s2);
        }
      } else {  // 3D isotropic Hooke, Voigt [xx, yy, zz, yz, xz, xy]
        T exx(0.0), eyy(0.0), ezz(0.0), gyz(0.0), gxz(0.0), gxy(0.0);
        for (int i = 0; i < 8; ++i) {
          exx += u[3 * i] * g[i][0];
          eyy += u[3 * i + 1] * g[i][1];
          ezz += u[3 * i + 2] * g[i][2];
          gyz += u[3 * i + 1] * g[i][2] + u[3 * i + 2] * g[i][1];
          gxz += u[3 * i] * g[i][2] + u[3 * i + 2] * g[i][0];
          gxy += u[3 * i] * g[i][1] + u[3 * i + 1] * g[i][0];
        }
        const T sxx = c11 * exx + c12 * eyy + c12 * ezz;
        const T syy = c12 * exx + c11 * eyy + c12 * ezz;
        const T szz = c12 * exx + c12 * eyy + c11 * ezz;
        const T syz = c33 * gyz, sxz = c33 * gxz, sxy = c33 * gxy;
        for (int i = 0; i < 8; ++i) {
          out[3 * i] += wdet * (g[i][0] * sxx + g[i][1] * sxy + g[i][2] * sxz);
          out[3 * i + 1] += wdet * (g[i][0] * sxy + g[i][1] * syy + g[i][2] * syz);
          out[3 * i + 2] += wdet * (g[i][0] * sxz + g[i][1] * syz + g[i][2] * szz);
        }
      }
    } else if (mat.model == J2) {
      T eps[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) eps[a][b] = T(0.0);
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          T hab(0.0), hba(0.0);
          for (int i = 0; i < npe; ++i) { hab += u[D * i + a] * g[i][b]; hba += u[D * i + b] * g[i][a]; }
          eps[a][b] = 0.5 * (hab + hba);
        }
      T sig[3][3];
      j2_stress<T>(mat, eps, hist ? hist + qi * kHist : nullptr, sig, hist_new ? hist_new + qi * kHist : nullptr);
      for (int i = 0; i < npe; ++i)
        for (int a = 0; a < D; ++a) {
          T t(0.0);
          for (int b = 0; b < D; ++b) t += sig[a][b] * g[i][b];
          out[D * i + a] += wdet * t;
        }
    } else if (mat.model == NEOHOOKE) {
      // psi = mu/2 (J^{-2/3} I1 - 3) + kappa/2 (J - 1)^2 (pow-only form: the reference's Dual has
      // no log, dual.hpp:162-177). P = mu J^{-2/3} F - (mu/3) I1 J^{-5/3} cof F + kappa (J-1) cof F.
      // Plane strain in 2D: F33 = 1.
      T F[3][3];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          T h(0.0);
          for (int i = 0; i < npe; ++i) h += u[D * i + a] * g[i][b];
          F[a][b] = a == b ? h + 1.0 : h;
        }
      T C[3][3];
      if constexpr (D == 2) {
        C[0][0] = F[1][1]; C[0][1] = -F[1][0]; C[1][0] = -F[0][1]; C[1][1] = F[0][0];
      } else {
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) {
            const int a1 = (a + 1) % 3, a2 = (a + 2) % 3, b1 = (b + 1) % 3, b2 = (b + 2) % 3;
            C[a][b] = F[a1][b1] * F[a2][b2] - F[a1][b2] * F[a2][b1];
          }
      }
      T J(0.0), I1(D == 2 ? 1.0 : 0.0);
      for (int b = 0; b < D; ++b) J += F[0][b] * C[0][b];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) I1 += F[a][b] * F[a][b];
      if (!(value_of(J) > 0.0)) throw InvertedElementError("stress_neohooke: deformation gradient determinant <= 0");
      const double mu = mat.mu(), kappa = mat.kappa();
      const T a23 = pow(J, -2.0 / 3.0);
      const T c1 = mu * a23;
      const T c2 = (mu / 3.0) * I1 * a23 / J;
      const T c3 = kappa * (J - 1.0);
      for (int i = 0; i < npe; ++i)
        for (int a = 0; a < D; ++a) {
          T t(0.0);
          for (int b = 0; b < D; ++b) t += (c1 * F[a][b] + (c3 - c2) * C[a][b]) * g[i][b];
          out[D * i + a] += wdet * t;
        }
    } else {  // St Venant-Kirchhoff (element.hpp:107-123, material.hpp:49-69)
      T F[3][3];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          T h(0.0);
          for (int i = 0; i < npe; ++i) h += u[D * i + a] * g[i][b];
          F[a][b] = a == b ? h + 1.0 : h;
        }
      T det;
      if constexpr (D == 2) det = F[0][0] * F[1][1] - F[0][1] * F[1][0];
      else
        det = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
              F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
              F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
      if (!(value_of(det) > 0.0))
        throw InvertedElementError("stress_svk: deformation gradient determinant <= 0");
      T Eg[3][3], S[3][3];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          T c(0.0);
          if constexpr (D == 2) c = F[0][a] * F[0][b] + F[1][a] * F[1][b];
          else c = F[0][a] * F[0][b] + F[1][a] * F[1][b] + F[2][a] * F[2][b];
          Eg[a][b] = 0.5 * (a == b ? c - 1.0 : c);
        }
      const double lam = mat.lambda(), mu = mat.mu();
      T tr;
      if constexpr (D == 2) tr = Eg[0][0] + Eg[1][1];
      else tr = Eg[0][0] + Eg[1][1] + Eg[2][2];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) S[a][b] = 2.0 * mu * Eg[a][b] + (a == b ? lam * tr : T(0.0));
      T P[3][3];
      for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
          if constexpr (D == 2) P[a][b] = F[a][0] * S[0][b] + F[a][1] * S[1][b];
          else P[a][b] = F[a][0] * S[0][b] + F[a][1] * S[1][b] + F[a][2] * S[2][b];
        }
      for (int i = 0; i < npe; ++i)
        for (int a = 0; a < D; ++a) {
          if constexpr (D == 2) out[2 * i + a] += wdet * (P[a][0] * g[i][0] + P[a][1] * g[i][1]);
          else out[3 * i + a] += wdet * (P[a][0] * g[i][0] + P[a][1] * g[i][1] + P[a][2] * g[i][2]);
        }
    }
  }
}

// ---------------------------------------------------------------- mesh (mesh.hpp:47-101)
struct Mesh {
  int dim = 2;
  std::vector<double> coords;  // n_nodes * dim
  std::vector<int> conn;       // n_elem * npe
  std::vector<int> phase;      // n_elem
  int nx = 0, ny = 0, nz = 0;
  double lx = 0, ly = 0, lz = 0;
  int64_t n_nodes() const { return (int64_t)coords.size() / dim; }
  int64_t n_elem() const { return (int64_t)phase.size(); }
  int64_t n_dof() const { return dim * n_nodes(); }
};

inline Mesh mesh2d(int nx, int ny, double lx, double ly, double cx0, double cy0, double radius) {
  if (nx < 1 || ny < 1) throw std::invalid_argument("mesh: cell counts must be >= 1");
  if (!(lx > 0.0) || !(ly > 0.0)) throw std::invalid_argument("mesh: domain lengths must be > 0");
  if (radius < 0.0) throw std::invalid_argument("mesh: inclusion radius must be >= 0");
  Mesh m; m.dim = 2; m.nx = nx; m.ny = ny; m.lx = lx; m.ly = ly;
  const double hx = lx / nx, hy = ly / ny;
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) { m.coords.push_back(i * hx); m.coords.push_back(j * hy); }
  const double r2 = radius * radius;
  auto node = [&](int i, int j) { return i + j * (nx + 1); };
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      m.conn.insert(m.conn.end(), {node(ex, ey), node(ex + 1, ey), node(ex + 1, ey + 1), node(ex, ey + 1)});
      const double cx = (ex + 0.5) * hx - cx0;
      const double cy = (ey + 0.5) * hy - cy0;
      m.phase.push_back(cx * cx + cy * cy < r2 ? 1 : 0);
    }
  return m;
}

// hex8 twin: node (i,j,k) = i + (nx+1)(j + (ny+1)k); element loop ez, ey, ex; fibres parallel to z;
// phase 1 iff the element centroid is strictly inside any fibre circle (mesh.hpp:79-81 analog).
inline Mesh mesh3d(int nx, int ny, int nz, double lx, double ly, double lz,
                   const std::vector<std::array<double, 2>>& fibres, double radius) {
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("mesh: cell counts must be >= 1");
  if (!(lx > 0.0) || !(ly > 0.0) || !(lz > 0.0)) throw std::invalid_argument("mesh: domain lengths must be > 0");
  if (radius < 0.0) throw std::invalid_argument("mesh: inclusion radius must be >= 0");
  Mesh m; m.dim = 3; m.nx = nx; m.ny = ny; m.nz = nz; m.lx = lx; m.ly = ly; m.lz = lz;
  const double hx = lx / nx, hy = ly / ny, hz = lz / nz;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        m.coords.push_back(i * hx); m.coords.push_back(j * hy); m.coords.push_back(k * hz);
      }
  const double r2 = radius * radius;
  auto node = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
  for (int ez = 0; ez < nz; ++ez)
    for (int ey = 0; ey < ny; ++ey)
      for (int ex = 0; ex < nx; ++ex) {
        m.conn.insert(m.conn.end(),
                      {node(ex, ey, ez), node(ex + 1, ey, ez), node(ex + 1, ey + 1, ez), node(ex, ey + 1, ez),
                       node(ex, ey, ez + 1), node(ex + 1, ey, ez + 1), node(ex + 1, ey + 1, ez + 1),
                       node(ex, ey + 1, ez + 1)});
        int ph = 0;
        for (const auto& f : fibres) {
          const double cx = (ex + 0.5) * hx - f[0];
          const double cy = (ey + 0.5) * hy - f[1];
          if (cx * cx + cy * cy < r2) { ph = 1; break; }
        }
        m.phase.push_back(ph);
      }
  return m;
}

inline std::vector<std::array<double, 2>> fibres(uint64_t seed, int n, double lx, double ly) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> ux(0.0, lx), uy(0.0, ly);
  std::vector<std::array<double, 2>> out;
  for (int i = 0; i < n; ++i) { const double x = ux(rng); const double y = uy(rng); out.push_back({x, y}); }
  return out;
}

struct Constraint { int node, comp; double value; };

// benchmark_bcs (mesh.hpp:89-101); 3D: x=0 face u_x=0 (k outer, j inner), node(0,0,0) u_y=u_z=0,
// node(0,0,nz) u_y=0 (kills the rotation about x), x=lx face u_x=strain*lx.
inline std::vector<Constraint> benchmark_bcs(int dim, int nx, int ny, int nz, double lx, double strain) {
  if (nx < 1 || ny < 1 || (dim == 3 && nz < 1))
    throw std::invalid_argument("benchmark_bcs: mesh lacks structured-grid metadata");
  std::vector<Constraint> c;
  const double u_right = strain * lx;
  if (dim == 2) {
    auto node = [&](int i, int j) { return i + j * (nx + 1); };
    for (int j = 0; j <= ny; ++j) c.push_back({node(0, j), 0, 0.0});
    c.push_back({node(0, 0), 1, 0.0});
    for (int j = 0; j <= ny; ++j) c.push_back({node(nx, j), 0, u_right});
  } else {
    auto node = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= ny; ++j) c.push_back({node(0, j, k), 0, 0.0});
    c.push_back({node(0, 0, 0), 1, 0.0});
    c.push_back({node(0, 0, 0), 2, 0.0});
    c.push_back({node(0, 0, nz), 1, 0.0});
    for (int k = 0; k <= nz; ++k)
      for (int j = 0; j <= ny; ++j) c.push_back({node(nx, j, k), 0, u_right});
  }
  return c;
}

// ---------------------------------------------------------------- sparse (sparse.hpp:28-59)
inline void sort_and_deduplicate(std::vector<double>& values, std::vector<int>& rows, std::vector<int>& cols) {
  if (rows.size() != cols.size() || rows.size() != values.size())
    throw std::invalid_argument("sort_and_deduplicate: array lengths differ");
  const std::size_t nnz = values.size();
  if (nnz == 0) return;
  std::vector<std::size_t> perm(nnz);
  std::iota(perm.begin(), perm.end(), std::size_t{0});
  std::stable_sort(perm.begin(), perm.end(), [&](std::size_t a, std::size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  std::vector<int> r_out, c_out;
  std::vector<double> v_out;
  r_out.reserve(nnz); c_out.reserve(nnz); v_out.reserve(nnz);
  for (std::size_t k = 0; k < nnz; ++k) {
    const std::size_t p = perm[k];
    if (!r_out.empty() && r_out.back() == rows[p] && c_out.back() == cols[p]) v_out.back() += values[p];
    else { r_out.push_back(rows[p]); c_out.push_back(cols[p]); v_out.push_back(values[p]); }
  }
  rows = std::move(r_out); cols = std::move(c_out); values = std::move(v_out);
}

struct Pattern {
  int64_t n_dof = 0;
  std::vector<int> rows, cols;
  std::vector<int64_t> row_ptr;
  std::size_t nnz() const { return cols.size(); }
};

// ---------------------------------------------------------------- batches (assembly.hpp:22-67)
struct Batch {
  std::vector<int> element_ids;
  std::vector<int> dof_map;      // size * ndpe
  std::vector<double> coords;    // size * npe * dim
  Material material;
  int quadrature = 2;
  const double* hist = nullptr;  // System::history (element-id indexed), J2 systems only
  std::size_t size() const { return element_ids.size(); }
};

struct ConstraintTable {
  std::vector<char> constrained;
  std::vector<double> prescribed;
};

// ---------------------------------------------------------------- the system
struct System {
  Mesh mesh;
  std::vector<Material> materials;
  std::vector<Batch> batches;
  Pattern pattern;
  ConstraintTable table;
  std::vector<Constraint> constraints;
  // committed Gauss-point history (J2): n_elem * nq * kHist, element-id indexed; empty otherwise.
  std::vector<double> history;
  int dim() const { return mesh.dim; }
  int nq() const { return mesh.dim == 2 ? 4 : 8; }
  void init_history() {
    bool j2 = false;
    for (const auto& m : materials) j2 |= m.model == J2;
    history.assign(j2 ? (std::size_t)mesh.n_elem() * nq() * kHist : 0, 0.0);
    for (auto& b : batches) b.hist = history.empty() ? nullptr : history.data();
  }
  int64_t n_dof() const { return mesh.n_dof(); }
};

inline std::vector<Batch> build_batches(const Mesh& mesh, const std::vector<Material>& mats) {
  const int D = mesh.dim, npe = D == 2 ? 4 : 8;
  int max_phase = -1;
  for (int p : mesh.phase) max_phase = std::max(max_phase, p);
  if (max_phase >= (int)mats.size())
    throw std::invalid_argument("build_batches: no material supplied for a mesh phase");
  for (const auto& m : mats) m.validate();
  std::vector<Batch> b(std::max(0, max_phase + 1));
  for (std::size_t p = 0; p < b.size(); ++p) b[p].material = mats[p];
  for (int64_t e = 0; e < mesh.n_elem(); ++e) {
    const int ph = mesh.phase[e];
    if (ph < 0) throw std::invalid_argument("build_batches: negative phase label");
    Batch& bb = b[ph];
    bb.element_ids.push_back((int)e);
    for (int k = 0; k < npe; ++k) {
      const int n = mesh.conn[e * npe + k];
      if (n < 0 || n >= mesh.n_nodes()) throw std::out_of_range("build_batches: node index outside mesh");
      for (int c = 0; c < D; ++c) bb.dof_map.push_back(D * n + c);
      for (int c = 0; c < D; ++c) bb.coords.push_back(mesh.coords[(std::size_t)n * D + c]);
    }
  }
  std::erase_if(b, [](const Batch& x) { return x.element_ids.empty(); });
  return b;
}

// precompute_sparsity (assembly.hpp:71-99)
inline Pattern precompute_sparsity(const std::vector<Batch>& batches, int64_t n_dof, int D) {
  const int nd = D == 2 ? 8 : 24;
  std::vector<int> rows, cols;
  for (const auto& b : batches)
    for (std::size_t e = 0; e < b.size(); ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int i = 0; i < nd; ++i)
        for (int j = 0; j < nd; ++j) {
          if (dofs[i] >= n_dof || dofs[j] >= n_dof)
            throw std::out_of_range("precompute_sparsity: dof index outside system");
          rows.push_back(dofs[i]);
          cols.push_back(dofs[j]);
        }
    }
  std::vector<double> dummy(rows.size(), 0.0);
  sort_and_deduplicate(dummy, rows, cols);
  Pattern p;
  p.n_dof = n_dof;
  p.row_ptr.assign(n_dof + 1, 0);
  for (int r : rows) ++p.row_ptr[r + 1];
  for (int64_t i = 0; i < n_dof; ++i) p.row_ptr[i + 1] += p.row_ptr[i];
  p.rows = std::move(rows);
  p.cols = std::move(cols);
  return p;
}

template <int D, class T>
inline void batch_kernel(const Batch& b, std::size_t e, const T* u, T* out) {
  const double* h = b.hist ? b.hist + (std::size_t)b.element_ids[e] * (D == 2 ? 4 : 8) * kHist : nullptr;
  element_internal_force<D, T>(&b.coords[e * ET<D>::npe * D], b.material, b.quadrature, u, out, h);
}

// History commit (J2): every Gauss point's committed history advances to the return-mapped state at u.
template <int D>
void commit_history(System& s, const double* u) {
  if (s.history.empty()) return;
  constexpr int nd = ET<D>::ndpe, nq = D == 2 ? 4 : 8;
  double ue[nd], re[nd];
  for (const auto& b : s.batches) {
    if (b.material.model != J2) continue;
    for (std::size_t e = 0; e < b.size(); ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int k = 0; k < nd; ++k) ue[k] = u[dofs[k]];
      double* h = s.history.data() + (std::size_t)b.element_ids[e] * nq * kHist;
      double hn[nq * kHist];
      element_internal_force<D, double>(&b.coords[e * ET<D>::npe * D], b.material, b.quadrature, ue, re, h, hn);
      std::copy(hn, hn + nq * kHist, h);
    }
  }
}

// assemble_residual (assembly.hpp:126-139)
template <int D>
std::vector<double> assemble_residual(const std::vector<Batch>& batches, const double* u, int64_t n) {
  constexpr int nd = ET<D>::ndpe;
  std::vector<double> r(n, 0.0);
  double ue[nd], re[nd];
  for (const auto& b : batches)
    for (std::size_t e = 0; e < b.size(); ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int k = 0; k < nd; ++k) ue[k] = u[dofs[k]];
      batch_kernel<D, double>(b, e, ue, re);
      for (int k = 0; k < nd; ++k) r[dofs[k]] += re[k];
    }
  return r;
}

// Element Jacobian by forward AD in seed blocks of 8 (autodiff.hpp:23, 53-98).
template <int D>
void element_jacobian(const Batch& b, std::size_t e, const double* ue, double* K /* nd*nd row-major */) {
  constexpr int nd = ET<D>::ndpe;
  for (int c0 = 0; c0 < nd; c0 += 8) {
    Dual<8> x[nd], y[nd];
    for (int i = 0; i < nd; ++i) {
      x[i] = Dual<8>(ue[i]);
      for (int k = 0; k < 8; ++k) x[i].d[k] = (i == c0 + k) ? 1.0 : 0.0;
    }
    batch_kernel<D, Dual<8>>(b, e, x, y);
    for (int i = 0; i < nd; ++i)
      for (int k = 0; k < 8; ++k) K[i * nd + c0 + k] = y[i].d[k];
  }
}

// assemble_jacobian (assembly.hpp:144-173): values in pattern order; indices must match the pattern.
template <int D>
std::vector<double> assemble_jacobian(const System& s, const double* u) {
  constexpr int nd = ET<D>::ndpe;
  std::vector<int> rows, cols;
  std::vector<double> vals;
  std::vector<double> K(nd * nd), ue(nd);
  for (const auto& b : s.batches)
    for (std::size_t e = 0; e < b.size(); ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int k = 0; k < nd; ++k) ue[k] = u[dofs[k]];
      element_jacobian<D>(b, e, ue.data(), K.data());
      for (int i = 0; i < nd; ++i)
        for (int j = 0; j < nd; ++j) {
          rows.push_back(dofs[i]); cols.push_back(dofs[j]); vals.push_back(K[i * nd + j]);
        }
    }
  sort_and_deduplicate(vals, rows, cols);
  if (rows != s.pattern.rows || cols != s.pattern.cols)
    throw std::logic_error("assemble_jacobian: produced indices leave the precomputed pattern");
  return vals;
}

// assemble_diagonal (assembly.hpp:177-188)
template <int D>
std::vector<double> assemble_diagonal(const std::vector<Batch>& batches, const double* u, int64_t n) {
  constexpr int nd = ET<D>::ndpe;
  std::vector<double> diag(n, 0.0), K(nd * nd), ue(nd);
  for (const auto& b : batches)
    for (std::size_t e = 0; e < b.size(); ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int k = 0; k < nd; ++k) ue[k] = u[dofs[k]];
      element_jacobian<D>(b, e, ue.data(), K.data());
      for (int k = 0; k < nd; ++k) diag[dofs[k]] += K[k * nd + k];
    }
  return diag;
}

// assemble_diagonal on host threads (bench/test sizing only): per-thread partial vectors over
// contiguous element ranges of each batch, summed in thread order afterwards.
template <int D>
std::vector<double> assemble_diagonal_mt(const std::vector<Batch>& batches, const double* u, int64_t n,
                                         int nthreads) {
  if (nthreads <= 1) return assemble_diagonal<D>(batches, u, n);
  constexpr int nd = ET<D>::ndpe;
  std::vector<std::vector<double>> part(nthreads, std::vector<double>(n, 0.0));
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t)
    th.emplace_back([&, t] {
      std::vector<double> K(nd * nd), ue(nd);
      for (const auto& b : batches) {
        const std::size_t lo = b.size() * t / nthreads, hi = b.size() * (t + 1) / nthreads;
        for (std::size_t e = lo; e < hi; ++e) {
          const int* dofs = &b.dof_map[e * nd];
          for (int k = 0; k < nd; ++k) ue[k] = u[dofs[k]];
          element_jacobian<D>(b, e, ue.data(), K.data());
          for (int k = 0; k < nd; ++k) part[t][dofs[k]] += K[k * nd + k];
        }
      }
    });
  for (auto& x : th) x.join();
  std::vector<double> diag(n, 0.0);
  for (int t = 0; t < nthreads; ++t)
    for (int64_t i = 0; i < n; ++i) diag[i] += part[t][i];
  return diag;
}

// constraint_table (assembly.hpp:197-211)
inline ConstraintTable constraint_table(const std::vector<Constraint>& cs, int64_t n_dof, int D) {
  ConstraintTable t;
  t.constrained.assign(n_dof, 0);
  t.prescribed.assign(n_dof, 0.0);
  for (const auto& c : cs) {
    const long dof = (long)D * c.node + c.comp;
    if (dof < 0 || dof >= n_dof) throw std::out_of_range("dirichlet: constrained dof outside system");
    if (t.constrained[dof]) throw std::invalid_argument("dirichlet: duplicate (node, component) pair");
    t.constrained[dof] = 1;
    t.prescribed[dof] = c.value;
  }
  return t;
}

// validate_dirichlet (mesh.hpp:105-116)
inline void validate_dirichlet(const std::vector<Constraint>& cs, int64_t n_nodes, int D) {
  std::vector<char> seen(n_nodes * D, 0);
  for (const auto& c : cs) {
    if (c.node < 0 || c.node >= n_nodes) throw std::out_of_range("dirichlet: constrained node outside mesh");
    if (c.comp < 0 || c.comp >= D) throw std::invalid_argument("dirichlet: component out of range");
    const std::size_t dof = (std::size_t)D * c.node + c.comp;
    if (seen[dof]) throw std::invalid_argument("dirichlet: duplicate (node, component) pair");
    seen[dof] = 1;
  }
}

// eliminate_dirichlet (assembly.hpp:218-238)
inline void eliminate_dirichlet(const Pattern& p, double* values, double* residual,
                                const ConstraintTable& t, const double* u) {
  const int64_t n = p.n_dof;
  for (int64_t i = 0; i < n; ++i) {
    const bool ci = t.constrained[i] != 0;
    for (int64_t k = p.row_ptr[i]; k < p.row_ptr[i + 1]; ++k) {
      const int j = p.cols[k];
      const bool cj = t.constrained[j] != 0;
      if (!ci && cj) {
        residual[i] += values[k] * (t.prescribed[j] - u[j]);
        values[k] = 0.0;
      } else if (ci) {
        values[k] = (i == j) ? 1.0 : 0.0;
      }
    }
  }
  for (int64_t d = 0; d < n; ++d)
    if (t.constrained[d]) residual[d] = u[d] - t.prescribed[d];
}

// ---------------------------------------------------------------- linear algebra (linalg.hpp:41-58)
inline double dot(const double* x, const double* y, std::size_t n) {
  double s = 0.0;
  for (std::size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
inline double norm2(const double* x, std::size_t n) { return std::sqrt(dot(x, x, n)); }
inline void axpy(double a, const double* x, double* y, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) y[i] += a * x[i];
}

// ---------------------------------------------------------------- operators (backend.hpp:117-236)
struct Operator {
  virtual ~Operator() = default;
  virtual int64_t dim() const = 0;
  virtual void apply(const double* x, double* y) const = 0;
  virtual std::vector<double> diagonal() const = 0;
};

// CsrMatrix::apply (sparse.hpp:106-117) + csr_diagonal (krylov.hpp:102-111)
struct ExplicitOperator : Operator {
  const Pattern* p;
  std::vector<double> values;
  int64_t dim() const override { return p->n_dof; }
  void apply(const double* x, double* y) const override {
    for (int64_t i = 0; i < p->n_dof; ++i) {
      double s = 0.0;
      for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k) s += values[k] * x[p->cols[k]];
      y[i] = s;
    }
  }
  std::vector<double> diagonal() const override {
    std::vector<double> d(p->n_dof, 0.0);
    for (int64_t i = 0; i < p->n_dof; ++i)
      for (int64_t k = p->row_ptr[i]; k < p->row_ptr[i + 1]; ++k)
        if (p->cols[k] == i) d[i] = values[k];
    return d;
  }
};

// LinearOperator MATRIX_FREE apply (backend.hpp:130-147): Dual<1> JVP per element.
template <int D>
struct MatrixFreeOperator : Operator {
  const System* s;
  std::vector<double> state, diag;
  int nthreads = 1;
  mutable std::vector<double> masked;
  int64_t dim() const override { return s->n_dof(); }

  void apply_range(const Batch& b, std::size_t e0, std::size_t e1, double* y) const {
    constexpr int nd = ET<D>::ndpe;
    Dual<1> ue[nd], re[nd];
    for (std::size_t e = e0; e < e1; ++e) {
      const int* dofs = &b.dof_map[e * nd];
      for (int k = 0; k < nd; ++k) { ue[k] = Dual<1>(state[dofs[k]]); ue[k].d[0] = masked[dofs[k]]; }
      batch_kernel<D, Dual<1>>(b, e, ue, re);
      for (int k = 0; k < nd; ++k) y[dofs[k]] += re[k].d[0];
    }
  }

  void apply(const double* x, double* y) const override {
    const int64_t n = dim();
    masked.assign(x, x + n);
    for (int64_t d = 0; d < n; ++d) if (s->table.constrained[d]) masked[d] = 0.0;
    std::fill(y, y + n, 0.0);
    if (nthreads <= 1) {
      for (const Batch& b : s->batches) apply_range(b, 0, b.size(), y);
    } else {  // bench CPU baseline only: per-thread partial vectors, fixed-order reduction
      std::vector<std::vector<double>> part(nthreads, std::vector<double>(n, 0.0));
      std::vector<std::thread> th;
      for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t] {
          for (const Batch& b : s->batches) {
            const std::size_t lo = b.size() * t / nthreads, hi = b.size() * (t + 1) / nthreads;
            apply_range(b, lo, hi, part[t].data());
          }
        });
      for (auto& x2 : th) x2.join();
      for (int t = 0; t < nthreads; ++t)
        for (int64_t i = 0; i < n; ++i) y[i] += part[t][i];
    }
    for (int64_t d = 0; d < n; ++d) if (s->table.constrained[d]) y[d] = x[d];
  }
  std::vector<double> diagonal() const override { return diag; }
};

// matrix_free_operator (backend.hpp:222-236)
template <int D>
MatrixFreeOperator<D> make_mf(const System& s, const double* u) {
  MatrixFreeOperator<D> op;
  op.s = &s;
  op.state.assign(u, u + s.n_dof());
  op.diag = assemble_diagonal<D>(s.batches, u, s.n_dof());
  for (int64_t d = 0; d < s.n_dof(); ++d) if (s.table.constrained[d]) op.diag[d] = 1.0;
  return op;
}

// ---------------------------------------------------------------- Krylov (krylov.hpp:43-530)
struct SolverConfig {
  int method = 0;  // 0 CG, 1 GMRES
  int precond = 0; // 0 NONE, 1 JACOBI
  double rtol = 1e-13;
  int max_iter = 10000;
  int restart = 30;
  void validate() const {
    if (!(rtol > 0.0)) throw std::invalid_argument("solver config: rtol must be > 0");
    if (max_iter < 1) throw std::invalid_argument("solver config: max_iter must be >= 1");
    if (restart < 1) throw std::invalid_argument("solver config: gmres_restart must be >= 1");
  }
};

struct SolveReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_history;
  double wall_time = 0.0;
  std::string failure;
};

struct Precond {
  bool jacobi = false;
  std::vector<double> inv;
  // ILU(0) (krylov.hpp:116-192): factor values on the pattern, diagonal positions
  bool ilu = false;
  const Pattern* pat = nullptr;
  std::vector<double> lu;
  std::vector<int64_t> diag;
  void apply(const double* r, double* z, std::size_t n) const {
    if (ilu) {
      const auto& rp = pat->row_ptr;
      const auto& ci = pat->cols;
      for (std::size_t i = 0; i < n; ++i) {
        double s = r[i];
        for (int64_t k = rp[i]; k < rp[i + 1] && ci[k] < (int)i; ++k) s -= lu[k] * z[ci[k]];
        z[i] = s;
      }
      for (int64_t i = (int64_t)n - 1; i >= 0; --i) {
        double s = z[i];
        const int64_t dk = diag[i];
        for (int64_t k = dk + 1; k < rp[i + 1]; ++k) s -= lu[k] * z[ci[k]];
        z[i] = s / lu[dk];
      }
      return;
    }
    if (!jacobi) { std::copy(r, r + n, z); return; }
    for (std::size_t i = 0; i < n; ++i) z[i] = r[i] * inv[i];
  }
  static Precond ilu0(const Pattern& p, const std::vector<double>& values) {  // krylov.hpp:120-152
    Precond m;
    m.ilu = true;
    m.pat = &p;
    m.lu = values;
    const int64_t n = p.n_dof;
    m.diag.assign(n, -1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = p.row_ptr[i]; k < p.row_ptr[i + 1]; ++k)
        if (p.cols[k] == i) m.diag[i] = k;
    for (int64_t i = 0; i < n; ++i)
      if (m.diag[i] < 0) throw FactorizationError("ilu0: structurally missing diagonal at row " + std::to_string(i));
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t kk = p.row_ptr[i]; kk < p.row_ptr[i + 1]; ++kk) {
        const int k = p.cols[kk];
        if (k >= i) break;
        const double ukk = m.lu[m.diag[k]];
        if (ukk == 0.0) throw FactorizationError("ilu0: zero pivot at row " + std::to_string(k));
        const double lik = m.lu[kk] / ukk;
        m.lu[kk] = lik;
        for (int64_t uk = m.diag[k] + 1; uk < p.row_ptr[k + 1]; ++uk) {
          const int j = p.cols[uk];
          const auto b = p.cols.begin() + p.row_ptr[i], e = p.cols.begin() + p.row_ptr[i + 1];
          const auto it = std::lower_bound(b, e, j);
          if (it != e && *it == j) m.lu[it - p.cols.begin()] -= lik * m.lu[uk];
        }
      }
      if (m.lu[m.diag[i]] == 0.0) throw FactorizationError("ilu0: zero pivot at row " + std::to_string(i));
    }
    return m;
  }
  static Precond from_diagonal(const std::vector<double>& d) {  // krylov.hpp:83-92
    Precond p; p.jacobi = true; p.inv.resize(d.size());
    for (std::size_t i = 0; i < d.size(); ++i) {
      if (d[i] == 0.0) throw FactorizationError("jacobi: zero diagonal at row " + std::to_string(i));
      p.inv[i] = 1.0 / d[i];
    }
    return p;
  }
};

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double seconds() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
};

inline double true_relative_residual(const Operator& a, const double* b, const double* x, double denom,
                                     std::vector<double>& scratch) {  // krylov.hpp:331-342
  const std::size_t n = a.dim();
  scratch.resize(n);
  a.apply(x, scratch.data());
  double s = 0.0;
  for (std::size_t i = 0; i < n; ++i) { const double d = b[i] - scratch[i]; s += d * d; }
  return std::sqrt(s) / denom;
}

// cg (krylov.hpp:350-408)
inline std::vector<double> cg(const Operator& a, const double* b, const SolverConfig& cfg, const Precond& m,
                              const double* x0, SolveReport& rep) {
  cfg.validate();
  Timer timer;
  const std::size_t n = a.dim();
  std::vector<double> x = x0 ? std::vector<double>(x0, x0 + n) : std::vector<double>(n, 0.0);
  const double bnorm = norm2(b, n);
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  std::vector<double> r(n), z(n), p(n), ap(n), scratch;
  a.apply(x.data(), ap.data());
  for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - ap[i];
  rep.residual_history.push_back(norm2(r.data(), n) / denom);
  while (true) {
    if (rep.residual_history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      m.apply(r.data(), z.data(), n);
      std::copy(z.begin(), z.end(), p.begin());
      double rz = dot(r.data(), z.data(), n);
      while (rep.iterations < cfg.max_iter && rep.residual_history.back() > cfg.rtol) {
        a.apply(p.data(), ap.data());
        const double pap = dot(p.data(), ap.data(), n);
        if (!(pap > 0.0)) {
          rep.failure = "cg: operator not positive definite (p^T A p <= 0 at iteration " +
                        std::to_string(rep.iterations + 1) + ")";
          break;
        }
        const double alpha = rz / pap;
        axpy(alpha, p.data(), x.data(), n);
        axpy(-alpha, ap.data(), r.data(), n);
        ++rep.iterations;
        rep.residual_history.push_back(norm2(r.data(), n) / denom);
        if (rep.residual_history.back() <= cfg.rtol) break;
        m.apply(r.data(), z.data(), n);
        const double rz_new = dot(r.data(), z.data(), n);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (std::size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
      }
    }
    const double true_rres = true_relative_residual(a, b, x.data(), denom, scratch);
    rep.residual_history.back() = true_rres;
    if (true_rres <= cfg.rtol) { rep.converged = rep.failure.empty(); break; }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    a.apply(x.data(), ap.data());
    for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - ap[i];
  }
  rep.wall_time = timer.seconds();
  return x;
}

// gmres (krylov.hpp:415-530)
inline std::vector<double> gmres(const Operator& a, const double* b, const SolverConfig& cfg, const Precond& m,
                                 const double* x0, SolveReport& rep) {
  cfg.validate();
  Timer timer;
  const std::size_t n = a.dim();
  const int restart = std::min<int>(cfg.restart, (int)n);
  std::vector<double> x = x0 ? std::vector<double>(x0, x0 + n) : std::vector<double>(n, 0.0);
  const double bnorm = norm2(b, n);
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  std::vector<double> tmp(n), scratch;
  m.apply(b, tmp.data(), n);
  const double pnorm = norm2(tmp.data(), n);
  const double pdenom = pnorm > 0.0 ? pnorm : 1.0;
  std::vector<std::vector<double>> v(restart + 1, std::vector<double>(n));
  std::vector<double> h((restart + 1) * restart, 0.0);
  auto H = [&](int i, int j) -> double& { return h[(std::size_t)i * restart + j]; };
  std::vector<double> cs(restart), sn(restart), g(restart + 1);
  std::vector<double> r(n), w(n);
  a.apply(x.data(), tmp.data());
  for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
  m.apply(r.data(), w.data(), n);
  rep.residual_history.push_back(norm2(w.data(), n) / pdenom);
  double true_rres = norm2(r.data(), n) / denom;
  while (true_rres > cfg.rtol && rep.iterations < cfg.max_iter && rep.failure.empty()) {
    m.apply(r.data(), w.data(), n);
    const double beta = norm2(w.data(), n);
    if (beta == 0.0) break;
    const double target_est = beta * std::min(1.0, 0.5 * cfg.rtol / true_rres);
    for (std::size_t i = 0; i < n; ++i) v[0][i] = w[i] / beta;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0, cols = 0;
    for (; j < restart && rep.iterations < cfg.max_iter; ++j) {
      a.apply(v[j].data(), tmp.data());
      m.apply(tmp.data(), w.data(), n);
      for (int i = 0; i <= j; ++i) {
        const double hij = dot(v[i].data(), w.data(), n);
        H(i, j) = hij;
        axpy(-hij, v[i].data(), w.data(), n);
      }
      const double hnext = norm2(w.data(), n);
      H(j + 1, j) = hnext;
      const bool happy = hnext <= beta * 1e-16;
      if (!happy) for (std::size_t i = 0; i < n; ++i) v[j + 1][i] = w[i] / hnext;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
        H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
        H(i, j) = t;
      }
      const double rr = std::hypot(H(j, j), H(j + 1, j));
      if (rr == 0.0) { cs[j] = 1.0; sn[j] = 0.0; }
      else { cs[j] = H(j, j) / rr; sn[j] = H(j + 1, j) / rr; }
      H(j, j) = rr;
      H(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] *= cs[j];
      ++rep.iterations;
      cols = j + 1;
      const double est = std::abs(g[j + 1]);
      rep.residual_history.push_back(est / pdenom);
      if (est <= target_est || happy) { ++j; break; }
    }
    std::vector<double> y(cols, 0.0);
    for (int i = cols - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < cols; ++k) s -= H(i, k) * y[k];
      if (H(i, i) == 0.0) { rep.failure = "gmres: singular least-squares system in restart cycle"; break; }
      y[i] = s / H(i, i);
    }
    if (!rep.failure.empty()) break;
    for (int k = 0; k < cols; ++k) axpy(y[k], v[k].data(), x.data(), n);
    a.apply(x.data(), tmp.data());
    for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
    true_rres = norm2(r.data(), n) / denom;
  }
  true_rres = true_relative_residual(a, b, x.data(), denom, scratch);
  rep.residual_history.push_back(true_rres);
  rep.converged = rep.failure.empty() && true_rres <= cfg.rtol;
  rep.wall_time = timer.seconds();
  return x;
}

// run_solver (backend.hpp:241-286), iterative branch

// bicgstab (krylov.hpp:535-620): unpreconditioned recurrence residual, rho / rhat.v / omega
// breakdowns reported as failures, early exit on a small s, true-residual re-verification with a
// restart from the fresh residual.
inline std::vector<double> bicgstab(const Operator& a, const double* b, const SolverConfig& cfg, const Precond& m,
                                    const double* x0, SolveReport& rep) {
  cfg.validate();
  Timer timer;
  const std::size_t n = a.dim();
  std::vector<double> x = x0 ? std::vector<double>(x0, x0 + n) : std::vector<double>(n, 0.0);
  const double bnorm = norm2(b, n);
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  std::vector<double> r(n), rhat(n), p(n, 0.0), v(n, 0.0), s(n), t(n), phat(n), shat(n), scratch;
  a.apply(x.data(), t.data());
  for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
  rhat = r;
  rep.residual_history.push_back(norm2(r.data(), n) / denom);
  while (true) {
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    while (rep.residual_history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      const double rho_new = dot(rhat.data(), r.data(), n);
      if (rho_new == 0.0) {
        rep.failure = "bicgstab: rho breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      const double beta = (rho_new / rho) * (alpha / omega);
      rho = rho_new;
      for (std::size_t i = 0; i < n; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
      m.apply(p.data(), phat.data(), n);
      a.apply(phat.data(), v.data());
      const double rhat_v = dot(rhat.data(), v.data(), n);
      if (rhat_v == 0.0) {
        rep.failure = "bicgstab: rhat^T v breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      alpha = rho / rhat_v;
      for (std::size_t i = 0; i < n; ++i) s[i] = r[i] - alpha * v[i];
      if (norm2(s.data(), n) / denom <= cfg.rtol) {
        axpy(alpha, phat.data(), x.data(), n);
        r = s;
        ++rep.iterations;
        rep.residual_history.push_back(norm2(r.data(), n) / denom);
        break;
      }
      m.apply(s.data(), shat.data(), n);
      a.apply(shat.data(), t.data());
      const double tt = dot(t.data(), t.data(), n);
      if (tt == 0.0) {
        rep.failure = "bicgstab: omega breakdown (t = 0) at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      omega = dot(t.data(), s.data(), n) / tt;
      if (omega == 0.0) {
        rep.failure = "bicgstab: omega breakdown at iteration " + std::to_string(rep.iterations + 1);
        break;
      }
      for (std::size_t i = 0; i < n; ++i) {
        x[i] += alpha * phat[i] + omega * shat[i];
        r[i] = s[i] - omega * t[i];
      }
      ++rep.iterations;
      rep.residual_history.push_back(norm2(r.data(), n) / denom);
    }
    const double true_rres = true_relative_residual(a, b, x.data(), denom, scratch);
    rep.residual_history.back() = true_rres;
    if (true_rres <= cfg.rtol) {
      rep.converged = rep.failure.empty();
      break;
    }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    a.apply(x.data(), t.data());
    for (std::size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
    rhat = r;
    std::fill(p.begin(), p.end(), 0.0);
    std::fill(v.begin(), v.end(), 0.0);
  }
  rep.wall_time = timer.seconds();
  return x;
}

inline std::vector<double> run_solver(const Operator& op, const double* b, const SolverConfig& cfg,
                                      const double* x0, SolveReport& rep) {
  cfg.validate();
  if (cfg.method < 0 || cfg.method > 2) throw std::invalid_argument("run_solver: only CG, GMRES and BiCGStab are restated");
  Precond m;
  if (cfg.precond == 1) m = Precond::from_diagonal(op.diagonal());
  else if (cfg.precond == 2) {  // ilu0_setup(op.csr()) (backend.hpp:282; csr() gate :151-156)
    const auto* e = dynamic_cast<const ExplicitOperator*>(&op);
    if (!e) throw CapabilityError("assembled matrix required, but the operator is matrix-free");
    m = Precond::ilu0(*e->p, e->values);
  } else if (cfg.precond != 0) throw CapabilityError("run_solver: preconditioner not restated");
  if (cfg.method == 2) return bicgstab(op, b, cfg, m, x0, rep);
  return cfg.method == 0 ? cg(op, b, cfg, m, x0, rep) : gmres(op, b, cfg, m, x0, rep);
}

// ---------------------------------------------------------------- Newton (newton.hpp:19-186)
struct NewtonConfig {
  double rtol = 1e-10, atol = 1e-14;
  int max_iter = 25;
  int operator_kind = 0;
  SolverConfig linear;
  void validate() const {
    if (!(rtol > 0.0) || !(atol > 0.0)) throw std::invalid_argument("newton config: tolerances must be > 0");
    if (max_iter < 1) throw std::invalid_argument("newton config: max_iter must be >= 1");
    linear.validate();
  }
};
struct NewtonReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_norms;
  std::vector<SolveReport> linear_reports;
  double total_time = 0.0;
  std::string failure;
};

inline double free_norm(const std::vector<double>& r, const ConstraintTable& t) {
  double s = 0.0;
  for (std::size_t i = 0; i < r.size(); ++i) if (!t.constrained[i]) s += r[i] * r[i];
  return std::sqrt(s);
}

template <int D>
std::vector<double> solve_bvp(System& s, const NewtonConfig& cfg, const double* x0, NewtonReport& rep) {
  cfg.validate();
  validate_dirichlet(s.constraints, s.mesh.n_nodes(), D);
  Timer timer;
  const int64_t n = s.n_dof();
  std::vector<double> u(n, 0.0);
  if (x0) u.assign(x0, x0 + n);
  for (int64_t d = 0; d < n; ++d) if (s.table.constrained[d]) u[d] = s.table.prescribed[d];
  std::vector<double> residual = assemble_residual<D>(s.batches, u.data(), n);
  double rnorm = free_norm(residual, s.table);
  const double r0 = rnorm;
  rep.residual_norms.push_back(rnorm);
  const double target = std::max(cfg.rtol * r0, cfg.atol);
  while (true) {
    if (!std::isfinite(rnorm)) {
      rep.failure = "newton: non-finite residual norm at iteration " + std::to_string(rep.iterations);
      break;
    }
    if (rnorm <= target) { rep.converged = true; break; }
    if (rep.iterations >= cfg.max_iter) {
      rep.failure = "newton: no convergence within " + std::to_string(cfg.max_iter) +
                    " iterations (residual " + std::to_string(rnorm) + ")";
      break;
    }
    std::vector<double> rhs = residual, du;
    SolveReport lin;
    if (cfg.operator_kind == 0) {
      ExplicitOperator op;
      op.p = &s.pattern;
      op.values = assemble_jacobian<D>(s, u.data());
      eliminate_dirichlet(s.pattern, op.values.data(), rhs.data(), s.table, u.data());
      for (double& v : rhs) v = -v;
      du = run_solver(op, rhs.data(), cfg.linear, nullptr, lin);
    } else {
      for (int64_t d = 0; d < n; ++d) if (s.table.constrained[d]) rhs[d] = u[d] - s.table.prescribed[d];
      for (double& v : rhs) v = -v;
      const auto op = make_mf<D>(s, u.data());
      du = run_solver(op, rhs.data(), cfg.linear, nullptr, lin);
    }
    rep.linear_reports.push_back(lin);
    if (!lin.converged) {
      rep.failure = "newton: linear solve failed at iteration " + std::to_string(rep.iterations + 1) +
                    (lin.failure.empty() ? " (tolerance not reached)" : " (" + lin.failure + ")");
      break;
    }
    for (int64_t d = 0; d < n; ++d) u[d] += du[d];
    for (int64_t d = 0; d < n; ++d) if (s.table.constrained[d]) u[d] = s.table.prescribed[d];
    residual = assemble_residual<D>(s.batches, u.data(), n);
    rnorm = free_norm(residual, s.table);
    ++rep.iterations;
    rep.residual_norms.push_back(rnorm);
  }
  rep.total_time = timer.seconds();
  return u;
}

}  // namespace orc
#endif
