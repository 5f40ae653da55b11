// tlfea_oracle.cpp — plain, slow, obviously-correct CPU ORACLE of the hot path
// of arXiv 2604.10357 (TL-FEA Part II), fp64.
//
// *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library. The
// product path (paper_2604_10357_b200 / libtlfea.so) never imports, links or
// calls it, and it shares no code, header, table or helper with the CUDA
// sources. Build: g++ -O2 -ffp-contract=off -std=c++17 -shared -fPIC (the
// all-core CPU baseline: the same source with -fopenmp, liboracle_omp.so;
// only orc_eval_chunked then runs its element loop on several threads).
//
// Citations: "P:n" = line n of PAPER.md (section / equation named); "Qn" =
// reading n of DESIGN.md (= SURVEY §8(c) table). Every function follows the
// textbook definition written out in the paper's notation with per-element
// loops in fixed order (element ascending, q ascending, a/b ascending); no
// blocking, fusion or reordering.
//
// Parity status: every function here is pinned by tests/test_oracle_*.py
// against closed forms, invariants, brute force, finite/complex-step
// differences or the paper's printed tables — except the ANCF3443 basis
// itself, which is pinned only by invariants (reading Q11; Part I, which
// defines the element, is unavailable): "parity unpinned" against the
// paper's own element.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

typedef std::complex<double> cplx;

// ------------------------------------------------------------ quadrature --
// P:390 ("5-point Keast rule", "4x4x3 Gauss-Legendre"); reading Q1.
int quadrature(int rule, double pts[][3], double* w) {
  if (rule == 0) {  // T10 4-point, degree 2: perms of (a,b,b,b), weight 1/24
    const double a = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0;
    const double b = (5.0 - std::sqrt(5.0)) / 20.0;
    for (int k = 0; k < 4; ++k) {
      double z[4] = {b, b, b, b};
      z[k] = a;
      pts[k][0] = z[1]; pts[k][1] = z[2]; pts[k][2] = z[3];   // xi = (z2, z3, z4)
      w[k] = 1.0 / 24.0;
    }
    return 4;
  }
  if (rule == 1) {  // Keast 5-point, degree 3 (S:116 sign convention)
    pts[0][0] = pts[0][1] = pts[0][2] = 0.25;
    w[0] = -4.0 / 5.0 / 6.0;
    for (int k = 0; k < 4; ++k) {
      double z[4] = {1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0};
      z[k] = 0.5;
      pts[1 + k][0] = z[1]; pts[1 + k][1] = z[2]; pts[1 + k][2] = z[3];
      w[1 + k] = 9.0 / 20.0 / 6.0;
    }
    return 5;
  }
  if (rule == 2) {  // Gauss-Legendre 4 x 4 x 3 on [-1,1]^3, xi-major
    const double s = std::sqrt(6.0 / 5.0);
    const double g4[4] = {-std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * s), -std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * s),
                          std::sqrt(3.0 / 7.0 - 2.0 / 7.0 * s), std::sqrt(3.0 / 7.0 + 2.0 / 7.0 * s)};
    const double w4[4] = {(18.0 - std::sqrt(30.0)) / 36.0, (18.0 + std::sqrt(30.0)) / 36.0,
                          (18.0 + std::sqrt(30.0)) / 36.0, (18.0 - std::sqrt(30.0)) / 36.0};
    const double g3[3] = {-std::sqrt(3.0 / 5.0), 0.0, std::sqrt(3.0 / 5.0)};
    const double w3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    int n = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        for (int k = 0; k < 3; ++k) {
          pts[n][0] = g4[i]; pts[n][1] = g4[j]; pts[n][2] = g3[k];
          w[n] = w4[i] * w4[j] * w3[k];
          ++n;
        }
    return n;
  }
  if (rule == 3) {  // Gauss-Legendre 3 x 2 x 2 on [-1,1]^3 (ANCF3243), xi-major
    const double g3[3] = {-std::sqrt(3.0 / 5.0), 0.0, std::sqrt(3.0 / 5.0)};
    const double w3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    const double g2[2] = {-1.0 / std::sqrt(3.0), 1.0 / std::sqrt(3.0)};
    int n = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k) {
          pts[n][0] = g3[i]; pts[n][1] = g2[j]; pts[n][2] = g2[k];
          w[n] = w3[i];
          ++n;
        }
    return n;
  }
  return -1;
}

// -------------------------------------------------------- shape functions --
// T10 (reading Q2): zeta1 = 1-xi-eta-zeta, zeta2..4 = xi, eta, zeta;
// corners N_i = z_i(2 z_i - 1); edge nodes 4 z_a z_b over the edges below.
const int kT10Edge[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};

template <class T>
void t10_shape(const T xi[3], T N[10], T dN[10][3]) {
  T z[4] = {T(1.0) - xi[0] - xi[1] - xi[2], xi[0], xi[1], xi[2]};
  const double dz[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int i = 0; i < 4; ++i) {
    N[i] = z[i] * (2.0 * z[i] - 1.0);
    for (int k = 0; k < 3; ++k) dN[i][k] = (4.0 * z[i] - 1.0) * dz[i][k];
  }
  for (int e = 0; e < 6; ++e) {
    const int a = kT10Edge[e][0], b = kT10Edge[e][1];
    N[4 + e] = 4.0 * z[a] * z[b];
    for (int k = 0; k < 3; ++k) dN[4 + e][k] = 4.0 * (z[b] * dz[a][k] + z[a] * dz[b][k]);
  }
}

// ANCF3443 (reading Q11): node k at (xi_k, eta_k), counter-clockwise from
// (-1,-1); local coefficient 4k+m, m = (r, r_x, r_y, r_z).
const double kAncfNode[4][2] = {{-1, -1}, {1, -1}, {1, 1}, {-1, 1}};

template <class T>
void ancf_shape(const T xi3[3], const double LWH[3], T S[16], T dS[16][3]) {
  const T xi = xi3[0], eta = xi3[1], zeta = xi3[2];
  const double L = LWH[0], W = LWH[1], H = LWH[2];
  for (int k = 0; k < 4; ++k) {
    const double xk = kAncfNode[k][0], ek = kAncfNode[k][1];
    const T a = 1.0 + xk * xi, b = 1.0 + ek * eta;
    const T c = 2.0 + xk * xi + ek * eta - xi * xi - eta * eta;
    // r
    S[4 * k + 0] = 0.125 * a * b * c;
    dS[4 * k + 0][0] = 0.125 * (xk * b * c + a * b * (xk - 2.0 * xi));
    dS[4 * k + 0][1] = 0.125 * (ek * a * c + a * b * (ek - 2.0 * eta));
    dS[4 * k + 0][2] = T(0.0);
    // r_x
    S[4 * k + 1] = (L / 16.0) * xk * (xi * xi - 1.0) * a * b;
    dS[4 * k + 1][0] = (L / 16.0) * xk * (2.0 * xi * a + (xi * xi - 1.0) * xk) * b;
    dS[4 * k + 1][1] = (L / 16.0) * xk * (xi * xi - 1.0) * a * ek;
    dS[4 * k + 1][2] = T(0.0);
    // r_y
    S[4 * k + 2] = (W / 16.0) * ek * (eta * eta - 1.0) * b * a;
    dS[4 * k + 2][0] = (W / 16.0) * ek * (eta * eta - 1.0) * b * xk;
    dS[4 * k + 2][1] = (W / 16.0) * ek * (2.0 * eta * b + (eta * eta - 1.0) * ek) * a;
    dS[4 * k + 2][2] = T(0.0);
    // r_z
    S[4 * k + 3] = (H / 8.0) * zeta * a * b;
    dS[4 * k + 3][0] = (H / 8.0) * zeta * xk * b;
    dS[4 * k + 3][1] = (H / 8.0) * zeta * a * ek;
    dS[4 * k + 3][2] = (H / 8.0) * a * b;
  }
}

// ANCF3243 beam (reading Q23): nodes A (xi = -1) and B (xi = +1), local
// coefficient 4k+m, m = (r, r_x, r_y, r_z); xi, eta, zeta in [-1,1] span L,
// W, H. Cubic Hermite along the axis for (r, r_x), linear for (r_y, r_z):
//   S_r^A = (xi^3 - 3 xi + 2)/4,        S_r^B = (-xi^3 + 3 xi + 2)/4,
//   S_x^A = L (xi^3 - xi^2 - xi + 1)/8,  S_x^B = L (xi^3 + xi^2 - xi - 1)/8,
//   S_y^k = W eta (1 -+ xi)/4,          S_z^k = H zeta (1 -+ xi)/4.
template <class T>
void beam_shape(const T xi3[3], const double LWH[3], T S[8], T dS[8][3]) {
  const T xi = xi3[0], eta = xi3[1], zeta = xi3[2];
  const double L = LWH[0], W = LWH[1], H = LWH[2];
  for (int k = 0; k < 2; ++k) {
    const double s = k == 0 ? -1.0 : 1.0;  // node side
    const T lin = 1.0 + s * xi;             // 1 - xi (A), 1 + xi (B)
    S[4 * k + 0] = 0.25 * (s * (-xi * xi * xi + 3.0 * xi) + 2.0);
    dS[4 * k + 0][0] = 0.25 * s * (-3.0 * xi * xi + 3.0);
    dS[4 * k + 0][1] = T(0.0);
    dS[4 * k + 0][2] = T(0.0);
    S[4 * k + 1] = (L / 8.0) * (xi * xi * xi + s * xi * xi - xi - s);
    dS[4 * k + 1][0] = (L / 8.0) * (3.0 * xi * xi + 2.0 * s * xi - 1.0);
    dS[4 * k + 1][1] = T(0.0);
    dS[4 * k + 1][2] = T(0.0);
    S[4 * k + 2] = (W / 4.0) * eta * lin;
    dS[4 * k + 2][0] = (W / 4.0) * eta * s;
    dS[4 * k + 2][1] = (W / 4.0) * lin;
    dS[4 * k + 2][2] = T(0.0);
    S[4 * k + 3] = (H / 4.0) * zeta * lin;
    dS[4 * k + 3][0] = (H / 4.0) * zeta * s;
    dS[4 * k + 3][1] = T(0.0);
    dS[4 * k + 3][2] = (H / 4.0) * lin;
  }
}

int n_en_of(int elem) { return elem == 0 ? 10 : (elem == 1 ? 16 : 8); }

// Coefficient ids of element e (ANCF: node k -> 4k .. 4k+3; 4 nodes for the
// shell, 2 for the beam).
void elem_coefs(int elem, const int32_t* conn, int64_t e, int64_t out[16]) {
  if (elem == 0) {
    for (int a = 0; a < 10; ++a) out[a] = conn[e * 10 + a];
  } else {
    const int nn = elem == 1 ? 4 : 2;
    for (int k = 0; k < nn; ++k)
      for (int m = 0; m < 4; ++m) out[4 * k + m] = 4 * (int64_t)conn[e * nn + k] + m;
  }
}

// -------------------------------------------------------------- 3x3 algebra --
template <class T> T det3(const T A[9]) {
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}
template <class T> void inv3(const T A[9], T out[9]) {  // adjugate / det
  const T d = det3(A);
  out[0] = (A[4] * A[8] - A[5] * A[7]) / d;
  out[1] = (A[2] * A[7] - A[1] * A[8]) / d;
  out[2] = (A[1] * A[5] - A[2] * A[4]) / d;
  out[3] = (A[5] * A[6] - A[3] * A[8]) / d;
  out[4] = (A[0] * A[8] - A[2] * A[6]) / d;
  out[5] = (A[2] * A[3] - A[0] * A[5]) / d;
  out[6] = (A[3] * A[7] - A[4] * A[6]) / d;
  out[7] = (A[1] * A[6] - A[0] * A[7]) / d;
  out[8] = (A[0] * A[4] - A[1] * A[3]) / d;
}
template <class T> void matmul3(const T A[9], const T B[9], T C[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      T s = T(0.0);
      for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
      C[3 * i + j] = s;
    }
}
template <class T> void transpose3(const T A[9], T B[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) B[3 * i + j] = A[3 * j + i];
}

// -------------------------------------------------------------- materials --
// mat[] = {E, nu, C10, C01, kappa, rho0, eta, lambda_d}; model 0 SVK, 1 MR.
// SVK (reading Q5): E = (F^T F - I)/2, S = lam tr(E) I + 2 mu E, P = F S.
template <class T>
void pk1_svk(const T F[9], double lam, double mu, T P[9]) {
  T Ft[9], C[9], E[9], S[9];
  transpose3(F, Ft);
  matmul3(Ft, F, C);
  for (int i = 0; i < 9; ++i) E[i] = 0.5 * (C[i] - ((i % 4 == 0) ? 1.0 : 0.0));
  const T trE = E[0] + E[4] + E[8];
  for (int i = 0; i < 9; ++i) S[i] = lam * trE * ((i % 4 == 0) ? 1.0 : 0.0) + 2.0 * mu * E[i];
  matmul3(F, S, P);
}
template <class T>
T energy_svk(const T F[9], double lam, double mu) {  // W = lam/2 tr(E)^2 + mu E:E
  T Ft[9], C[9], E[9];
  transpose3(F, Ft);
  matmul3(Ft, F, C);
  for (int i = 0; i < 9; ++i) E[i] = 0.5 * (C[i] - ((i % 4 == 0) ? 1.0 : 0.0));
  const T trE = E[0] + E[4] + E[8];
  T EE = T(0.0);
  for (int i = 0; i < 9; ++i) EE += E[i] * E[i];
  return 0.5 * lam * trE * trE + mu * EE;
}

// Compressible Mooney-Rivlin (reading Q6):
//   W = C10 (I1b - 3) + C01 (I2b - 3) + kappa/2 (J-1)^2,
//   I1b = J^{-2/3} I1, I2b = J^{-4/3} I2, I1 = tr C, I2 = (I1^2 - tr C^2)/2.
// Closed-form second Piola stress (derivative of W w.r.t. E = (C-I)/2):
//   S = 2 C10 J^{-2/3} (I - I1/3 C^{-1}) + 2 C01 J^{-4/3} (I1 I - C - 2 I2/3 C^{-1})
//       + kappa J (J-1) C^{-1},   P = F S.
template <class T>
T energy_mr(const T F[9], double C10, double C01, double kappa) {
  T Ft[9], C[9], C2[9];
  transpose3(F, Ft);
  matmul3(Ft, F, C);
  matmul3(C, C, C2);
  const T J = det3(F);
  const T I1 = C[0] + C[4] + C[8];
  const T I2 = 0.5 * (I1 * I1 - (C2[0] + C2[4] + C2[8]));
  const T Jm23 = std::pow(J, -2.0 / 3.0);
  return C10 * (Jm23 * I1 - 3.0) + C01 * (Jm23 * Jm23 * I2 - 3.0) + 0.5 * kappa * (J - 1.0) * (J - 1.0);
}
template <class T>
void pk1_mr(const T F[9], double C10, double C01, double kappa, T P[9]) {
  T Ft[9], C[9], C2[9], Ci[9], S[9];
  transpose3(F, Ft);
  matmul3(Ft, F, C);
  matmul3(C, C, C2);
  inv3(C, Ci);
  const T J = det3(F);
  const T I1 = C[0] + C[4] + C[8];
  const T I2 = 0.5 * (I1 * I1 - (C2[0] + C2[4] + C2[8]));
  const T Jm23 = std::pow(J, -2.0 / 3.0);
  const T Jm43 = Jm23 * Jm23;
  for (int i = 0; i < 9; ++i) {
    const double Iij = (i % 4 == 0) ? 1.0 : 0.0;
    S[i] = 2.0 * C10 * Jm23 * (Iij - I1 / 3.0 * Ci[i]) +
           2.0 * C01 * Jm43 * (I1 * Iij - C[i] - 2.0 * I2 / 3.0 * Ci[i]) +
           kappa * J * (J - 1.0) * Ci[i];
  }
  matmul3(F, S, P);
}

// Kelvin-Voigt on the Green-Lagrange rate (reading Q7):
//   Edot = (Fdot^T F + F^T Fdot)/2, S_v = 2 eta Edot + lam_d tr(Edot) I, P_v = F S_v.
template <class T>
void pk1_kv(const T F[9], const T Fd[9], double eta, double lamd, T P[9]) {
  T Ft[9], Fdt[9], A[9], B[9], Ed[9], S[9];
  transpose3(F, Ft);
  transpose3(Fd, Fdt);
  matmul3(Fdt, F, A);
  matmul3(Ft, Fd, B);
  for (int i = 0; i < 9; ++i) Ed[i] = 0.5 * (A[i] + B[i]);
  const T tr = Ed[0] + Ed[4] + Ed[8];
  for (int i = 0; i < 9; ++i) S[i] = 2.0 * eta * Ed[i] + lamd * tr * ((i % 4 == 0) ? 1.0 : 0.0);
  matmul3(F, S, P);
}

void lame(const double* mat, double* lam, double* mu) {
  const double E = mat[0], nu = mat[1];
  *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  *mu = E / (2.0 * (1.0 + nu));
}

// Elastic first Piola stress P_el(F).
template <class T>
void pk1_elastic(int model, const double* mat, const T F[9], T P[9]) {
  if (model == 0) {
    double lam, mu;
    lame(mat, &lam, &mu);
    pk1_svk(F, lam, mu, P);
  } else {
    pk1_mr(F, mat[2], mat[3], mat[4], P);
  }
}
template <class T>
T energy_elastic(int model, const double* mat, const T F[9]) {
  if (model == 0) {
    double lam, mu;
    lame(mat, &lam, &mu);
    return energy_svk(F, lam, mu);
  }
  return energy_mr(F, mat[2], mat[3], mat[4]);
}
bool has_kv(const double* mat) { return mat[6] != 0.0 || mat[7] != 0.0; }

// Total P = P_el + P_vis.
void pk1_total(int model, const double* mat, const double F[9], const double* Fd, double P[9]) {
  pk1_elastic(model, mat, F, P);
  if (Fd && has_kv(mat)) {
    double Pv[9];
    pk1_kv(F, Fd, mat[6], mat[7], Pv);
    for (int i = 0; i < 9; ++i) P[i] += Pv[i];
  }
}

// Elastic tangent A_iJkL = dP_iJ / dF_kL by complex-step differentiation of
// pk1_elastic (exact to rounding; independent of any hand-derived tangent).
void tangent_csd(int model, const double* mat, const double F[9], double A[81]) {
  const double hcs = 1e-30;
  for (int kl = 0; kl < 9; ++kl) {
    cplx Fc[9], Pc[9];
    for (int i = 0; i < 9; ++i) Fc[i] = cplx(F[i], 0.0);
    Fc[kl] += cplx(0.0, hcs);
    pk1_elastic(model, mat, Fc, Pc);
    for (int ij = 0; ij < 9; ++ij) A[ij * 9 + kl] = Pc[ij].imag() / hcs;
  }
}

// ----------------------------------------------------- per-(e,q) geometry --
// J = dX/dxi = sum_a X_a (x) dN_a/dxi over ALL element nodes
// (isoparametric, reading Q3); J0 = det J; grad_X N_a = (dN_a/dxi) J^{-1}.
// Returns J0; writes gradN[n_en][3].
double geom_at(int elem, const double* X, const int64_t* cf, const double* LWH,
               const double xi[3], double gradN[16][3], double* Nval) {
  double N[16], dN[16][3];
  const int nen = n_en_of(elem);
  if (elem == 0) {
    double N10[10], dN10[10][3];
    t10_shape(xi, N10, dN10);
    for (int a = 0; a < 10; ++a) {
      N[a] = N10[a];
      for (int k = 0; k < 3; ++k) dN[a][k] = dN10[a][k];
    }
  } else if (elem == 1) {
    ancf_shape(xi, LWH, N, dN);
  } else {
    beam_shape(xi, LWH, N, dN);
  }
  double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int a = 0; a < nen; ++a)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) J[3 * i + j] += X[3 * cf[a] + i] * dN[a][j];
  const double J0 = det3(J);
  double Ji[9];
  inv3(J, Ji);
  for (int a = 0; a < nen; ++a)
    for (int k = 0; k < 3; ++k) {
      double s = 0.0;
      for (int j = 0; j < 3; ++j) s += dN[a][j] * Ji[3 * j + k];
      gradN[a][k] = s;
    }
  if (Nval)
    for (int a = 0; a < nen; ++a) Nval[a] = N[a];
  return J0;
}

const double* dims_of(int elem, const double* dims, int64_t e) {
  return elem != 0 ? dims + 3 * e : nullptr;
}

// ------------------------------------------------------- element routines --
// Element force (Eq. fint_local): f_a = sum_q P grad_X N_a J0 w_q,
// with F = sum_a x_a (x) grad_X N_a (Eq. F_assembly) and
// Fdot = sum_a v_a (x) grad_X N_a.
// Element tangent (Eq. tangent_block):
//   K[3a+i][3b+k] = sum_q sum_JL A_iJkL gradN_aJ gradN_bL J0 w_q (elastic only, Q8).
void element_fK(int elem, int rule, int model, const double* mat, const double* X,
                const int64_t* cf, const double* LWH, const double* x, const double* v,
                double* fe, double* Ke) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem), nd = 3 * nen;
  for (int r = 0; r < nd; ++r) fe[r] = 0.0;
  if (Ke)
    for (int r = 0; r < nd * nd; ++r) Ke[r] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double gN[16][3];
    const double J0 = geom_at(elem, X, cf, LWH, pts[q], gN, nullptr);
    const double J0w = J0 * w[q];
    double F[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, Fd[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i)
        for (int J = 0; J < 3; ++J) {
          F[3 * i + J] += x[3 * cf[a] + i] * gN[a][J];
          if (v) Fd[3 * i + J] += v[3 * cf[a] + i] * gN[a][J];
        }
    double P[9];
    pk1_total(model, mat, F, v ? Fd : nullptr, P);
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i) {
        double s = 0.0;
        for (int J = 0; J < 3; ++J) s += P[3 * i + J] * gN[a][J];
        fe[3 * a + i] += s * J0w;
      }
    if (Ke) {
      double A[81];
      tangent_csd(model, mat, F, A);
      for (int a = 0; a < nen; ++a)
        for (int i = 0; i < 3; ++i)
          for (int b = 0; b < nen; ++b)
            for (int k = 0; k < 3; ++k) {
              double s = 0.0;
              for (int J = 0; J < 3; ++J)
                for (int L = 0; L < 3; ++L) s += A[(3 * i + J) * 9 + 3 * k + L] * gN[a][J] * gN[b][L];
              Ke[(3 * a + i) * nd + 3 * b + k] += s * J0w;
            }
    }
  }
}

// Element internal force f_e[3 nen] (Eq. fint_local) from LOCAL
// coordinates xe and velocities ve [3 nen], generic in the scalar type so the
// complex step can differentiate it: F = sum_a x_a (x) grad N_a, Fdot =
// sum_a v_a (x) grad N_a, P = P_el(F) + P_v(F, Fdot) (Q7, Q9).
template <class T>
void element_force_t(int elem, int rule, int model, const double* mat, const double* X,
                     const int64_t* cf, const double* LWH, const T* xe, const T* ve, T* fe) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem);
  for (int r = 0; r < 3 * nen; ++r) fe[r] = T(0.0);
  for (int q = 0; q < nq; ++q) {
    double gN[16][3];
    const double J0w = geom_at(elem, X, cf, LWH, pts[q], gN, nullptr) * w[q];
    T F[9], Fd[9];
    for (int i = 0; i < 9; ++i) F[i] = Fd[i] = T(0.0);
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i)
        for (int J = 0; J < 3; ++J) {
          F[3 * i + J] += xe[3 * a + i] * gN[a][J];
          Fd[3 * i + J] += ve[3 * a + i] * gN[a][J];
        }
    T P[9], Pv[9];
    pk1_elastic(model, mat, F, P);
    pk1_kv(F, Fd, mat[6], mat[7], Pv);
    for (int i = 0; i < 9; ++i) P[i] += Pv[i];
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i) {
        T s = T(0.0);
        for (int J = 0; J < 3; ++J) s += P[3 * i + J] * gN[a][J];
        fe[3 * a + i] += s * J0w;
      }
  }
}

// Consistent Kelvin-Voigt element tangent (SURVEY §8(f) NEXT-4, P:497-501,
// P:526): the derivative of the element force of the velocity residual
// g(v) = M (v - v_n)/h + f_int(q_n + h v, v) - ... (Eq. residual P:101-113,
// reading Q9) with respect to the element's velocities, x and v moving
// together (dx = h dv):
//   Kc[r][s] = d f_e[r] / d v_e[s] = h df/dx + df/dv
//            = Im f_e(x + i h eps e_s, v + i eps e_s) / eps   (complex step).
// With eta = lambda_d = 0 it is h K_e (the elastic tangent of element_fK).
void element_Kc_csd(int elem, int rule, int model, const double* mat, const double* X,
                    const int64_t* cf, const double* LWH, const double* x, const double* v,
                    double h, double* Kc) {
  const int nen = n_en_of(elem), nd = 3 * nen;
  const double eps = 1e-30;
  std::vector<cplx> xe(nd), ve(nd), fe(nd);
  for (int s = 0; s < nd; ++s) {
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i) {
        xe[3 * a + i] = cplx(x[3 * cf[a] + i], 0.0);
        ve[3 * a + i] = cplx(v ? v[3 * cf[a] + i] : 0.0, 0.0);
      }
    xe[s] += cplx(0.0, h * eps);
    ve[s] += cplx(0.0, eps);
    element_force_t<cplx>(elem, rule, model, mat, X, cf, LWH, xe.data(), ve.data(), fe.data());
    for (int r = 0; r < nd; ++r) Kc[r * nd + s] = fe[r].imag() / eps;
  }
}

// Element strain energy Pi_e = sum_q W(F) J0 w_q (Eq. cost), generic
// in the coordinate scalar type so complex-step d(Pi)/dx can pin the force.
template <class T>
T element_energy_t(int elem, int rule, int model, const double* mat, const double* X,
                   const int64_t* cf, const double* LWH, const T* xe) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem);
  T Pi = T(0.0);
  for (int q = 0; q < nq; ++q) {
    double gN[16][3];
    const double J0 = geom_at(elem, X, cf, LWH, pts[q], gN, nullptr);
    T F[9];
    for (int i = 0; i < 9; ++i) F[i] = T(0.0);
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < 3; ++i)
        for (int J = 0; J < 3; ++J) F[3 * i + J] += xe[3 * a + i] * gN[a][J];
    Pi += energy_elastic(model, mat, F) * (J0 * w[q]);
  }
  return Pi;
}

// Consistent mass: m_ab = int rho0 N_a N_b dV.
//  T10 mass_rule 0 ("exact", reading Q4): closed form of the straight-sided
//    quadratic tetrahedron, rho V / 420 x {corner-corner 6 | 1; corner-edge
//    -4 if the corner is on the edge else -6; edge-edge 32 | 16 sharing a
//    vertex | 8 opposite} (textbook; requires an affine element).
//  otherwise: the element's quadrature rule, sum_q rho0 N_a N_b J0 w_q
//    (P:309-310 literally; for ANCF3443 GL 4x4x3 is exact).
// Gauss-Legendre nodes/weights on [-1,1] by Newton's method on P_n (plain).
void gauss_legendre(int n, double* x, double* w) {
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

bool t10_is_affine(const double* X, const int64_t* cf) {
  double h = 0.0, dev = 0.0;
  for (int m = 0; m < 6; ++m)
    for (int k = 0; k < 3; ++k) {
      const double xa = X[3 * cf[kT10Edge[m][0]] + k], xb = X[3 * cf[kT10Edge[m][1]] + k];
      h = std::max(h, std::fabs(xa - xb));
      dev = std::max(dev, std::fabs(X[3 * cf[4 + m] + k] - 0.5 * (xa + xb)));
    }
  return dev <= 1e-12 * h;
}

void element_mass(int elem, int rule, int mass_rule, double rho, const double* X,
                  const int64_t* cf, const double* LWH, double* me) {
  const int nen = n_en_of(elem);
  if (elem == 0 && mass_rule == 0 && !t10_is_affine(X, cf)) {
    // Exact mass of a curved T10 (reading Q4): N_a N_b det J has degree <= 7;
    // collapsed (Duffy) 6x6x6 Gauss-Legendre rule, exact to degree 9.
    double g[6], gw[6];
    gauss_legendre(6, g, gw);
    for (int r = 0; r < 100; ++r) me[r] = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j)
        for (int k = 0; k < 6; ++k) {
          const double u = 0.5 * (g[i] + 1.0), s = 0.5 * (g[j] + 1.0), t = 0.5 * (g[k] + 1.0);
          const double xi[3] = {u, s * (1.0 - u), t * (1.0 - u) * (1.0 - s)};
          const double wq = 0.125 * gw[i] * gw[j] * gw[k] * (1.0 - u) * (1.0 - u) * (1.0 - s);
          double gN[16][3], N[16];
          const double J0 = geom_at(elem, X, cf, LWH, xi, gN, N);
          for (int a = 0; a < 10; ++a)
            for (int b = 0; b < 10; ++b) me[a * 10 + b] += rho * N[a] * N[b] * J0 * wq;
        }
    return;
  }
  if (elem == 0 && mass_rule == 0) {
    const double* p[4];
    for (int i = 0; i < 4; ++i) p[i] = X + 3 * cf[i];
    double D[9];
    for (int i = 0; i < 3; ++i) {
      D[3 * i + 0] = p[1][i] - p[0][i];
      D[3 * i + 1] = p[2][i] - p[0][i];
      D[3 * i + 2] = p[3][i] - p[0][i];
    }
    const double V = det3(D) / 6.0;
    for (int a = 0; a < 10; ++a)
      for (int b = 0; b < 10; ++b) {
        double m;
        if (a < 4 && b < 4) {
          m = (a == b) ? 6.0 : 1.0;
        } else if (a >= 4 && b >= 4) {
          const int* ea = kT10Edge[a - 4];
          const int* eb = kT10Edge[b - 4];
          const int shared = (ea[0] == eb[0]) + (ea[0] == eb[1]) + (ea[1] == eb[0]) + (ea[1] == eb[1]);
          m = (a == b) ? 32.0 : (shared ? 16.0 : 8.0);
        } else {
          const int c = a < 4 ? a : b;
          const int* ed = kT10Edge[(a < 4 ? b : a) - 4];
          m = (ed[0] == c || ed[1] == c) ? -4.0 : -6.0;
        }
        me[a * 10 + b] = rho * V / 420.0 * m;
      }
    return;
  }
  double pts[48][3], w[48];
  int nq = quadrature(rule, pts, w);
  if (elem == 2 && mass_rule == 0) {
    // exact beam mass (reading Q4 / Q23): N_a N_b det J has degree <= 10 in
    // xi and <= 3 in eta, zeta -> Gauss-Legendre 6 x 2 x 2
    double g6[6], w6[6];
    gauss_legendre(6, g6, w6);
    const double g2 = 1.0 / std::sqrt(3.0);
    nq = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k) {
          pts[nq][0] = g6[i]; pts[nq][1] = j ? g2 : -g2; pts[nq][2] = k ? g2 : -g2;
          w[nq] = w6[i];
          ++nq;
        }
  }
  for (int r = 0; r < nen * nen; ++r) me[r] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double gN[16][3], N[16];
    const double J0 = geom_at(elem, X, cf, LWH, pts[q], gN, N);
    for (int a = 0; a < nen; ++a)
      for (int b = 0; b < nen; ++b) me[a * nen + b] += rho * N[a] * N[b] * J0 * w[q];
  }
}

int64_t find_col(const int64_t* cols, int64_t lo, int64_t hi, int64_t c) {
  const int64_t* it = std::lower_bound(cols + lo, cols + hi, c);
  if (it == cols + hi || *it != c) return -1;
  return it - cols;
}

}  // namespace

// =========================================================== C interface ==
extern "C" {

int orc_quadrature(int rule, double* pts, double* w) {
  double p[48][3];
  const int n = quadrature(rule, p, w);
  for (int q = 0; q < n; ++q)
    for (int k = 0; k < 3; ++k) pts[3 * q + k] = p[q][k];
  return n;
}

void orc_t10_shape(const double* xi, double* N, double* dN) {
  double d[10][3];
  t10_shape(xi, N, d);
  for (int a = 0; a < 10; ++a)
    for (int k = 0; k < 3; ++k) dN[3 * a + k] = d[a][k];
}

// Complex-step probe of the T10 basis: returns Im N(xi + i h e_dir)/h.
void orc_t10_shape_csd(const double* xi, int dir, double* dNdir) {
  cplx x[3] = {xi[0], xi[1], xi[2]}, N[10], d[10][3];
  x[dir] += cplx(0.0, 1e-30);
  t10_shape(x, N, d);
  for (int a = 0; a < 10; ++a) dNdir[a] = N[a].imag() / 1e-30;
}

void orc_ancf_shape(const double* xi, const double* LWH, double* S, double* dS) {
  double d[16][3];
  ancf_shape(xi, LWH, S, d);
  for (int a = 0; a < 16; ++a)
    for (int k = 0; k < 3; ++k) dS[3 * a + k] = d[a][k];
}

void orc_ancf_shape_csd(const double* xi, const double* LWH, int dir, double* dSdir) {
  cplx x[3] = {xi[0], xi[1], xi[2]}, S[16], d[16][3];
  x[dir] += cplx(0.0, 1e-30);
  ancf_shape(x, LWH, S, d);
  for (int a = 0; a < 16; ++a) dSdir[a] = S[a].imag() / 1e-30;
}

void orc_beam_shape(const double* xi, const double* LWH, double* S, double* dS) {
  double d[8][3];
  beam_shape(xi, LWH, S, d);
  for (int a = 0; a < 8; ++a)
    for (int k = 0; k < 3; ++k) dS[3 * a + k] = d[a][k];
}

void orc_beam_shape_csd(const double* xi, const double* LWH, int dir, double* dSdir) {
  cplx x[3] = {xi[0], xi[1], xi[2]}, S[8], d[8][3];
  x[dir] += cplx(0.0, 1e-30);
  beam_shape(x, LWH, S, d);
  for (int a = 0; a < 8; ++a) dSdir[a] = S[a].imag() / 1e-30;
}

// a-1: gradN [n_el][nq][nen][3], J0w [n_el][nq]. Returns -1 on
// success or the first element with J0 <= 0.
int64_t orc_precompute(int elem, int rule, int64_t n_el, const int32_t* conn, const double* X,
                       const double* dims, double* gradN, double* J0w) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem);
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    for (int q = 0; q < nq; ++q) {
      double gN[16][3];
      const double J0 = geom_at(elem, X, cf, dims_of(elem, dims, e), pts[q], gN, nullptr);
      if (!(J0 > 0.0)) return e;
      for (int a = 0; a < nen; ++a)
        for (int k = 0; k < 3; ++k) gradN[((e * nq + q) * nen + a) * 3 + k] = gN[a][k];
      J0w[e * nq + q] = J0 * w[q];
    }
  }
  return -1;
}

// a-2 pattern: keys I*2^32 + J for every element-local pair,
// sorted and de-duplicated; rowptr by counting. Two calls: with rowptr==NULL
// returns nnz; otherwise fills rowptr [n_coef+1] and cols [nnz].
int64_t orc_coef_pattern(int elem, int64_t n_el, const int32_t* conn, int64_t n_coef,
                         int64_t* rowptr, int64_t* cols) {
  const int nen = n_en_of(elem);
  std::vector<uint64_t> keys;
  keys.reserve((size_t)n_el * nen * nen);
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    for (int a = 0; a < nen; ++a)
      for (int b = 0; b < nen; ++b) keys.push_back(((uint64_t)cf[a] << 32) | (uint64_t)cf[b]);
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  const int64_t nnz = (int64_t)keys.size();
  if (!rowptr) return nnz;
  for (int64_t i = 0; i <= n_coef; ++i) rowptr[i] = 0;
  for (int64_t p = 0; p < nnz; ++p) {
    rowptr[(keys[p] >> 32) + 1] += 1;
    cols[p] = (int64_t)(keys[p] & 0xffffffffu);
  }
  for (int64_t i = 0; i < n_coef; ++i) rowptr[i + 1] += rowptr[i];
  return nnz;
}

// a-2 lift: DOF row 3I+d holds columns 3J+e, J over the sorted
// coefficient columns of row I, then e = 0,1,2.
void orc_lift(int64_t n_coef, const int64_t* rowptr_c, const int64_t* cols_c, int64_t* rowptr,
              int64_t* cols) {
  int64_t p = 0;
  rowptr[0] = 0;
  for (int64_t I = 0; I < n_coef; ++I)
    for (int d = 0; d < 3; ++d) {
      for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k)
        for (int e = 0; e < 3; ++e) cols[p++] = 3 * cols_c[k] + e;
      rowptr[3 * I + d + 1] = p;
    }
}

// a-2 slot map (reading Q16): slots[e][3a+d][3b+f] = CSR index of
// (3 conn[e][a] + d, 3 conn[e][b] + f), by binary search in the row.
void orc_slot_map(int elem, int64_t n_el, const int32_t* conn, const int64_t* rowptr,
                  const int64_t* cols, int64_t* slots) {
  const int nen = n_en_of(elem), nd = 3 * nen;
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    for (int a = 0; a < nen; ++a)
      for (int d = 0; d < 3; ++d)
        for (int b = 0; b < nen; ++b)
          for (int f = 0; f < 3; ++f) {
            const int64_t r = 3 * cf[a] + d;
            slots[(e * nd + 3 * a + d) * nd + 3 * b + f] = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cf[b] + f);
          }
  }
}

// a-2 mass on the coefficient pattern, element order.
void orc_mass(int elem, int rule, int mass_rule, double rho, int64_t n_el, const int32_t* conn,
              const double* X, const double* dims, int64_t n_coef, const int64_t* rowptr_c,
              const int64_t* cols_c, double* M) {
  const int nen = n_en_of(elem);
  for (int64_t p = 0; p < rowptr_c[n_coef]; ++p) M[p] = 0.0;
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    double me[256];
    element_mass(elem, rule, mass_rule, rho, X, cf, dims_of(elem, dims, e), me);
    for (int a = 0; a < nen; ++a)
      for (int b = 0; b < nen; ++b) {
        const int64_t p = find_col(cols_c, rowptr_c[cf[a]], rowptr_c[cf[a] + 1], cf[b]);
        M[p] += me[a * nen + b];
      }
  }
}

void orc_element_mass(int elem, int rule, int mass_rule, double rho, const int32_t* conn_e,
                      const double* X, const double* LWH, double* me) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  element_mass(elem, rule, mass_rule, rho, X, cf, LWH, me);
}

// f_ff[3I+d] = g_d sum_J M_IJ (reading Q10).
void orc_force_field(int64_t n_coef, const int64_t* rowptr_c, const double* M, const double* g,
                     double* fff) {
  for (int64_t I = 0; I < n_coef; ++I) {
    double s = 0.0;
    for (int64_t p = rowptr_c[I]; p < rowptr_c[I + 1]; ++p) s += M[p];
    for (int d = 0; d < 3; ++d) fff[3 * I + d] = g[d] * s;
  }
}

// Constitutive functions: mat = {E, nu, C10, C01, kappa, rho0, eta, lambda_d}.
void orc_pk1(int model, const double* mat, const double* F, const double* Fd, double* P) {
  pk1_total(model, mat, F, Fd, P);
}
void orc_pk1_elastic(int model, const double* mat, const double* F, double* P) {
  pk1_elastic(model, mat, F, P);
}
void orc_pk1_viscous(const double* mat, const double* F, const double* Fd, double* P) {
  pk1_kv(F, Fd, mat[6], mat[7], P);
}
double orc_energy(int model, const double* mat, const double* F) {
  return energy_elastic(model, mat, F);
}
// Complex-step derivative of W: dW/dF [9] (pins the closed-form P).
void orc_energy_grad_csd(int model, const double* mat, const double* F, double* dW) {
  for (int kl = 0; kl < 9; ++kl) {
    cplx Fc[9];
    for (int i = 0; i < 9; ++i) Fc[i] = F[i];
    Fc[kl] += cplx(0.0, 1e-30);
    dW[kl] = energy_elastic(model, mat, Fc).imag() / 1e-30;
  }
}
void orc_tangent(int model, const double* mat, const double* F, double* A) {
  tangent_csd(model, mat, F, A);
}

// One element: fe [3nen], Ke [(3nen)^2] (nullable). conn_e = this element's
// connectivity row (10 node ids, or 4 for ANCF); xe/ve are GLOBAL arrays.
void orc_element(int elem, int rule, int model, const double* mat, const int32_t* conn_e,
                 const double* X, const double* LWH, const double* x, const double* v, double* fe,
                 double* Ke) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  element_fK(elem, rule, model, mat, X, cf, LWH, x, v, fe, Ke);
}

// Element force from LOCAL xe, ve [3 nen] (for FD pins of the consistent tangent).
void orc_element_force_local(int elem, int rule, int model, const double* mat, const int32_t* conn_e,
                             const double* X, const double* LWH, const double* xe, const double* ve,
                             double* fe) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  element_force_t<double>(elem, rule, model, mat, X, cf, LWH, xe, ve, fe);
}
// Consistent Kelvin-Voigt element tangent Kc [3 nen][3 nen] (x, v global).
void orc_element_kvc(int elem, int rule, int model, const double* mat, const int32_t* conn_e,
                     const double* X, const double* LWH, const double* x, const double* v, double h,
                     double* Kc) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  element_Kc_csd(elem, rule, model, mat, X, cf, LWH, x, v, h, Kc);
}

// Element energy with LOCAL coordinates xe [3 nen] (for FD / CSD pins).
double orc_element_energy(int elem, int rule, int model, const double* mat, const int32_t* conn_e,
                          const double* X, const double* LWH, const double* xe) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  return element_energy_t<double>(elem, rule, model, mat, X, cf, LWH, xe);
}
// d(Pi_e)/d(xe) by complex step, [3 nen].
void orc_element_energy_grad_csd(int elem, int rule, int model, const double* mat,
                                 const int32_t* conn_e, const double* X, const double* LWH,
                                 const double* xe, double* grad) {
  int64_t cf[16];
  elem_coefs(elem, conn_e, 0, cf);
  const int nd = 3 * n_en_of(elem);
  for (int r = 0; r < nd; ++r) {
    std::vector<cplx> xc(nd);
    for (int s = 0; s < nd; ++s) xc[s] = xe[s];
    xc[r] += cplx(0.0, 1e-30);
    grad[r] = element_energy_t<cplx>(elem, rule, model, mat, X, cf, LWH, xc.data()).imag() / 1e-30;
  }
}

// Stage 1 alone: P [n_el][nq][9] = P_el + P_vis.
void orc_stress(int elem, int rule, int model, const double* mat, int64_t n_el, const int32_t* conn,
                const double* X, const double* dims, const double* x, const double* v, double* Pout) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem);
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    for (int q = 0; q < nq; ++q) {
      double gN[16][3];
      geom_at(elem, X, cf, dims_of(elem, dims, e), pts[q], gN, nullptr);
      double F[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, Fd[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int a = 0; a < nen; ++a)
        for (int i = 0; i < 3; ++i)
          for (int J = 0; J < 3; ++J) {
            F[3 * i + J] += x[3 * cf[a] + i] * gN[a][J];
            if (v) Fd[3 * i + J] += v[3 * cf[a] + i] * gN[a][J];
          }
      pk1_total(model, mat, F, v ? Fd : nullptr, Pout + (e * nq + q) * 9);
    }
  }
}

// Stage 2 force from a stress buffer (Eqs. fint_local / fint_global).
void orc_force_from_stress(int elem, int rule, int64_t n_el, const int32_t* conn, const double* X,
                           const double* dims, const double* Pbuf, int64_t n_coef, double* fint) {
  double pts[48][3], w[48];
  const int nq = quadrature(rule, pts, w);
  const int nen = n_en_of(elem);
  for (int64_t i = 0; i < 3 * n_coef; ++i) fint[i] = 0.0;
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    for (int q = 0; q < nq; ++q) {
      double gN[16][3];
      const double J0 = geom_at(elem, X, cf, dims_of(elem, dims, e), pts[q], gN, nullptr);
      const double* P = Pbuf + (e * nq + q) * 9;
      for (int a = 0; a < nen; ++a)
        for (int i = 0; i < 3; ++i) {
          double s = 0.0;
          for (int J = 0; J < 3; ++J) s += P[3 * i + J] * gN[a][J];
          fint[3 * cf[a] + i] += s * J0 * w[q];
        }
    }
  }
}

// Full evaluation (Alg. 3 assembly; Eq. residual, Eq. hessian
// P:495-501), element order, on the full DOF CSR (rowptr, cols):
//   f_int[3I+d] += f_e[a][d];  H[slot] += h K_e[r][s];
//   H(3I+d, 3J+d) += M_IJ / h;  g = (1/h) M (v - v_n) + f_int - f_ext - f_ff.
// H may be NULL (force-only). v_n, f_ext, fff may be NULL (= 0).
void orc_eval(int elem, int rule, int model, const double* mat, int64_t n_el, const int32_t* conn,
              int64_t n_coef, const double* X, const double* dims, const int64_t* rowptr_c,
              const int64_t* cols_c, const double* M, const double* fff, const int64_t* rowptr,
              const int64_t* cols, const double* x, const double* v, const double* vn,
              const double* fext, double h, double* g, double* H, double* fint) {
  const int nen = n_en_of(elem), nd = 3 * nen;
  const int64_t ndof = 3 * n_coef;
  for (int64_t i = 0; i < ndof; ++i) fint[i] = 0.0;
  if (H)
    for (int64_t p = 0; p < rowptr[ndof]; ++p) H[p] = 0.0;
  std::vector<double> fe(nd), Ke((size_t)nd * nd);
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    element_fK(elem, rule, model, mat, X, cf, dims_of(elem, dims, e), x, v, fe.data(),
               H ? Ke.data() : nullptr);
    for (int a = 0; a < nen; ++a)
      for (int d = 0; d < 3; ++d) fint[3 * cf[a] + d] += fe[3 * a + d];
    if (H)
      for (int a = 0; a < nen; ++a)
        for (int d = 0; d < 3; ++d)
          for (int b = 0; b < nen; ++b)
            for (int f = 0; f < 3; ++f) {
              const int64_t r = 3 * cf[a] + d;
              const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cf[b] + f);
              H[p] += h * Ke[(3 * a + d) * nd + 3 * b + f];
            }
  }
  if (H)
    for (int64_t I = 0; I < n_coef; ++I)
      for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k)
        for (int d = 0; d < 3; ++d) {
          const int64_t r = 3 * I + d;
          const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cols_c[k] + d);
          H[p] += M[k] / h;
        }
  if (g)
    for (int64_t I = 0; I < n_coef; ++I)
      for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k) {
          const int64_t J = cols_c[k];
          s += M[k] * (v[3 * J + d] - (vn ? vn[3 * J + d] : 0.0));
        }
        const int64_t i = 3 * I + d;
        g[i] = s / h + fint[i] - (fext ? fext[i] : 0.0) - (fff ? fff[i] : 0.0);
      }
}

// The evaluation with the CONSISTENT Kelvin-Voigt tangent (NEXT-4): g and
// f_int exactly as orc_eval, and
//   H = M/h + sum_e Kc_e,   Kc_e = h df_e/dx + df_e/dv   (element_Kc_csd),
// i.e. H = dg/dv of Eq. residual with x = q_n + h v; in general
// non-symmetric. Element order, full DOF CSR (rowptr, cols).
void orc_eval_kvc(int elem, int rule, int model, const double* mat, int64_t n_el, const int32_t* conn,
                  int64_t n_coef, const double* X, const double* dims, const int64_t* rowptr_c,
                  const int64_t* cols_c, const double* M, const double* fff, const int64_t* rowptr,
                  const int64_t* cols, const double* x, const double* v, const double* vn,
                  const double* fext, double h, double* g, double* H, double* fint) {
  orc_eval(elem, rule, model, mat, n_el, conn, n_coef, X, dims, rowptr_c, cols_c, M, fff, rowptr, cols,
           x, v, vn, fext, h, g, nullptr, fint);
  const int nen = n_en_of(elem), nd = 3 * nen;
  const int64_t ndof = 3 * n_coef;
  for (int64_t p = 0; p < rowptr[ndof]; ++p) H[p] = 0.0;
  std::vector<double> Kc((size_t)nd * nd);
  for (int64_t e = 0; e < n_el; ++e) {
    int64_t cf[16];
    elem_coefs(elem, conn, e, cf);
    element_Kc_csd(elem, rule, model, mat, X, cf, dims_of(elem, dims, e), x, v, h, Kc.data());
    for (int a = 0; a < nen; ++a)
      for (int d = 0; d < 3; ++d)
        for (int b = 0; b < nen; ++b)
          for (int f = 0; f < 3; ++f) {
            const int64_t r = 3 * cf[a] + d;
            const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cf[b] + f);
            H[p] += Kc[(3 * a + d) * nd + 3 * b + f];
          }
  }
  for (int64_t I = 0; I < n_coef; ++I)
    for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k)
      for (int d = 0; d < 3; ++d) {
        const int64_t r = 3 * I + d;
        const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cols_c[k] + d);
        H[p] += M[k] / h;
      }
}

// The same evaluation with the element routine run on all host cores
// (the all-core CPU baseline): elements are computed in
// chunks, in parallel (OpenMP build liboracle_omp.so; a plain build runs the
// loop serially), each into its own slot of a chunk buffer (thread-private
// element blocks), and the chunk is then assembled in ascending element order
// exactly as orc_eval does. The arithmetic and the summation order are those
// of orc_eval, so the results are bitwise equal to it.
void orc_eval_chunked(int elem, int rule, int model, const double* mat, int64_t n_el, const int32_t* conn,
                      int64_t n_coef, const double* X, const double* dims, const int64_t* rowptr_c,
                      const int64_t* cols_c, const double* M, const double* fff, const int64_t* rowptr,
                      const int64_t* cols, const double* x, const double* v, const double* vn,
                      const double* fext, double h, double* g, double* H, double* fint) {
  const int nen = n_en_of(elem), nd = 3 * nen;
  const int64_t ndof = 3 * n_coef, chunk = 2048;
  for (int64_t i = 0; i < ndof; ++i) fint[i] = 0.0;
  if (H)
    for (int64_t p = 0; p < rowptr[ndof]; ++p) H[p] = 0.0;
  std::vector<double> fe((size_t)chunk * nd), Ke(H ? (size_t)chunk * nd * nd : 0);
  for (int64_t e0 = 0; e0 < n_el; e0 += chunk) {
    const int64_t ne = std::min(chunk, n_el - e0);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = 0; k < ne; ++k) {
      int64_t cf[16];
      elem_coefs(elem, conn, e0 + k, cf);
      element_fK(elem, rule, model, mat, X, cf, dims_of(elem, dims, e0 + k), x, v, &fe[(size_t)k * nd],
                 H ? &Ke[(size_t)k * nd * nd] : nullptr);
    }
    // merge: thread th owns the nodes I with I % nt == th and adds the chunk's
    // element blocks to their rows in ascending element order (the serial order)
#pragma omp parallel
    {
      int nt = 1, th = 0;
#ifdef _OPENMP
      nt = omp_get_num_threads();
      th = omp_get_thread_num();
#endif
      for (int64_t k = 0; k < ne; ++k) {
        int64_t cf[16];
        elem_coefs(elem, conn, e0 + k, cf);
        const double* fk = &fe[(size_t)k * nd];
        const double* Kk = H ? &Ke[(size_t)k * nd * nd] : nullptr;
        for (int a = 0; a < nen; ++a)
          for (int d = 0; d < 3; ++d) {
            const int64_t r = 3 * cf[a] + d;
            if (cf[a] % nt != th) continue;
            fint[r] += fk[3 * a + d];
            if (H)
              for (int b = 0; b < nen; ++b)
                for (int f = 0; f < 3; ++f) {
                  const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cf[b] + f);
                  H[p] += h * Kk[(3 * a + d) * nd + 3 * b + f];
                }
          }
      }
    }
  }
  if (H)
#pragma omp parallel for schedule(static)
    for (int64_t I = 0; I < n_coef; ++I)
      for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k)
        for (int d = 0; d < 3; ++d) {
          const int64_t r = 3 * I + d;
          const int64_t p = find_col(cols, rowptr[r], rowptr[r + 1], 3 * cols_c[k] + d);
          H[p] += M[k] / h;
        }
  if (g)
#pragma omp parallel for schedule(static)
    for (int64_t I = 0; I < n_coef; ++I)
      for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int64_t k = rowptr_c[I]; k < rowptr_c[I + 1]; ++k) {
          const int64_t J = cols_c[k];
          s += M[k] * (v[3 * J + d] - (vn ? vn[3 * J + d] : 0.0));
        }
        const int64_t i = 3 * I + d;
        g[i] = s / h + fint[i] - (fext ? fext[i] : 0.0) - (fff ? fff[i] : 0.0);
      }
}

int orc_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// Sampled rows (for parity at sizes the full oracle cannot hold): for each
// coefficient node in `nodes` (n_s of them), the assembled f_int (3), the
// H row-block as dense coefficient-column lists. The caller provides
// incidence: inc_ptr [n_s+1], inc_elem [...] = ascending element ids that
// contain node s. Outputs: cols_out [n_s][max_cols] coefficient columns
// ascending (-1 padded), H_out [n_s][3][max_cols][3] (= H(3I+d, 3J+f) for
// J = cols_out), fint_out [n_s][3], mass_out [n_s][max_cols] = M_IJ.
// Returns the max number of columns needed (call again with a larger
// max_cols if it exceeds the given one).
int64_t orc_eval_rows(int elem, int rule, int mass_rule, int model, const double* mat,
                      const int32_t* conn, const double* X, const double* dims, const double* x,
                      const double* v, double h, int64_t n_s, const int64_t* nodes,
                      const int64_t* inc_ptr, const int64_t* inc_elem, int64_t max_cols,
                      int64_t* cols_out, double* H_out, double* fint_out, double* mass_out) {
  const int nen = n_en_of(elem), nd = 3 * nen;
  int64_t need = 0;
  std::vector<double> fe(nd), Ke((size_t)nd * nd), me((size_t)nen * nen);
  for (int64_t s = 0; s < n_s; ++s) {
    const int64_t I = nodes[s];
    std::vector<int64_t> colset;
    for (int64_t t = inc_ptr[s]; t < inc_ptr[s + 1]; ++t) {
      int64_t cf[16];
      elem_coefs(elem, conn, inc_elem[t], cf);
      for (int b = 0; b < nen; ++b) colset.push_back(cf[b]);
    }
    std::sort(colset.begin(), colset.end());
    colset.erase(std::unique(colset.begin(), colset.end()), colset.end());
    const int64_t nc = (int64_t)colset.size();
    need = std::max(need, nc);
    if (nc > max_cols) continue;
    for (int64_t c = 0; c < max_cols; ++c) cols_out[s * max_cols + c] = c < nc ? colset[c] : -1;
    double* Hs = H_out + s * 9 * max_cols;
    for (int64_t c = 0; c < 9 * max_cols; ++c) Hs[c] = 0.0;
    for (int64_t c = 0; c < max_cols; ++c) mass_out[s * max_cols + c] = 0.0;
    for (int d = 0; d < 3; ++d) fint_out[3 * s + d] = 0.0;
    for (int64_t t = inc_ptr[s]; t < inc_ptr[s + 1]; ++t) {
      const int64_t e = inc_elem[t];
      int64_t cf[16];
      elem_coefs(elem, conn, e, cf);
      element_fK(elem, rule, model, mat, X, cf, dims_of(elem, dims, e), x, v, fe.data(), Ke.data());
      element_mass(elem, rule, mass_rule, mat[5], X, cf, dims_of(elem, dims, e), me.data());
      for (int a = 0; a < nen; ++a) {
        if (cf[a] != I) continue;
        for (int d = 0; d < 3; ++d) fint_out[3 * s + d] += fe[3 * a + d];
        for (int b = 0; b < nen; ++b) {
          const int64_t c = std::lower_bound(colset.begin(), colset.end(), cf[b]) - colset.begin();
          mass_out[s * max_cols + c] += me[a * nen + b];
          for (int d = 0; d < 3; ++d)
            for (int f = 0; f < 3; ++f)
              Hs[(d * max_cols + c) * 3 + f] += h * Ke[(3 * a + d) * nd + 3 * b + f];
        }
      }
    }
    for (int64_t c = 0; c < nc; ++c)
      for (int d = 0; d < 3; ++d) Hs[(d * max_cols + c) * 3 + d] += mass_out[s * max_cols + c] / h;
  }
  return need;
}

// AdamW velocity update of inner iteration l (Alg. 2), one DOF at a
// time in the algorithm's order: first moment, second moment, bias correction,
// velocity update with decoupled weight decay, backward-Euler step map.
// prm = (alpha, beta1, beta2, eps, weight_decay). m, s, v updated in place.
void orc_adamw_update(int64_t n, int l, const double* prm, const double* g, double* m, double* s, double* v,
                      const double* q_n, double h, double* q) {
  const double alpha = prm[0], b1 = prm[1], b2 = prm[2], eps = prm[3], wd = prm[4];
  const double c1 = 1.0 - std::pow(b1, l), c2 = 1.0 - std::pow(b2, l);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];                   // first moment
    s[i] = b2 * s[i] + (1.0 - b2) * g[i] * g[i];            // second moment
    const double mh = m[i] / c1, sh = s[i] / c2;            // bias correction
    v[i] = (1.0 - alpha * wd) * v[i] - alpha * mh / (std::sqrt(sh) + eps);  // velocity update
    q[i] = q_n[i] + h * v[i];                               // q = q_n + h v
  }
}

}  // extern "C"
