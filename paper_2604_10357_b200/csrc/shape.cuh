// shape.cuh — quadrature rules and element shape functions of libtlfea.
//  T10 quadratic tetrahedron: corners N_i = z_i (2 z_i - 1), edges 4 z_a z_b,
//    z = (1-xi-eta-zeta, xi, eta, zeta), edges (0,1),(1,2),(2,0),(0,3),(1,3),(2,3)
//    (§4.1; local order: DESIGN.md reading Q2).
//  ANCF3443 shell: 4 nodes x (r, r_x, r_y, r_z), incomplete-bicubic plate basis
//    (reading Q11; the element of P:390).
//  Rules: T10 4-point (degree 2), Keast 5-point (degree 3, negative
//    centroid weight), Gauss-Legendre 4x4x3 for the shell (xi-major).
#pragma once
#include <cmath>

namespace tlfea {

// Host: fill a rule; returns the number of points.
inline int make_rule(int rule, double* xi /*[n][3]*/, double* w) {
  if (rule == TLFEA_Q_T10_4PT) {
    const double r5 = std::sqrt(5.0);
    const double alpha = 0.25 + 0.15 * r5;     // (5 + 3 sqrt5)/20
    const double beta = 0.25 - 0.05 * r5;      // (5 - sqrt5)/20
    for (int p = 0; p < 4; ++p) {
      double bary[4] = {beta, beta, beta, beta};
      bary[p] = alpha;
      xi[3 * p + 0] = bary[1];
      xi[3 * p + 1] = bary[2];
      xi[3 * p + 2] = bary[3];
      w[p] = 1.0 / 24.0;
    }
    return 4;
  }
  if (rule == TLFEA_Q_T10_KEAST5) {
    xi[0] = xi[1] = xi[2] = 0.25;
    w[0] = -2.0 / 15.0;
    for (int p = 0; p < 4; ++p) {
      double bary[4] = {1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0};
      bary[p] = 0.5;
      xi[3 * (p + 1) + 0] = bary[1];
      xi[3 * (p + 1) + 1] = bary[2];
      xi[3 * (p + 1) + 2] = bary[3];
      w[p + 1] = 3.0 / 40.0;
    }
    return 5;
  }
  if (rule == TLFEA_Q_GL_3x2x2) {  // beam: 3 points along the axis, 2 x 2 over the section
    const double p3[3] = {-std::sqrt(0.6), 0.0, std::sqrt(0.6)}, q3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    const double p2 = 1.0 / std::sqrt(3.0);
    int n = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k, ++n) {
          xi[3 * n + 0] = p3[i];
          xi[3 * n + 1] = j ? p2 : -p2;
          xi[3 * n + 2] = k ? p2 : -p2;
          w[n] = q3[i];
        }
    return n;
  }
  // Gauss-Legendre: 4 points (roots of P4), 3 points (roots of P3)
  const double t = 2.0 * std::sqrt(1.2) / 7.0;
  const double x4o = std::sqrt(3.0 / 7.0 + t), x4i = std::sqrt(3.0 / 7.0 - t);
  const double w4o = 0.5 - std::sqrt(30.0) / 36.0, w4i = 0.5 + std::sqrt(30.0) / 36.0;
  const double p4[4] = {-x4o, -x4i, x4i, x4o}, q4[4] = {w4o, w4i, w4i, w4o};
  const double p3[3] = {-std::sqrt(0.6), 0.0, std::sqrt(0.6)}, q3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  int n = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 3; ++k, ++n) {
        xi[3 * n + 0] = p4[i];
        xi[3 * n + 1] = p4[j];
        xi[3 * n + 2] = p3[k];
        w[n] = q4[i] * q4[j] * q3[k];
      }
  return n;
}

// Host: collapsed (Duffy) Gauss rule with 5 points per direction on the unit
// tetrahedron: exact for polynomials of total degree <= 7, i.e. for
// N_a N_b det J of curved (isoparametric) T10 elements; used for the exact
// consistent mass (reading Q4). 125 points.
constexpr int kMassRuleT10 = 125;
inline int make_mass_rule_t10(double* xi, double* w) {
  const double r = 2.0 * std::sqrt(10.0 / 7.0);
  const double xo = std::sqrt(5.0 + r) / 3.0, xi_ = std::sqrt(5.0 - r) / 3.0;
  const double wo = (322.0 - 13.0 * std::sqrt(70.0)) / 900.0, wi = (322.0 + 13.0 * std::sqrt(70.0)) / 900.0;
  const double g[5] = {-xo, -xi_, 0.0, xi_, xo}, gw[5] = {wo, wi, 128.0 / 225.0, wi, wo};
  int n = 0;
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j)
      for (int k = 0; k < 5; ++k, ++n) {
        const double u = 0.5 * (g[i] + 1.0), s = 0.5 * (g[j] + 1.0), r = 0.5 * (g[k] + 1.0);
        xi[3 * n + 0] = u;
        xi[3 * n + 1] = s * (1.0 - u);
        xi[3 * n + 2] = r * (1.0 - u) * (1.0 - s);
        w[n] = gw[i] * gw[j] * gw[k] * 0.125 * (1.0 - u) * (1.0 - u) * (1.0 - s);
      }
  return n;
}

// Host: exact consistent-mass rule of the ANCF3243 beam (reading Q23):
// N_a N_b det J has degree <= 10 along the axis and <= 3 across the section
// -> Gauss-Legendre 6 x 2 x 2 (24 points).
constexpr int kMassRuleBeam = 24;
inline int make_mass_rule_beam(double* xi, double* w) {
  const double g6[6] = {-0.9324695142031519, -0.6612093864662645, -0.2386191860831969,
                        0.2386191860831969,  0.6612093864662645,  0.9324695142031519};
  const double w6[6] = {0.17132449237917027, 0.3607615730481387, 0.46791393457269104,
                        0.46791393457269104, 0.3607615730481387, 0.17132449237917027};
  const double p2 = 1.0 / std::sqrt(3.0);
  int n = 0;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 2; ++j)
      for (int k = 0; k < 2; ++k, ++n) {
        xi[3 * n + 0] = g6[i];
        xi[3 * n + 1] = j ? p2 : -p2;
        xi[3 * n + 2] = k ? p2 : -p2;
        w[n] = w6[i];
      }
  return n;
}

// Device/host: ANCF3243 beam values and parent gradients (reading Q23). With
// s = (1 + xi)/2 along the axis: cubic Hermite h00, L h10 (node A) and h01,
// L h11 (node B) for (r, r_x); (W/2) eta and (H/2) zeta times (1 - s) / s for
// (r_y, r_z). Local coefficient 4k + m, k = A, B, m = (r, r_x, r_y, r_z).
__host__ __device__ inline void beam_shape(const double* xi3, const double* LWH, double* S, double (*dS)[3]) {
  const double s = 0.5 * (1.0 + xi3[0]), y = xi3[1], z = xi3[2];
  const double L = LWH[0], W = LWH[1], H = LWH[2];
  const double s2 = s * s, s3 = s2 * s;
  // values and d/ds of the Hermite cubics
  const double h[4] = {1.0 - 3.0 * s2 + 2.0 * s3, s - 2.0 * s2 + s3, 3.0 * s2 - 2.0 * s3, s3 - s2};
  const double dh[4] = {6.0 * s2 - 6.0 * s, 1.0 - 4.0 * s + 3.0 * s2, 6.0 * s - 6.0 * s2, 3.0 * s2 - 2.0 * s};
  const double lin[2] = {1.0 - s, s}, dlin[2] = {-1.0, 1.0};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double hr = h[2 * k], hx = L * h[2 * k + 1];
    if (S) {
      S[4 * k + 0] = hr;
      S[4 * k + 1] = hx;
      S[4 * k + 2] = 0.5 * W * y * lin[k];
      S[4 * k + 3] = 0.5 * H * z * lin[k];
    }
    // d/dxi = 0.5 d/ds
    dS[4 * k + 0][0] = 0.5 * dh[2 * k];
    dS[4 * k + 0][1] = 0.0;
    dS[4 * k + 0][2] = 0.0;
    dS[4 * k + 1][0] = 0.5 * L * dh[2 * k + 1];
    dS[4 * k + 1][1] = 0.0;
    dS[4 * k + 1][2] = 0.0;
    dS[4 * k + 2][0] = 0.25 * W * y * dlin[k];
    dS[4 * k + 2][1] = 0.5 * W * lin[k];
    dS[4 * k + 2][2] = 0.0;
    dS[4 * k + 3][0] = 0.25 * H * z * dlin[k];
    dS[4 * k + 3][1] = 0.0;
    dS[4 * k + 3][2] = 0.5 * H * lin[k];
  }
}

// Device/host: T10 values and parent-domain gradients.
__host__ __device__ inline void t10_shape(const double* xi, double* N, double (*dN)[3]) {
  const double z[4] = {1.0 - xi[0] - xi[1] - xi[2], xi[0], xi[1], xi[2]};
  // d z_i / d xi_k
  const double G[4][3] = {{-1.0, -1.0, -1.0}, {1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  const int ea[6] = {0, 1, 2, 0, 1, 2}, eb[6] = {1, 2, 0, 3, 3, 3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (N) N[i] = z[i] * (2.0 * z[i] - 1.0);
#pragma unroll
    for (int k = 0; k < 3; ++k) dN[i][k] = (4.0 * z[i] - 1.0) * G[i][k];
  }
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    const int a = ea[m], b = eb[m];
    if (N) N[4 + m] = 4.0 * z[a] * z[b];
#pragma unroll
    for (int k = 0; k < 3; ++k) dN[4 + m][k] = 4.0 * (z[a] * G[b][k] + z[b] * G[a][k]);
  }
}

// Device/host: ANCF3443 values and parent gradients; LWH = element (L, W, H).
__host__ __device__ inline void ancf_shape(const double* xi3, const double* LWH, double* S,
                                           double (*dS)[3]) {
  const double x = xi3[0], y = xi3[1], z = xi3[2];
  const double sx[4] = {-1.0, 1.0, 1.0, -1.0}, sy[4] = {-1.0, -1.0, 1.0, 1.0};
  const double L = LWH[0], W = LWH[1], H = LWH[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double px = 1.0 + sx[k] * x, py = 1.0 + sy[k] * y;
    const double bub = 2.0 + sx[k] * x + sy[k] * y - x * x - y * y;
    const double ux = x * x - 1.0, uy = y * y - 1.0;
    double* d0 = dS[4 * k + 0];
    double* d1 = dS[4 * k + 1];
    double* d2 = dS[4 * k + 2];
    double* d3 = dS[4 * k + 3];
    if (S) {
      S[4 * k + 0] = 0.125 * px * py * bub;
      S[4 * k + 1] = 0.0625 * L * sx[k] * ux * px * py;
      S[4 * k + 2] = 0.0625 * W * sy[k] * uy * px * py;
      S[4 * k + 3] = 0.125 * H * z * px * py;
    }
    d0[0] = 0.125 * py * (sx[k] * bub + px * (sx[k] - 2.0 * x));
    d0[1] = 0.125 * px * (sy[k] * bub + py * (sy[k] - 2.0 * y));
    d0[2] = 0.0;
    d1[0] = 0.0625 * L * sx[k] * py * (2.0 * x * px + ux * sx[k]);
    d1[1] = 0.0625 * L * sx[k] * ux * px * sy[k];
    d1[2] = 0.0;
    d2[0] = 0.0625 * W * sy[k] * uy * py * sx[k];
    d2[1] = 0.0625 * W * sy[k] * px * (2.0 * y * py + uy * sy[k]);
    d2[2] = 0.0;
    d3[0] = 0.125 * H * z * sx[k] * py;
    d3[1] = 0.125 * H * z * px * sy[k];
    d3[2] = 0.125 * H * px * py;
  }
}

}  // namespace tlfea
