// material.cuh — device constitutive laws of libtlfea (§4.3,
// P:398-405; forms fixed by DESIGN.md readings Q5-Q8).
//   SVK : S = lam tr(E) I + 2 mu E,  E = (C - I)/2, P = F S
//   MR  : S = 2C10 J^{-2/3}(I - I1/3 C^-1) + 2C01 J^{-4/3}(I1 I - C - 2I2/3 C^-1)
//             + kappa J (J-1) C^-1   (energy C10(I1b-3)+C01(I2b-3)+kappa/2 (J-1)^2)
//   KV  : S_v = 2 eta Edot + lam_d tr(Edot) I, Edot = (Fdot^T F + F^T Fdot)/2
// Symmetric tensors are stored as 6-vectors in Voigt order
//   0:(0,0) 1:(1,1) 2:(2,2) 3:(1,2) 4:(0,2) 5:(0,1).
// The material tangent dS/dE is a symmetric 6x6 matrix Cv[v][w] (engineering
// shear in the strain slot), so that the element tangent block is
//   K_ab = (grad N_a . S grad N_b) I + B_a^T Cv B_b          (Eq. tangent_block)
// with B_a[v][i] the Green-Lagrange strain operator of node a.
#pragma once
#include <cmath>

namespace tlfea {

__host__ __device__ __forceinline__ int vidx(int i, int j) {
  return i == j ? i : (3 - i - j) + 3;  // (1,2)->3, (0,2)->4, (0,1)->5
}
__host__ __device__ __forceinline__ void voigt_pair(int v, int& i, int& j) {
  // (0,0) (1,1) (2,2) (1,2) (0,2) (0,1) — arithmetic, so a runtime v stays in registers
  i = v < 3 ? v : (v == 3 ? 1 : 0);
  j = v < 3 ? v : (v == 5 ? 1 : 2);
}

// C = F^T F (Voigt)
__host__ __device__ __forceinline__ void right_cauchy_green(const double F[9], double C[6]) {
#pragma unroll
  for (int v = 0; v < 6; ++v) {
    int I, J;
    voigt_pair(v, I, J);
    C[v] = F[I] * F[J] + F[3 + I] * F[3 + J] + F[6 + I] * F[6 + J];
  }
}

__host__ __device__ __forceinline__ double det3(const double F[9]) {
  return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
         F[2] * (F[3] * F[7] - F[4] * F[6]);
}

// symmetric 3x3 (Voigt) inverse and determinant
__host__ __device__ __forceinline__ double sym_inv(const double C[6], double Ci[6]) {
  const double a = C[0], b = C[1], c = C[2], d = C[3], e = C[4], f = C[5];
  // [[a f e],[f b d],[e d c]]
  const double A00 = b * c - d * d, A11 = a * c - e * e, A22 = a * b - f * f;
  const double A12 = e * f - a * d, A02 = f * d - b * e, A01 = d * e - f * c;
  const double det = a * A00 + f * A01 + e * A02;
  const double r = 1.0 / det;
  Ci[0] = A00 * r; Ci[1] = A11 * r; Ci[2] = A22 * r;
  Ci[3] = A12 * r; Ci[4] = A02 * r; Ci[5] = A01 * r;
  return det;
}

// full symmetric 3x3 access of a Voigt vector
__host__ __device__ __forceinline__ double sget(const double A[6], int i, int j) {
  return A[vidx(i, j)];
}

// ---------------------------------------------------------------- SVK
__host__ __device__ __forceinline__ void svk_S(const double F[9], double lam, double mu,
                                               double S[6]) {
  double C[6];
  right_cauchy_green(F, C);
  const double trE = 0.5 * (C[0] + C[1] + C[2] - 3.0);
#pragma unroll
  for (int v = 0; v < 6; ++v) S[v] = mu * (C[v] - (v < 3 ? 1.0 : 0.0)) + (v < 3 ? lam * trE : 0.0);
}

__host__ __device__ __forceinline__ void svk_Cv(double lam, double mu, double Cv[36]) {
#pragma unroll
  for (int v = 0; v < 6; ++v)
#pragma unroll
    for (int w = 0; w < 6; ++w)
      Cv[6 * v + w] = (v < 3 && w < 3 ? lam : 0.0) + (v == w ? (v < 3 ? 2.0 * mu : mu) : 0.0);
}

// ---------------------------------------------------------------- Mooney-Rivlin
struct MRState {
  double C[6], Ci[6], J, I1, I2, J23, J43;
};

// 1/3 as a product: fp64 division is a long instruction sequence on the GPU
constexpr double kThird = 1.0 / 3.0;

__host__ __device__ __forceinline__ void mr_state(const double F[9], MRState& s) {
  right_cauchy_green(F, s.C);
  sym_inv(s.C, s.Ci);
  s.J = det3(F);
  s.I1 = s.C[0] + s.C[1] + s.C[2];
  const double CC = s.C[0] * s.C[0] + s.C[1] * s.C[1] + s.C[2] * s.C[2] +
                    2.0 * (s.C[3] * s.C[3] + s.C[4] * s.C[4] + s.C[5] * s.C[5]);
  s.I2 = 0.5 * (s.I1 * s.I1 - CC);
#ifdef __CUDA_ARCH__
  s.J23 = rcbrt(s.J * s.J);
#else
  s.J23 = 1.0 / cbrt(s.J * s.J);
#endif
  s.J43 = s.J23 * s.J23;
}

__host__ __device__ __forceinline__ void mr_S(const MRState& s, double C10, double C01,
                                              double kappa, double S[6]) {
  const double a = 2.0 * C10 * s.J23, b = 2.0 * C01 * s.J43;
  const double cinv = -(a * s.I1 + 2.0 * b * s.I2) * kThird + kappa * s.J * (s.J - 1.0);
#pragma unroll
  for (int v = 0; v < 6; ++v) {
    const double id = v < 3 ? 1.0 : 0.0;
    S[v] = a * id + b * (s.I1 * id - s.C[v]) + cinv * s.Ci[v];
  }
}

// Column w of the MR tangent: dS for the unit Voigt strain direction w
// (normal: dE_KK = 1; shear: dE_KL = dE_LK = 1/2), i.e. dC = 2 dE.
__host__ __device__ __forceinline__ void mr_Cv_column(const MRState& s, double C10, double C01,
                                                      double kappa, int w, double col[6]) {
  int K, L;
  voigt_pair(w, K, L);
  // dC (symmetric): normal -> 2 e_K e_K^T ; shear -> e_K e_L^T + e_L e_K^T
  const double CiCdC = (K == L) ? 2.0 * sget(s.Ci, K, K) : 2.0 * sget(s.Ci, K, L);  // Ci : dC
  const double CdC = (K == L) ? 2.0 * sget(s.C, K, K) : 2.0 * sget(s.C, K, L);      // C : dC
  const double dI1 = (K == L) ? 2.0 : 0.0;
  const double tau = 0.5 * CiCdC;                   // dJ = J tau
  const double dI2 = s.I1 * dI1 - CdC;
  const double a = 2.0 * C10 * s.J23, b = 2.0 * C01 * s.J43;
  const double da = -(2.0 / 3.0) * tau * a, db = -(4.0 / 3.0) * tau * b;
  const double cinv = -(a * s.I1 + 2.0 * b * s.I2) * kThird + kappa * s.J * (s.J - 1.0);
  const double dcinv = -(da * s.I1 + a * dI1 + 2.0 * (db * s.I2 + b * dI2)) * kThird +
                       kappa * (2.0 * s.J - 1.0) * s.J * tau;
#pragma unroll
  for (int v = 0; v < 6; ++v) {
    int i, j;
    voigt_pair(v, i, j);
    // dCi_ij = -(Ci dC Ci)_ij
    double dCi;
    if (K == L)
      dCi = -2.0 * sget(s.Ci, i, K) * sget(s.Ci, K, j);
    else
      dCi = -(sget(s.Ci, i, K) * sget(s.Ci, L, j) + sget(s.Ci, i, L) * sget(s.Ci, K, j));
    const double id = v < 3 ? 1.0 : 0.0;
    const double dC = (v == w) ? (K == L ? 2.0 : 1.0) : 0.0;
    col[v] = da * id + db * (s.I1 * id - s.C[v]) + b * (dI1 * id - dC) + dcinv * s.Ci[v] +
             cinv * dCi;
  }
}

// Column selection with a compile-time column so MRState stays in registers.
template <int W>
__host__ __device__ __forceinline__ void mr_Cv_col_t(const MRState& s, double C10, double C01, double kappa,
                                                     double col[6]) {
  mr_Cv_column(s, C10, C01, kappa, W, col);
}
__host__ __device__ __forceinline__ void mr_Cv_column_dispatch(const MRState& s, double C10, double C01,
                                                               double kappa, int w, double col[6]) {
  switch (w) {
    case 0: mr_Cv_col_t<0>(s, C10, C01, kappa, col); break;
    case 1: mr_Cv_col_t<1>(s, C10, C01, kappa, col); break;
    case 2: mr_Cv_col_t<2>(s, C10, C01, kappa, col); break;
    case 3: mr_Cv_col_t<3>(s, C10, C01, kappa, col); break;
    case 4: mr_Cv_col_t<4>(s, C10, C01, kappa, col); break;
    default: mr_Cv_col_t<5>(s, C10, C01, kappa, col); break;
  }
}

// ---------------------------------------------------------------- Kelvin-Voigt
__host__ __device__ __forceinline__ void kv_S(const double F[9], const double Fd[9], double eta,
                                              double lamd, double S[6]) {
  double Ed[6];
#pragma unroll
  for (int v = 0; v < 6; ++v) {
    int I, J;
    voigt_pair(v, I, J);
    Ed[v] = 0.5 * (Fd[I] * F[J] + Fd[3 + I] * F[3 + J] + Fd[6 + I] * F[6 + J] +
                   F[I] * Fd[J] + F[3 + I] * Fd[3 + J] + F[6 + I] * Fd[6 + J]);
  }
  const double tr = Ed[0] + Ed[1] + Ed[2];
#pragma unroll
  for (int v = 0; v < 6; ++v) S[v] = 2.0 * eta * Ed[v] + (v < 3 ? lamd * tr : 0.0);
}

// P = F S (full 3x3 row-major)
__host__ __device__ __forceinline__ void pk1_from_S(const double F[9], const double S[6],
                                                    double P[9]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int J = 0; J < 3; ++J)
      P[3 * i + J] = F[3 * i + 0] * sget(S, 0, J) + F[3 * i + 1] * sget(S, 1, J) +
                     F[3 * i + 2] * sget(S, 2, J);
}

}  // namespace tlfea
