// fgather.cuh — the per-DOF force gather / residual of libtlfea (eval.cu).
//
//   f_int[3i+d] = sum of the node's element forces (ascending element order)
//   g[3i+d]     = (1/h) sum_J M_IJ (v - v_n)_{3J+d} + f_int - f_ext - f_ff
// (Eq. residual / grad_L; f_ff the body force of Eq. residual).
#pragma once
#include "common.cuh"

namespace tlfea {

#ifndef TLFEA_FG_UNROLL
#define TLFEA_FG_UNROLL 4
#endif
constexpr int kFgUnroll = TLFEA_FG_UNROLL;

struct FArgs {
  int64_t n_own;
  const int32_t* node_ptr;   // [n_own+1] node-sorted force scratch ranges
  const double* fscr;        // node-sorted element forces [..][3]
  const double* fpart_in;    // mode 2: f_int given
  const int32_t* own_nodes;
  const int32_t* rowptr_c;
  const int32_t* cols_c;
  const double* M;
  const double* fff;
  const double* v;
  const double* vn;
  const double* fext;
  double h;
  int mode;                  // 0 full (f + residual), 1 f only, 2 residual from fpart_in,
                             // 3 residual from a scratch that includes the element inertia
  double* g;
  double* fint;
};

// One owned DOF t = 3 i + d (the three threads of a node share its mass row via L1).
__device__ __forceinline__ void gather_f_dof_one(int64_t t, const FArgs& A) {
  const int64_t i = t / 3;
  const int d = (int)(t - 3 * i);
  double f = 0.0;
  if (A.mode == 2) {
    f = A.fpart_in[t];
  } else {
    const int32_t t0 = A.node_ptr[i], t1 = A.node_ptr[i + 1];
#pragma unroll kFgUnroll
    for (int32_t s = t0; s < t1; ++s) f += A.fscr[3 * (int64_t)s + d];
  }
  if (A.fint) A.fint[t] = f;
  if (A.mode == 1 || !A.g) return;
  if (A.mode == 3) {  // the scratch already holds f_a + (1/h) (m_e (v - v_n))_a per element
    const int64_t I = A.own_nodes[i];
    A.g[t] = f - (A.fext ? A.fext[3 * I + d] : 0.0) - A.fff[t];
    return;
  }
  double m = 0.0;
  const int32_t p0 = A.rowptr_c[i], p1 = A.rowptr_c[i + 1];
#pragma unroll kFgUnroll
  for (int32_t p = p0; p < p1; ++p) {
    const int64_t J = A.cols_c[p];
    m += A.M[p] * (A.v[3 * J + d] - (A.vn ? A.vn[3 * J + d] : 0.0));
  }
  const int64_t I = A.own_nodes[i];
  A.g[t] = m / A.h + f - (A.fext ? A.fext[3 * I + d] : 0.0) - A.fff[t];
}

}  // namespace tlfea
