// eval.cu — the evaluation kernels of libtlfea (B200 / sm_100a, fp64).
//
// Element kernel (Stage 1 + Stage 2 fused, §4.3-4.4.2):
//   one lane per element node a (T10: 10 lanes, 3 elements per warp; ANCF3443:
//   32 lanes = 2 per node, 1 element per warp). Per quadrature point the lanes
//   reduce F = sum_a x_a (x) grad N_a (Eq. F_assembly) through shared memory,
//   evaluate S / P (Stage 1, never written to HBM), accumulate
//   f_a = sum_q P grad N_a J0 w (Eq. fint_local) and the symmetric tangent
//   blocks K_ab (Eq. tangent_block) that each lane owns (a circulant split of
//   the n(n+1)/2 upper blocks: 5-6 blocks per T10 lane, 4-5 per ANCF lane).
//   SVK uses the structured form K_ab = s_ab I + lam g_a g_b^T + mu g_b g_a^T
//   + mu d_ab F F^T (g_a = F grad N_a, s_ab = grad N_a . S grad N_b,
//   d_ab = grad N_a . grad N_b); MR uses K_ab = s_ab I + B_a^T C B_b.
//   Outputs go to the element scratch (f_e, upper K blocks).
// Gather kernels (deterministic scatter, north-star (d)): one thread per CSR
//   coefficient block / owned node sums its contributions in ascending element
//   order through the precomputed inverse slot map, adds M/h and
//   writes every H value exactly once — no floating-point atomics.
#include "common.cuh"
#include "fgather.cuh"
#include "material.cuh"

namespace tlfea {

static inline unsigned grid_for(int64_t n, int block) {
  return (unsigned)std::max<int64_t>(1, (n + block - 1) / block);
}

// Node-sorted force scratch: one thread per (owned node, component) so the
// dependent index -> value loads of the mass row have 3x the parallelism;
// the three threads of a node share its row through L1.
// mode: 0 full (f + residual), 1 f only, 2 residual from fpart_in.
#ifndef TLFEA_FG_BLOCK
#define TLFEA_FG_BLOCK 128  // config 3: 1.189 ms (128) vs 1.208 (256), 1.237 (512), 1.198 (64)
#endif
constexpr int kFgBlock = TLFEA_FG_BLOCK;
__global__ void k_gather_f_dof(FArgs A) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < 3 * A.n_own) gather_f_dof_one(t, A);
}

static FArgs f_args(const Context* c, const double* fscr, const double* fpart_in, const double* v, const double* vn,
                    const double* fext, double h, int mode, double* g, double* fint) {
  FArgs A;
  A.n_own = c->n_own;
  A.node_ptr = c->node_ptr;
  A.fscr = fscr;
  A.fpart_in = fpart_in;
  A.own_nodes = c->own_nodes;
  A.rowptr_c = c->rowptr_c;
  A.cols_c = c->cols_c;
  A.M = c->M;
  A.fff = c->fff;
  A.v = v;
  A.vn = vn;
  A.fext = fext;
  A.h = h;
  A.mode = mode;
  A.g = g;
  A.fint = fint;
  return A;
}

// ------------------------------------------------ Stage 1 / Stage 2 alone

template <int MODEL>
__device__ __forceinline__ void stress_at(const double F[9], const double Fd[9], const MatDev& m,
                                          bool kv, double P[9], double* J) {
  double S[6];
  if (MODEL == 0) {
    svk_S(F, m.lam, m.mu, S);
    *J = 1.0;
  } else {
    MRState s;
    mr_state(F, s);
    mr_S(s, m.C10, m.C01, m.kappa, S);
    *J = s.J;
  }
  if (kv) {
    double Sv[6];
    kv_S(F, Fd, m.eta, m.lamd, Sv);
    for (int r = 0; r < 6; ++r) S[r] += Sv[r];
  }
  pk1_from_S(F, S, P);
}

template <int MODEL>
__global__ void k_stress(int64_t n_el, int nq, int nen, const int32_t* __restrict__ conn,
                         const double* __restrict__ gradN, const double* __restrict__ x,
                         const double* __restrict__ v, MatDev m, double* __restrict__ P,
                         unsigned long long* __restrict__ err) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_el * nq) return;
  const int64_t e = t / nq;
  double F[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, Fd[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double* gN = gradN + t * nen * 3;
  for (int a = 0; a < nen; ++a) {
    const int64_t I = conn[e * nen + a];
    for (int i = 0; i < 3; ++i) {
      const double xi = x[3 * I + i];
      const double vi = m.kv ? v[3 * I + i] : 0.0;
      for (int J = 0; J < 3; ++J) {
        F[3 * i + J] += xi * gN[3 * a + J];
        Fd[3 * i + J] += vi * gN[3 * a + J];
      }
    }
  }
  double J;
  stress_at<MODEL>(F, Fd, m, m.kv != 0, P + t * 9, &J);
  if (MODEL == 1 && !(J > 0.0)) atomicMin(err, (unsigned long long)(e * 64 + (t % nq)));
}

__global__ void k_force_from_stress(int64_t n_el, int nq, int nen, const double* __restrict__ gradN,
                                    const double* __restrict__ J0w, const double* __restrict__ P,
                                    const int32_t* __restrict__ fdest, double* __restrict__ fscr) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_el * nen) return;
  const int64_t e = t / nen;
  const int a = (int)(t % nen);
  double f[3] = {0, 0, 0};
  for (int q = 0; q < nq; ++q) {
    const double* Pq = P + (e * nq + q) * 9;
    const double* gN = gradN + ((e * nq + q) * nen + a) * 3;
    const double w = J0w[e * nq + q];
    for (int i = 0; i < 3; ++i) f[i] += w * (Pq[3 * i] * gN[0] + Pq[3 * i + 1] * gN[1] + Pq[3 * i + 2] * gN[2]);
  }
  const int64_t pos = fdest ? (int64_t)fdest[t] : t;
  for (int i = 0; i < 3; ++i) fscr[pos * 3 + i] = f[i];
}

// ------------------------------------------------------ constitutive hook

template <int MODEL>
__global__ void k_constitutive(int64_t n, MatDev m, const double* __restrict__ F,
                               const double* __restrict__ Fd, double* __restrict__ P,
                               double* __restrict__ A) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  double f[9], fd[9];
  for (int r = 0; r < 9; ++r) {
    f[r] = F[9 * t + r];
    fd[r] = Fd ? Fd[9 * t + r] : 0.0;
  }
  double J;
  stress_at<MODEL>(f, fd, m, m.kv != 0 && Fd != nullptr, P + 9 * t, &J);
  if (!A) return;
  double S[6], Cv[36];
  if (MODEL == 0) {
    svk_S(f, m.lam, m.mu, S);
    svk_Cv(m.lam, m.mu, Cv);
  } else {
    MRState s;
    mr_state(f, s);
    mr_S(s, m.C10, m.C01, m.kappa, S);
    for (int w = 0; w < 6; ++w) {
      double col[6];
      mr_Cv_column(s, m.C10, m.C01, m.kappa, w, col);
      for (int vv = 0; vv < 6; ++vv) Cv[6 * vv + w] = col[vv];
    }
  }
  // A_iJkL = delta_ik S_JL + F_iI C_IJKL F_kK
  for (int i = 0; i < 3; ++i)
    for (int Jx = 0; Jx < 3; ++Jx)
      for (int k = 0; k < 3; ++k)
        for (int L = 0; L < 3; ++L) {
          double s = (i == k) ? sget(S, Jx, L) : 0.0;
          for (int I = 0; I < 3; ++I)
            for (int Kx = 0; Kx < 3; ++Kx) s += f[3 * i + I] * Cv[6 * vidx(I, Jx) + vidx(Kx, L)] * f[3 * k + Kx];
          A[81 * t + (3 * i + Jx) * 9 + 3 * k + L] = s;
        }
}

// ------------------------------------------------------------- launchers

// The AdamW gradient from a force scratch that already holds the element
// inertia (k_force_t10_aff<.., INR>): g = sum - f_ext - f_ff, no f_int.
tlfea_status launch_gradient_inertia(Context* c, const double* fext, double* g, cudaStream_t s) {
  if (c->n_own == 0) return TLFEA_OK;
  k_gather_f_dof<<<grid_for(3 * c->n_own, kFgBlock), kFgBlock, 0, s>>>(
      f_args(c, c->fscr, nullptr, nullptr, nullptr, fext, 1.0, 3, g, nullptr));
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_gather_f(Context* c, const double* v, const double* vn, const double* fext, double h,
                             double* g, double* fint, bool partial_only, cudaStream_t s) {
  if (c->n_own == 0) return TLFEA_OK;
  k_gather_f_dof<<<grid_for(3 * c->n_own, kFgBlock), kFgBlock, 0, s>>>(
      f_args(c, c->fscr, nullptr, v, vn, fext, h, partial_only ? 1 : 0, g, fint));
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

// ------------------------------------- linear constraints (NEXT-3, Q22)
// c_k = C_k q - b_k, one thread per constraint (Alg. 2)
__global__ void k_con_residual(int64_t m, const int32_t* __restrict__ ptr, const int32_t* __restrict__ cols,
                               const double* __restrict__ vals, const double* __restrict__ b,
                               const double* __restrict__ q, double* __restrict__ c) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  double s = -b[k];
  for (int32_t p = ptr[k]; p < ptr[k + 1]; ++p) s += vals[p] * q[cols[p]];
  c[k] = s;
}

// g_i += h sum_k C_ki (lambda_k + rho c_k) over the C^T row of DOF i, in
// ascending k (one thread per DOF, no write conflicts)
__global__ void k_con_grad(int64_t n_dof, const int32_t* __restrict__ tptr, const int32_t* __restrict__ trows,
                           const double* __restrict__ tvals, const double* __restrict__ lam, double rho,
                           const double* __restrict__ c, double h, double* __restrict__ g) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_dof) return;
  const int32_t p0 = tptr[i], p1 = tptr[i + 1];
  if (p0 == p1) return;
  double gi = g[i];
  for (int32_t p = p0; p < p1; ++p) {
    const int32_t k = trows[p];
    gi += h * tvals[p] * ((lam ? lam[k] : 0.0) + rho * c[k]);
  }
  g[i] = gi;
}

// H[slot] += h^2 rho (C^T C)_ij, one thread per distinct pair (P:541-543 without atomics)
__global__ void k_con_hess(int64_t n, const int64_t* __restrict__ slot, const double* __restrict__ val,
                           double h2rho, double* __restrict__ H) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) H[slot[t]] += h2rho * val[t];
}

// lambda_k += rho c_k (Eq. lambda_update)
__global__ void k_con_dual(int64_t m, double rho, const double* __restrict__ c, double* __restrict__ lam) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) lam[k] += rho * c[k];
}

tlfea_status launch_constraint_residual(Context* c, const double* q, double* c_out, cudaStream_t st) {
  if (c->n_con == 0) return TLFEA_OK;
  k_con_residual<<<grid_for(c->n_con, 256), 256, 0, st>>>(c->n_con, c->con_ptr, c->con_cols, c->con_vals, c->con_b,
                                                          q, c_out);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_constraint_terms(Context* c, const double* q, const double* lam, double rho, double h,
                                     double* g, double* H, cudaStream_t st) {
  if (c->n_con == 0) return TLFEA_OK;
  TL_TRY_LAUNCH(launch_constraint_residual(c, q, c->con_c, st));
  if (g) {
    const int64_t n_dof = 3 * c->n_coef;
    k_con_grad<<<grid_for(n_dof, 256), 256, 0, st>>>(n_dof, c->conT_ptr, c->conT_rows, c->conT_vals, lam, rho,
                                                     c->con_c, h, g);
    TL_CHECK_LAUNCH();
  }
  if (H && c->n_gram > 0) {
    k_con_hess<<<grid_for(c->n_gram, 256), 256, 0, st>>>(c->n_gram, c->gram_ij, c->gram_val, h * h * rho, H);
    TL_CHECK_LAUNCH();
  }
  return TLFEA_OK;
}

tlfea_status launch_dual_update(Context* c, const double* q, double rho, double* lam, double* c_out,
                                cudaStream_t st) {
  if (c->n_con == 0) return TLFEA_OK;
  double* cbuf = c_out ? c_out : c->con_c;
  TL_TRY_LAUNCH(launch_constraint_residual(c, q, cbuf, st));
  k_con_dual<<<grid_for(c->n_con, 256), 256, 0, st>>>(c->n_con, rho, cbuf, lam);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

// ------------------------------------------------ AdamW (Alg. 2, NEXT-2)
// One thread per DOF: moments, bias correction, velocity update with
// decoupled weight decay, backward-Euler step map.
__global__ void k_adamw_update(int64_t n, double c1, double c2, double alpha, double b1, double b2, double eps,
                               double wd, const double* __restrict__ g, double* __restrict__ m,
                               double* __restrict__ s, double* __restrict__ v, const double* __restrict__ q_n,
                               double h, double* __restrict__ q, const double* __restrict__ vn,
                               double* __restrict__ dv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double gi = g[i];
  const double mi = b1 * m[i] + (1.0 - b1) * gi;
  const double si = b2 * s[i] + (1.0 - b2) * gi * gi;
  const double vi = (1.0 - alpha * wd) * v[i] - alpha * (mi / c1) / (sqrt(si / c2) + eps);
  m[i] = mi;
  s[i] = si;
  v[i] = vi;
  q[i] = q_n[i] + h * vi;
  if (dv) dv[i] = vi - vn[i];  // the element-level inertia input of the gradient
}

// ||a||^2 and ||b||^2 in a fixed reduction order: kNormBlocks blocks of
// grid-stride partials, then one block sums the partials (bitwise reproducible)
constexpr int kNormBlocks = 296, kNormThreads = 256;

__device__ __forceinline__ void block_sum2(double& x, double& y) {
  __shared__ double sx[kNormThreads], sy[kNormThreads];
  sx[threadIdx.x] = x;
  sy[threadIdx.x] = y;
  __syncthreads();
  for (int w = kNormThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sx[threadIdx.x] += sx[threadIdx.x + w];
      sy[threadIdx.x] += sy[threadIdx.x + w];
    }
    __syncthreads();
  }
  x = sx[0];
  y = sy[0];
}

__global__ void __launch_bounds__(kNormThreads) k_sumsq_partial(int64_t n, const double* __restrict__ a,
                                                                const double* __restrict__ b,
                                                                double* __restrict__ part) {
  double x = 0.0, y = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kNormThreads + threadIdx.x; i < n; i += (int64_t)kNormBlocks * kNormThreads) {
    x = fma(a[i], a[i], x);
    y = fma(b[i], b[i], y);
  }
  block_sum2(x, y);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
}

__global__ void __launch_bounds__(kNormThreads) k_sumsq_final(const double* __restrict__ part,
                                                              double* __restrict__ out) {
  double x = 0.0, y = 0.0;
  for (int i = threadIdx.x; i < kNormBlocks; i += kNormThreads) {
    x += part[2 * i];
    y += part[2 * i + 1];
  }
  block_sum2(x, y);
  if (threadIdx.x == 0) {
    out[0] = sqrt(x);
    out[1] = sqrt(y);
  }
}

tlfea_status launch_adamw_update(Context* c, int l, const tlfea_adamw_params& p, const double* g, double* m,
                                 double* s, double* v, const double* q_n, double h, double* q, cudaStream_t st,
                                 const double* vn, double* dv) {
  const int64_t n = 3 * c->n_coef;
  if (n == 0) return TLFEA_OK;
  const double c1 = 1.0 - std::pow(p.beta1, l), c2 = 1.0 - std::pow(p.beta2, l);
  k_adamw_update<<<grid_for(n, 256), 256, 0, st>>>(n, c1, c2, p.alpha, p.beta1, p.beta2, p.eps, p.weight_decay, g,
                                                     m, s, v, q_n, h, q, vn, dv);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_norms2(Context* c, const double* a, const double* b, double* out, cudaStream_t st) {
  const int64_t n = 3 * c->n_coef;
  if (!c->norm_part) {
    const tlfea_status st_alloc = c->alloc(&c->norm_part, (size_t)2 * kNormBlocks);
    if (st_alloc != TLFEA_OK) return st_alloc;
  }
  k_sumsq_partial<<<kNormBlocks, kNormThreads, 0, st>>>(n, a, b, c->norm_part);
  TL_CHECK_LAUNCH();
  k_sumsq_final<<<1, kNormThreads, 0, st>>>(c->norm_part, out);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_residual(Context* c, const double* fint, const double* v, const double* vn,
                             const double* fext, double h, double* g, cudaStream_t s) {
  if (c->n_own == 0) return TLFEA_OK;
  if (!g) return TLFEA_OK;  // nothing to write
  k_gather_f_dof<<<grid_for(3 * c->n_own, kFgBlock), kFgBlock, 0, s>>>(
      f_args(c, c->fscr, fint, v, vn, fext, h, 2, g, nullptr));
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_stress_only(Context* c, const double* x, const double* v, double* P, cudaStream_t s) {
  const int64_t n = c->n_el * c->nq;
  if (n == 0) return TLFEA_OK;
  MatDev m = c->mat;
  if (!v) m.kv = 0;
  if (m.model == TLFEA_SVK)
    k_stress<0><<<grid_for(n, 128), 128, 0, s>>>(c->n_el, c->nq, c->nen, c->conn, c->gradN, x, v, m, P, c->err_flag);
  else
    k_stress<1><<<grid_for(n, 128), 128, 0, s>>>(c->n_el, c->nq, c->nen, c->conn, c->gradN, x, v, m, P, c->err_flag);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_force_from_stress(Context* c, const double* P, cudaStream_t s) {
  const int64_t n = c->n_el * c->nen;
  if (n == 0) return TLFEA_OK;
  k_force_from_stress<<<grid_for(n, 128), 128, 0, s>>>(c->n_el, c->nq, c->nen, c->gradN, c->J0w, P, c->fdest, c->fscr);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_test_constitutive(const MatDev& m, int64_t n, const double* F, const double* Fd, double* P,
                                      double* A) {
  if (n <= 0) return TLFEA_OK;
  if (m.model == TLFEA_SVK)
    k_constitutive<0><<<grid_for(n, 128), 128>>>(n, m, F, Fd, P, A);
  else
    k_constitutive<1><<<grid_for(n, 128), 128>>>(n, m, F, Fd, P, A);
  TL_CHECK_LAUNCH();
  TL_CUDA(cudaDeviceSynchronize());
  return TLFEA_OK;
}

}  // namespace tlfea
