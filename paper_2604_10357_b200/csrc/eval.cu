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
#include "material.cuh"

namespace tlfea {

static inline unsigned grid_for(int64_t n, int block) {
  return (unsigned)std::max<int64_t>(1, (n + block - 1) / block);
}

template <int ELEM>
struct Geo;
template <>
struct Geo<0> {  // T10
  static constexpr int NEN = 10, GROUP = 10, EPW = 3, NUB = 55;
};
template <>
struct Geo<1> {  // ANCF3443
  static constexpr int NEN = 16, GROUP = 32, EPW = 1, NUB = 136;
};

__host__ __device__ __forceinline__ int ublk(int n, int a, int b) {  // a <= b
  return a * n - (a * (a - 1)) / 2 + (b - a);
}

constexpr int kWarps = 4;  // warps per CTA of the element kernel

template <int ELEM>
__device__ __forceinline__ int max_blocks() {
  return ELEM == 0 ? 6 : 5;
}

// Blocks owned by a lane: index j -> partner b (returns -1 when none).
template <int ELEM>
__device__ __forceinline__ int partner(int a, int half, int j) {
  if (ELEM == 0) {
    if (j < 5) return (a + j) % 10;
    return a < 5 ? a + 5 : -1;
  } else {
    if (half == 0) return j < 4 ? (a + j) & 15 : -1;
    if (j < 4) return (a + 4 + j) & 15;
    return a < 8 ? a + 8 : -1;
  }
}

template <int ELEM, int NQ, int MODEL, bool KV, bool TAN>
__global__ void __launch_bounds__(kWarps * 32)
    k_element(int64_t n_el, const int32_t* __restrict__ conn, const double* __restrict__ gradN,
              const double* __restrict__ J0w, const double* __restrict__ x, const double* __restrict__ v,
              MatDev mat, double* __restrict__ fscr, double* __restrict__ Kscr,
              unsigned long long* __restrict__ err) {
  using G = Geo<ELEM>;
  constexpr int NEN = G::NEN, GROUP = G::GROUP, EPW = G::EPW, NUB = G::NUB;
  constexpr int NB = ELEM == 0 ? 6 : 5;
  constexpr int ND = MODEL == 0 ? 6 : 21;  // per-node shared data for the blocks
  __shared__ double s_part[kWarps][32][KV ? 18 : 9];
  __shared__ double s_F[kWarps][EPW][KV ? 18 : 9];
  __shared__ double s_node[kWarps][32][TAN ? ND : 1];
  __shared__ double s_C[kWarps][EPW][MODEL == 1 && TAN ? 36 : 1];

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = ELEM == 0 ? (lane < EPW * GROUP) : true;
  const int g = (ELEM == 0 && lane_active) ? lane / GROUP : 0;  // element slot in the warp
  const int a = ELEM == 0 ? (lane_active ? lane % GROUP : 0) : (lane & 15);
  const int half = ELEM == 0 ? 0 : (lane >> 4);
  const int64_t e = ((int64_t)blockIdx.x * kWarps + wib) * EPW + (lane_active ? g : 0);
  const bool valid = lane_active && e < n_el;
  const int gbase = g * GROUP;  // first lane of this element's group

  // gather nodal coordinates (and velocities) once
  double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
  if (valid) {
    const int64_t I = conn[e * NEN + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) xa[i] = x[3 * I + i];
    if (KV) {
#pragma unroll
      for (int i = 0; i < 3; ++i) va[i] = v[3 * I + i];
    }
  }
  double fa[3] = {0, 0, 0};
  double K[TAN ? NB : 1][9];
#pragma unroll
  for (int j = 0; j < (TAN ? NB : 1); ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) K[j][r] = 0.0;

  for (int q = 0; q < NQ; ++q) {
    double gN[3] = {0, 0, 0}, w = 0.0;
    if (valid) {
      const double* src = gradN + ((e * NQ + q) * NEN + a) * 3;
      gN[0] = src[0];
      gN[1] = src[1];
      gN[2] = src[2];
      w = J0w[e * NQ + q];
    }
    // ---- F (and Fdot) reduction over the element's nodes
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int J = 0; J < 3; ++J) {
        s_part[wib][lane][3 * i + J] = xa[i] * gN[J];
        if (KV) s_part[wib][lane][9 + 3 * i + J] = va[i] * gN[J];
      }
    __syncwarp();
    {
      // lanes 0..8 (ANCF also 16..24 for Fdot) of each group reduce one component
      const int comp = ELEM == 0 ? a : (lane & 15);
      const int which = ELEM == 0 ? 0 : half;  // ANCF: half 1 reduces Fdot
      if (lane_active && comp < 9 && (KV || which == 0)) {
        if (ELEM == 0) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < NEN; ++b) s += s_part[wib][gbase + b][comp];
          s_F[wib][g][comp] = s;
          if (KV) {
            double sd = 0.0;
#pragma unroll
            for (int b = 0; b < NEN; ++b) sd += s_part[wib][gbase + b][9 + comp];
            s_F[wib][g][9 + comp] = sd;
          }
        } else {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < NEN; ++b) s += s_part[wib][b][9 * which + comp];
          s_F[wib][0][9 * which + comp] = s;
        }
      }
    }
    __syncwarp();
    double F[9], Fd[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      F[r] = s_F[wib][g][r];
      if (KV) Fd[r] = s_F[wib][g][9 + r];
    }
    // ---- Stage 1: constitutive update (never leaves the SM)
    double S[6], St[6];
    MRState ms;
    if (MODEL == 0) {
      svk_S(F, mat.lam, mat.mu, S);
    } else {
      mr_state(F, ms);
      if (valid && !(ms.J > 0.0) && a == 0 && half == 0) atomicMin(err, (unsigned long long)(e * 64 + q));
      mr_S(ms, mat.C10, mat.C01, mat.kappa, S);
    }
#pragma unroll
    for (int r = 0; r < 6; ++r) St[r] = S[r];
    if (KV) {
      double Sv[6];
      kv_S(F, Fd, mat.eta, mat.lamd, Sv);
#pragma unroll
      for (int r = 0; r < 6; ++r) St[r] += Sv[r];
    }
    // ---- Stage 2 force: f_a += w F (S_tot grad N_a)
    {
      double t[3];
#pragma unroll
      for (int I = 0; I < 3; ++I) t[I] = sget(St, I, 0) * gN[0] + sget(St, I, 1) * gN[1] + sget(St, I, 2) * gN[2];
#pragma unroll
      for (int i = 0; i < 3; ++i) fa[i] += w * (F[3 * i] * t[0] + F[3 * i + 1] * t[1] + F[3 * i + 2] * t[2]);
    }
    if (TAN) {
      double te[3];  // elastic S grad N_a (geometric stiffness)
#pragma unroll
      for (int I = 0; I < 3; ++I) te[I] = sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2];
      if (MODEL == 0) {
        double ga[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) ga[i] = F[3 * i] * gN[0] + F[3 * i + 1] * gN[1] + F[3 * i + 2] * gN[2];
        double B[6];  // F F^T
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int i, k;
          voigt_pair(vv, i, k);
          B[vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
        }
        s_node[wib][lane][0] = ga[0];
        s_node[wib][lane][1] = ga[1];
        s_node[wib][lane][2] = ga[2];
        s_node[wib][lane][3] = gN[0];
        s_node[wib][lane][4] = gN[1];
        s_node[wib][lane][5] = gN[2];
        __syncwarp();
        const double lw = mat.lam * w, mw = mat.mu * w;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int b = partner<ELEM>(a, half, j);
          if (b < 0) continue;
          const double* nb = s_node[wib][gbase + b];
          const double gb0 = nb[0], gb1 = nb[1], gb2 = nb[2];
          const double s = w * (te[0] * nb[3] + te[1] * nb[4] + te[2] * nb[5]);
          const double d = mw * (gN[0] * nb[3] + gN[1] * nb[4] + gN[2] * nb[5]);
          const double gb[3] = {gb0, gb1, gb2};
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k)
              K[j][3 * i + k] += lw * ga[i] * gb[k] + mw * gb[i] * ga[k] + d * B[vidx(i, k)] + (i == k ? s : 0.0);
        }
      } else {
        // MR: material tangent columns (6 lanes per element), B_a, C B_a
        if (lane_active) {
          const int col = ELEM == 0 ? a : lane;
          if (col < 6 && (ELEM == 0 || half == 0)) {
            double cc[6];
            mr_Cv_column(ms, mat.C10, mat.C01, mat.kappa, col, cc);
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) s_C[wib][g][6 * vv + col] = cc[vv];
          }
        }
        double Ba[6][3];
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int I, J;
          voigt_pair(vv, I, J);
#pragma unroll
          for (int i = 0; i < 3; ++i)
            Ba[vv][i] = (I == J) ? F[3 * i + I] * gN[I] : F[3 * i + I] * gN[J] + F[3 * i + J] * gN[I];
        }
#pragma unroll
        for (int vv = 0; vv < 6; ++vv)
#pragma unroll
          for (int i = 0; i < 3; ++i) s_node[wib][lane][3 * vv + i] = Ba[vv][i];
        s_node[wib][lane][18] = gN[0];
        s_node[wib][lane][19] = gN[1];
        s_node[wib][lane][20] = gN[2];
        __syncwarp();
        double CB[6][3];
#pragma unroll
        for (int vv = 0; vv < 6; ++vv)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double s = 0.0;
#pragma unroll
            for (int ww = 0; ww < 6; ++ww) s += s_C[wib][g][6 * vv + ww] * Ba[ww][i];
            CB[vv][i] = w * s;
          }
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int b = partner<ELEM>(a, half, j);
          if (b < 0) continue;
          const double* nb = s_node[wib][gbase + b];
          const double s = w * (te[0] * nb[18] + te[1] * nb[19] + te[2] * nb[20]);
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              double acc = (i == k ? s : 0.0);
#pragma unroll
              for (int vv = 0; vv < 6; ++vv) acc += CB[vv][i] * nb[3 * vv + k];
              K[j][3 * i + k] += acc;
            }
        }
      }
    }
    __syncwarp();
  }

  if (!valid) return;
  if (ELEM == 0 || half == 0) {
    double* fo = fscr + (e * NEN + a) * 3;
    fo[0] = fa[0];
    fo[1] = fa[1];
    fo[2] = fa[2];
  }
  if (TAN) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = partner<ELEM>(a, half, j);
      if (b < 0) continue;
      if (a <= b) {
        double* o = Kscr + (e * NUB + ublk(NEN, a, b)) * 9;
#pragma unroll
        for (int r = 0; r < 9; ++r) o[r] = K[j][r];
      } else {  // store K_ba = K_ab^T
        double* o = Kscr + (e * NUB + ublk(NEN, b, a)) * 9;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) o[3 * k + i] = K[j][3 * i + k];
      }
    }
  }
}

// ------------------------------------------------------------------ gathers

__device__ __forceinline__ void sum_block(const uint32_t* __restrict__ ent, int32_t t0, int32_t t1, int nen,
                                          int nub, const double* __restrict__ Kscr, double acc[9]) {
#pragma unroll
  for (int r = 0; r < 9; ++r) acc[r] = 0.0;
  for (int32_t t = t0; t < t1; ++t) {
    const uint32_t en = ent[t];
    const int64_t e = en >> 8;
    const int a = (en >> 4) & 15, b = en & 15;
    if (a <= b) {
      const double* s = Kscr + (e * nub + ublk(nen, a, b)) * 9;
#pragma unroll
      for (int r = 0; r < 9; ++r) acc[r] += s[r];
    } else {
      const double* s = Kscr + (e * nub + ublk(nen, b, a)) * 9;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[3 * i + k] += s[3 * k + i];
    }
  }
}

// H = M/h (diagonal of each 3x3 block) + h K, one thread per
// coefficient block, every H value written once.
__global__ void k_gather_H(int64_t nnz_c, int nen, int nub, const int32_t* __restrict__ blk_row,
                           const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ blk_ptr,
                           const uint32_t* __restrict__ blk_ent, const double* __restrict__ Kscr,
                           const double* __restrict__ M, double h, double* __restrict__ H) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz_c) return;
  const int32_t i = blk_row[p], b0 = rowptr_c[i], deg = rowptr_c[i + 1] - b0, k = (int32_t)p - b0;
  double acc[9];
  sum_block(blk_ent, blk_ptr[p], blk_ptr[p + 1], nen, nub, Kscr, acc);
  const double mh = M[p] / h;
  double* out = H + 9 * (int64_t)b0 + 3 * k;
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int f = 0; f < 3; ++f) out[3 * d * deg + f] = h * acc[3 * d + f] + (d == f ? mh : 0.0);
}

// f_int and the residual g = (1/h) M (v - v_n) + f_int - f_ext - f_ff
// (Eq. residual / grad_L), one thread per owned node.
__global__ void k_gather_f(int64_t n_own, int nen, const int32_t* __restrict__ node_ptr,
                           const uint32_t* __restrict__ node_ent, const double* __restrict__ fscr,
                           const double* __restrict__ fpart_in, const int32_t* __restrict__ own_nodes,
                           const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ cols_c,
                           const double* __restrict__ M, const double* __restrict__ fff,
                           const double* __restrict__ v, const double* __restrict__ vn,
                           const double* __restrict__ fext, double h, int mode,
                           double* __restrict__ g, double* __restrict__ fint) {
  // mode 0: full (f from scratch + residual); 1: f only -> fint; 2: residual from fpart_in
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_own) return;
  double f0 = 0.0, f1 = 0.0, f2 = 0.0;
  if (mode == 2) {
    f0 = fpart_in[3 * i];
    f1 = fpart_in[3 * i + 1];
    f2 = fpart_in[3 * i + 2];
  } else {
    for (int32_t t = node_ptr[i]; t < node_ptr[i + 1]; ++t) {
      const uint32_t en = node_ent[t];
      const double* s = fscr + ((int64_t)(en >> 4) * nen + (en & 15)) * 3;
      f0 += s[0];
      f1 += s[1];
      f2 += s[2];
    }
  }
  if (fint) {
    fint[3 * i] = f0;
    fint[3 * i + 1] = f1;
    fint[3 * i + 2] = f2;
  }
  if (mode == 1 || !g) return;
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  for (int32_t p = rowptr_c[i]; p < rowptr_c[i + 1]; ++p) {
    const int64_t J = cols_c[p];
    const double mm = M[p];
    m0 += mm * (v[3 * J] - (vn ? vn[3 * J] : 0.0));
    m1 += mm * (v[3 * J + 1] - (vn ? vn[3 * J + 1] : 0.0));
    m2 += mm * (v[3 * J + 2] - (vn ? vn[3 * J + 2] : 0.0));
  }
  const int64_t I = own_nodes[i];
  const double r = 1.0 / h;
  g[3 * i] = m0 * r + f0 - (fext ? fext[3 * I] : 0.0) - fff[3 * i];
  g[3 * i + 1] = m1 * r + f1 - (fext ? fext[3 * I + 1] : 0.0) - fff[3 * i + 1];
  g[3 * i + 2] = m2 * r + f2 - (fext ? fext[3 * I + 2] : 0.0) - fff[3 * i + 2];
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
                                    double* __restrict__ fscr) {
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
  for (int i = 0; i < 3; ++i) fscr[t * 3 + i] = f[i];
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

template <int ELEM, int NQ, int MODEL, bool KV, bool TAN>
static tlfea_status launch_el(Context* c, const double* x, const double* v, cudaStream_t s) {
  using G = Geo<ELEM>;
  const int64_t per_cta = (int64_t)kWarps * G::EPW;
  const unsigned grid = (unsigned)((c->n_el + per_cta - 1) / per_cta);
  if (grid == 0) return TLFEA_OK;
  k_element<ELEM, NQ, MODEL, KV, TAN><<<grid, kWarps * 32, 0, s>>>(c->n_el, c->conn, c->gradN, c->J0w, x, v,
                                                                   c->mat, c->fscr, c->Kscr, c->err_flag);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

template <int ELEM, int NQ, int MODEL>
static tlfea_status launch_el_kv(Context* c, const double* x, const double* v, bool tan, cudaStream_t s) {
  const bool kv = c->mat.kv && v != nullptr;
  if (tan) return kv ? launch_el<ELEM, NQ, MODEL, true, true>(c, x, v, s) : launch_el<ELEM, NQ, MODEL, false, true>(c, x, v, s);
  return kv ? launch_el<ELEM, NQ, MODEL, true, false>(c, x, v, s) : launch_el<ELEM, NQ, MODEL, false, false>(c, x, v, s);
}

template <int ELEM, int NQ>
static tlfea_status launch_el_model(Context* c, const double* x, const double* v, bool tan, cudaStream_t s) {
  if (c->mat.model == TLFEA_SVK) return launch_el_kv<ELEM, NQ, 0>(c, x, v, tan, s);
  return launch_el_kv<ELEM, NQ, 1>(c, x, v, tan, s);
}

tlfea_status launch_element_kernel(Context* c, const double* x, const double* v, bool tangent,
                                   cudaStream_t s) {
  if (c->element == TLFEA_T10) {
    if (c->nq == 4) return launch_el_model<0, 4>(c, x, v, tangent, s);
    return launch_el_model<0, 5>(c, x, v, tangent, s);
  }
  return launch_el_model<1, 48>(c, x, v, tangent, s);
}

tlfea_status launch_gather_H(Context* c, double h, double* H, cudaStream_t s) {
  if (c->nnz_c == 0) return TLFEA_OK;
  k_gather_H<<<grid_for(c->nnz_c, 256), 256, 0, s>>>(c->nnz_c, c->nen, n_ublk_of(c->nen), c->blk_row, c->rowptr_c,
                                                     c->blk_ptr, c->blk_ent, c->Kscr, c->M, h, H);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_gather_f(Context* c, const double* v, const double* vn, const double* fext, double h,
                             double* g, double* fint, bool partial_only, cudaStream_t s) {
  if (c->n_own == 0) return TLFEA_OK;
  k_gather_f<<<grid_for(c->n_own, 256), 256, 0, s>>>(c->n_own, c->nen, c->node_ptr, c->node_ent, c->fscr, nullptr,
                                                     c->own_nodes, c->rowptr_c, c->cols_c, c->M, c->fff, v, vn,
                                                     fext, h, partial_only ? 1 : 0, g, fint);
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

tlfea_status launch_residual(Context* c, const double* fint, const double* v, const double* vn,
                             const double* fext, double h, double* g, cudaStream_t s) {
  if (c->n_own == 0) return TLFEA_OK;
  k_gather_f<<<grid_for(c->n_own, 256), 256, 0, s>>>(c->n_own, c->nen, c->node_ptr, c->node_ent, c->fscr, fint,
                                                     c->own_nodes, c->rowptr_c, c->cols_c, c->M, c->fff, v, vn,
                                                     fext, h, 2, g, nullptr);
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
  k_force_from_stress<<<grid_for(n, 128), 128, 0, s>>>(c->n_el, c->nq, c->nen, c->gradN, c->J0w, P, c->fscr);
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
