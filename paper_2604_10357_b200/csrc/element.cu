// element.cu — fused Stage 1 + Stage 2 element kernel and the deterministic
// symmetric H gather of libtlfea (B200 / sm_100a, fp64).
//
// k_element (§4.3 Stage 1/2, Eq. tangent_block):
//   one lane per element node a (T10: 10 lanes, 3 elements per warp; ANCF3443:
//   32 lanes = 2 per node, 1 element per warp). Per quadrature point the lanes
//   reduce F = sum_a x_a (x) grad N_a (Eq. F_assembly) through a conflict-light
//   shared-memory transpose, evaluate S and P in registers (Stage 1 never
//   touches HBM), accumulate f_a = sum_q P grad N_a J0 w (Eq. fint_local) and
//   the upper 3x3 tangent blocks K_ab (a <= b) each lane owns: a circulant
//   split of the n(n+1)/2 blocks (5-6 per T10 lane, 4-5 per ANCF lane).
//   SVK: K_ab = s_ab I + lam g_a g_b^T + mu g_b g_a^T + mu d_ab F F^T with
//   g_a = F grad N_a, s_ab = grad N_a . S grad N_b, d_ab = grad N_a . grad N_b
//   (three FMAs per entry); MR: K_ab = s_ab I + B_a^T C B_b (C the 6x6
//   material tangent, 6 lanes per element build its columns).
//   Reference data come either from per-(e,q) tables in HBM (the paper's
//   layout) or, for congruent elements, from per-class tables staged once per
//   CTA in shared memory (no per-q global loads).
// k_gather_units (north star (d), deterministic scatter): one thread per
//   symmetric pair of coefficient blocks {(I,J),(J,I)}: sums the contributing
//   element blocks in ascending element order through the inverse slot map,
//   writes h K + M/h to (I,J) and its transpose to (J,I); every H value is
//   written exactly once and every scratch block is read exactly once.
#include <cooperative_groups.h>

#include "common.cuh"
#include "fgather.cuh"
#include "material.cuh"

namespace tlfea {

static inline unsigned gridn(int64_t n, int block) {
  return (unsigned)std::max<int64_t>(1, (n + block - 1) / block);
}

template <int ELEM>
struct Geo;
template <>
struct Geo<0> {  // T10
  static constexpr int NEN = 10, GROUP = 10, EPW = 3, NUB = 55, NB = 6;
};
template <>
struct Geo<1> {  // ANCF3443
  static constexpr int NEN = 16, GROUP = 32, EPW = 1, NUB = 136, NB = 5;
};
template <>
struct Geo<2> {  // ANCF3243 beam: 8 lanes per element, 4 elements per warp
  static constexpr int NEN = 8, GROUP = 8, EPW = 4, NUB = 36, NB = 5;
};

__host__ __device__ __forceinline__ int ublk(int n, int a, int b) {  // a <= b
  return a * n - (a * (a - 1)) / 2 + (b - a);
}

constexpr int kWarps = kElWarps;  // warps per CTA

// Tangent scratch stores carry the streaming hint (st.global.cs): measured
// on config 3, 10.93 vs 11.21 ms for the element kernel; the same hint on the
// H writes of the gather changes nothing (8.06 vs 8.06 ms), so those stay plain.
// TLFEA_CHECK builds (the bounds-checked library of tests/ and tools/, in place
// of compute-sanitizer): every store into the tangent scratch, the force
// scratch and H, and every TMA window of the gather, is checked against the
// buffer the host registered for the launch (g_rng: [lo, hi) of Kscr, fscr,
// H); a miss prints the address and traps.
#ifndef TLFEA_CHECK
#define TLFEA_CHECK 0
#endif
__device__ const double* g_rng[6];
__device__ __forceinline__ void tl_chk(const double* p, int which, int line) {
  if (TLFEA_CHECK && (p < g_rng[2 * which] || p >= g_rng[2 * which + 1])) {
    printf("tlfea bounds check: buffer %d, line %d: %p outside [%p, %p)\n", which, line, (const void*)p,
           (const void*)g_rng[2 * which], (const void*)g_rng[2 * which + 1]);
    __trap();
  }
}
#define TL_FCHK(fo) tl_chk((fo) + 2, 1, __LINE__), tl_chk((fo), 1, __LINE__)
__device__ __forceinline__ void k_store(double* p, double v) {
  if (TLFEA_CHECK) tl_chk(p, 0, __LINE__);
  __stcs(p, v);
}
__device__ __forceinline__ void h_store(double* p, double v) {
  if (TLFEA_CHECK) tl_chk(p, 2, __LINE__);
  *p = v;
}
constexpr int kLD = 33;    // padded lane stride of the per-warp shared tables

// Blocks owned by a lane: index j -> partner b (-1 when none).
template <int ELEM>
__device__ __forceinline__ int partner(int a, int half, int j) {
  if (ELEM == 0) {
    if (j < 5) return (a + j) % 10;
    return a < 5 ? a + 5 : -1;
  } else if (ELEM == 2) {
    if (j < 4) return (a + j) & 7;
    return a < 4 ? a + 4 : -1;
  } else {
    if (half == 0) return j < 4 ? (a + j) & 15 : -1;
    if (j < 4) return (a + 4 + j) & 15;
    return a < 8 ? a + 8 : -1;
  }
}

// Block passes per lane. One pass keeps all of a lane's upper blocks live
// (T10: 6 x 9 fp64 = 108 registers) and caps occupancy at 3 CTAs with
// spills at the 168-register bound; two passes redo the per-q kinematics but
// halve the accumulators, so T10 SVK fits 4 CTAs (128 registers) without
// spills — measured faster (config 3: 11.2 vs 11.4-12.8 ms). Mooney-Rivlin
// and ANCF measured slower with two passes (their per-q work is larger).
#ifndef TLFEA_2PH_QUNROLL
#define TLFEA_2PH_QUNROLL 1  // phase-B quadrature loop (config 3, 2 passes / 3 CTAs: 1 -> 9.96 ms, 2 -> 10.02)
#endif
constexpr int kQUnroll = TLFEA_2PH_QUNROLL;
#ifndef TLFEA_2PH_AUNROLL
#define TLFEA_2PH_AUNROLL 10
#endif
constexpr int kAUnroll = TLFEA_2PH_AUNROLL;  // phase A node loops
#ifndef TLFEA_T10_SVK_NPASS
#define TLFEA_T10_SVK_NPASS 2
#endif
#ifndef TLFEA_T10_MINB
#define TLFEA_T10_MINB 3  // T10 SVK, one pass: 3 CTAs of 4 warps per SM (<= 168 registers)
#endif
#ifndef TLFEA_T10_MINB2P
#define TLFEA_T10_MINB2P 4  // T10 SVK, two passes: 4 CTAs (<= 128 registers)
#endif

template <int ELEM, int MODEL>
__host__ __device__ constexpr int el_npass() {
  return (ELEM == 0 && MODEL == 0) ? TLFEA_T10_SVK_NPASS : 1;
}

template <int ELEM, int MODEL, int NPASS>
__host__ __device__ constexpr int el_minb() {
  return (ELEM == 0 && MODEL == 0)   ? (NPASS == 1 ? TLFEA_T10_MINB : TLFEA_T10_MINB2P)
         : (ELEM == 2 && MODEL == 0) ? 3
                                     : (NPASS == 1 ? 2 : 3);
}

// Element arguments shared by k_element and the fused persistent kernel.
struct ElArgs {
  int64_t n_el;
  const int32_t* conn;
  const double* gradN;
  const double* J0w;
  const uint8_t* cls;
  const double* cls_tab;
  int n_cls;
  const double* aff;  // affine (min) layout: [n_el][13] = grad_X z_0..3, J0 (straight-sided T10)
  const double* jinv;  // curved T10: [n_el][NQ][10] = J^-1 (row-major), J0 w_q
  int64_t g0;         // first warp group of the launch (element range [EPW g0, n_el))
  const double* x;
  const double* v;
  MatDev mat;
  double* fscr;
  double* Kscr;
  const int32_t* dest;
  const int32_t* fdest;
  unsigned long long* err;
  double inv_h;  // consistent KV tangent only: 1/h of the evaluation (k_element_kvc)
  // element-level inertia (k_force_t10_aff<.., INR>, v = v - v_n): f_a += (1/h) sum_b m_ab (v - v_n)_b
  const double* cls_mass;
  int mass_closed;   // 1: exact consistent mass (mass_rule 0) of straight-sided T10 -> closed form
};

__device__ __forceinline__ void pf_cp4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void pf_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

#ifndef TLFEA_DEST_ASYNC
#define TLFEA_DEST_ASYNC 1  // k_element: gather-sorted destinations via cp.async at group start
#endif

// One warp group (EPW elements of warp group `grp`) of Stage 1 + Stage 2.
// DA: the group's gather-sorted destinations are copied to shared memory with
// cp.async when the group starts and consumed by the store phase, so the
// scattered index loads never stall the warp.
template <int ELEM, int NQ, int MODEL, bool KV, bool TAN, bool CLS, int NPASS, bool DA = false>
__device__ __forceinline__ void element_group(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab) {
  using G = Geo<ELEM>;
  constexpr int NEN = G::NEN, GROUP = G::GROUP, EPW = G::EPW, NUB = G::NUB, NB = G::NB;
  constexpr int NC = KV ? 18 : 9;            // reduced components (F, Fdot)
  constexpr int ND = MODEL == 0 ? 6 : 21;    // per-node data shared for the blocks
  constexpr int TABW = NEN * 3 + 1;          // class table row: gradN (3 NEN) + J0w
  __shared__ double s_part[kWarps][NC][kLD];
  __shared__ double s_F[kWarps][EPW][NC];
  __shared__ double s_node[kWarps][TAN ? ND : 1][kLD];
  __shared__ double s_C[kWarps][EPW][MODEL == 1 && TAN ? 36 : 1];
  const int64_t n_el = A.n_el;
  const int32_t* __restrict__ conn = A.conn;
  const double* __restrict__ gradN = A.gradN;
  const double* __restrict__ J0w = A.J0w;
  const uint8_t* __restrict__ cls = A.cls;
  const double* __restrict__ x = A.x;
  const double* __restrict__ v = A.v;
  const MatDev& mat = A.mat;
  double* __restrict__ fscr = A.fscr;
  double* __restrict__ Kscr = A.Kscr;
  const int32_t* __restrict__ dest = A.dest;
  const int32_t* __restrict__ fdest = A.fdest;
  unsigned long long* __restrict__ err = A.err;

  // MULTI: several elements per warp, one lane per element node (T10, beam);
  // otherwise one element per warp, two lanes per node (ANCF3443)
  constexpr bool MULTI = ELEM != 1;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = MULTI ? (lane < EPW * GROUP) : true;
  const int g = (MULTI && lane_active) ? lane / GROUP : 0;
  const int a = MULTI ? (lane_active ? lane % GROUP : 0) : (lane & 15);
  const int half = MULTI ? 0 : (lane >> 4);
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < n_el;
  const int gbase = g * GROUP;
  // (SVK only: the Mooney-Rivlin tables already fill the 48 KB of static shared memory)
  constexpr bool DAX = DA && TAN && MODEL == 0;
  __shared__ int32_t s_dst[kWarps][DAX ? EPW * NUB : 1];
  if (DAX && dest) {
    const int64_t e0 = grp * EPW, lim = (n_el - e0) * NUB;
    for (int t = lane; t < EPW * NUB; t += 32)
      if (t < lim) pf_cp4(&s_dst[wib][t], dest + e0 * NUB + t);
  }

  double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
  int ce = 0;
  if (valid) {
    const int64_t I = conn[e * NEN + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) xa[i] = x[3 * I + i];
    if (KV) {
#pragma unroll
      for (int i = 0; i < 3; ++i) va[i] = v[3 * I + i];
    }
    if (CLS) ce = cls[e];
  }
  double fa[3] = {0, 0, 0};
  // NPASS > 1 splits each lane's blocks over sequential passes that redo the
  // per-q kinematics: fewer live accumulators -> more resident warps.
  constexpr int NBP = (NB + NPASS - 1) / NPASS;
  double K[TAN ? NBP : 1][9];

#pragma unroll 1
  for (int pass = 0; pass < (TAN ? NPASS : 1); ++pass) {
#pragma unroll
  for (int j = 0; j < (TAN ? NBP : 1); ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) K[j][r] = 0.0;

#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    double gN[3] = {0, 0, 0}, w = 0.0;
    if (valid) {
      if (CLS) {
        const double* t = s_tab + (ce * NQ + q) * TABW;
        gN[0] = t[3 * a];
        gN[1] = t[3 * a + 1];
        gN[2] = t[3 * a + 2];
        w = t[3 * NEN];
      } else {
        const double* src = gradN + ((e * NQ + q) * NEN + a) * 3;
        gN[0] = src[0];
        gN[1] = src[1];
        gN[2] = src[2];
        w = J0w[e * NQ + q];
      }
    }
    // ---- F (and Fdot) = sum_a x_a (x) grad N_a, reduced over the element's lanes
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int J = 0; J < 3; ++J) {
        s_part[wib][3 * i + J][lane] = xa[i] * gN[J];
        if (KV) s_part[wib][9 + 3 * i + J][lane] = va[i] * gN[J];
      }
    __syncwarp();
    if (ELEM == 0) {
      if (lane_active && a < 9) {
        // pairwise tree over the 10 node partials (short dependency chain)
        const double* p = &s_part[wib][a][gbase];
        s_F[wib][g][a] = (((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]))) + (p[8] + p[9]);
        if (KV) {
          const double* pd = &s_part[wib][9 + a][gbase];
          s_F[wib][g][9 + a] =
              (((pd[0] + pd[1]) + (pd[2] + pd[3])) + ((pd[4] + pd[5]) + (pd[6] + pd[7]))) + (pd[8] + pd[9]);
        }
      }
    } else if (ELEM == 2) {
      // 8 lanes, 9 (18) components: lane a reduces components a, a + 8, ...
#pragma unroll
      for (int cc = 0; cc < (KV ? 3 : 2); ++cc) {
        const int comp = a + 8 * cc;
        if (comp < NC) {
          const double* p = &s_part[wib][comp][gbase];
          s_F[wib][g][comp] = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
        }
      }
    } else {
      const int comp = lane & 15;
      if (comp < 9 && (KV || half == 0)) {
        // pairwise tree over the 16 node partials (depth 4 instead of a 16-long chain)
        const double* p = &s_part[wib][9 * half + comp][0];
        double t8[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) t8[b] = p[2 * b] + p[2 * b + 1];
        s_F[wib][0][9 * half + comp] =
            ((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]));
      }
    }
    __syncwarp();
    double F[9], Fd[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      F[r] = s_F[wib][g][r];
      if (KV) Fd[r] = s_F[wib][g][9 + r];
    }
    // ---- Stage 1: constitutive update (registers only)
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
    // ---- Stage 2 force: f_a += F (w S_tot grad N_a)
    {
      double t[3];
#pragma unroll
      for (int I = 0; I < 3; ++I)
        t[I] = w * (sget(St, I, 0) * gN[0] + sget(St, I, 1) * gN[1] + sget(St, I, 2) * gN[2]);
      if (pass == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i) fa[i] = fma(F[3 * i], t[0], fma(F[3 * i + 1], t[1], fma(F[3 * i + 2], t[2], fa[i])));
      }
    }
    if (TAN) {
      double tw[3];  // w * S_el grad N_a (geometric stiffness)
#pragma unroll
      for (int I = 0; I < 3; ++I)
        tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
      if (MODEL == 0) {
        double ga[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) ga[i] = F[3 * i] * gN[0] + F[3 * i + 1] * gN[1] + F[3 * i + 2] * gN[2];
        double B[6];  // F F^T (Voigt)
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int i, k;
          voigt_pair(vv, i, k);
          B[vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
        }
        s_node[wib][0][lane] = ga[0];
        s_node[wib][1][lane] = ga[1];
        s_node[wib][2][lane] = ga[2];
        s_node[wib][3][lane] = gN[0];
        s_node[wib][4][lane] = gN[1];
        s_node[wib][5][lane] = gN[2];
        const double lw = mat.lam * w, mw = mat.mu * w;
        const double gl[3] = {lw * ga[0], lw * ga[1], lw * ga[2]};
        const double gm[3] = {mw * ga[0], mw * ga[1], mw * ga[2]};
        const double gNm[3] = {mw * gN[0], mw * gN[1], mw * gN[2]};
        __syncwarp();
#pragma unroll
        for (int jj = 0; jj < NBP; ++jj) {
          const int j = pass * NBP + jj;
          const int b = j < NB ? partner<ELEM>(a, half, j) : -1;
          if (b < 0) continue;
          double* Kj = K[jj];
          const int lb = gbase + b;
          const double gb[3] = {s_node[wib][0][lb], s_node[wib][1][lb], s_node[wib][2][lb]};
          const double nb[3] = {s_node[wib][3][lb], s_node[wib][4][lb], s_node[wib][5][lb]};
          const double s = fma(tw[0], nb[0], fma(tw[1], nb[1], tw[2] * nb[2]));
          const double d = fma(gNm[0], nb[0], fma(gNm[1], nb[1], gNm[2] * nb[2]));
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              double acc = fma(gl[i], gb[k], fma(gb[i], gm[k], fma(d, B[vidx(i, k)], Kj[3 * i + k])));
              Kj[3 * i + k] = (i == k) ? acc + s : acc;
            }
        }
      } else {
        // MR: material tangent columns (6 lanes per element), B_a, w C B_a
        if (lane_active && (MULTI || half == 0)) {
          const int col = MULTI ? a : lane;
          if (col < 6) {
            double cc[6];
            mr_Cv_column_dispatch(ms, mat.C10, mat.C01, mat.kappa, col, cc);
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) s_C[wib][g][6 * vv + col] = w * cc[vv];
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
          for (int i = 0; i < 3; ++i) s_node[wib][3 * vv + i][lane] = Ba[vv][i];
        s_node[wib][18][lane] = gN[0];
        s_node[wib][19][lane] = gN[1];
        s_node[wib][20][lane] = gN[2];
        __syncwarp();
        double CB[6][3];
#pragma unroll
        for (int vv = 0; vv < 6; ++vv)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double s = 0.0;
#pragma unroll
            for (int ww = 0; ww < 6; ++ww) s = fma(s_C[wib][g][6 * vv + ww], Ba[ww][i], s);
            CB[vv][i] = s;
          }
#pragma unroll
        for (int jj = 0; jj < NBP; ++jj) {
          const int j = pass * NBP + jj;
          const int b = j < NB ? partner<ELEM>(a, half, j) : -1;
          if (b < 0) continue;
          double* Kj = K[jj];
          const int lb = gbase + b;
          const double s = fma(tw[0], s_node[wib][18][lb], fma(tw[1], s_node[wib][19][lb], tw[2] * s_node[wib][20][lb]));
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double bb[6];
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) bb[vv] = s_node[wib][3 * vv + k][lb];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double acc = Kj[3 * i + k];
#pragma unroll
              for (int vv = 0; vv < 6; ++vv) acc = fma(CB[vv][i], bb[vv], acc);
              Kj[3 * i + k] = (i == k) ? acc + s : acc;
            }
          }
        }
      }
    }
    __syncwarp();
  }

  if (valid && pass == 0 && (MULTI || half == 0)) {
    const int64_t fp = fdest ? (int64_t)fdest[e * NEN + a] : e * NEN + a;
    double* fo = fscr + fp * 3;
    if (TLFEA_CHECK) TL_FCHK(fo);
    fo[0] = fa[0];
    fo[1] = fa[1];
    fo[2] = fa[2];
  }
  // Tangent blocks -> scratch. Each lane's blocks go to scattered 72-byte
  // slots; storing them lane-by-lane would issue one 8-byte sector request per
  // value (measured: half of the kernel time). Instead each round stages one
  // block per lane (already in the orientation its receiver needs) in shared
  // memory and the warp writes the round's blocks as consecutive doubles, so a
  // warp store covers 3-4 whole blocks.
  if (TAN) {
    __shared__ int32_t s_pos[kWarps][32];  // block position (< 2^31, checked at setup)
    // store mapping: lane = 9 bi + r writes entry r of block 3 it + bi
    constexpr int NLB = MULTI ? EPW * GROUP : 32;  // lanes holding blocks
    constexpr int NIT = (NLB + 2) / 3;
    const int bi = lane / 9, rr = lane - 9 * (lane / 9);
    if (DAX && dest) {
      pf_wait();
      __syncwarp();
    }
#pragma unroll
    for (int jj = 0; jj < NBP; ++jj) {
      const int j = pass * NBP + jj;
      const int b = (valid && j < NB) ? partner<ELEM>(a, half, j) : -1;
      int32_t pos = -1;
      if (b >= 0) {
        const double* Kj = K[jj];
        const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
        // element-major: store the upper block K_{min,max}; gather-sorted: the
        // orientation the receiving unit needs (dest low bit)
        bool tr = a > b;
        pos = (int32_t)(e * NUB + ub);
        if (dest) {
          const int32_t d = DAX ? s_dst[wib][g * NUB + ub] : dest[e * NUB + ub];
          pos = d >> 1;
          tr = tr != ((d & 1) != 0);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) s_part[wib][tr ? 3 * k + i : 3 * i + k][lane] = Kj[3 * i + k];
      }
      s_pos[wib][lane] = pos;
      __syncwarp();
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int blk = 3 * it + bi;
        if (lane < 27 && blk < NLB) {
          const int32_t p = s_pos[wib][blk];
          if (p >= 0) k_store(Kscr + (int64_t)p * 9 + rr, s_part[wib][rr][blk]);
        }
      }
      __syncwarp();
    }
  }
  }  // pass
}

// T10 + SVK (no Kelvin-Voigt) + geometry classes, two phases per warp group.
// The lane-per-node layout of element_group recomputes the per-q kinematics
// (F reduction, S, F F^T, g_a) on all 10 lanes of an element and again in
// every block pass: about half of its fp64 instructions. Here
//   phase A: lane (element, q), 15 of 32 lanes, computes F = sum_a x_a (x) grad N_a
//            (Eq. F_assembly), S (reading Q5), F F^T and g_b = F grad N_b for the
//            element's 10 nodes once, into shared memory;
//   phase B: lane (element, node a) accumulates its upper blocks
//            K_ab = s_ab I + lam g_a g_b^T + mu g_b g_a^T + mu d_ab F F^T
//            (Eq. tangent_block) and f_a = sum_q F (w S grad N_a)
//            (Eq. fint_local) from shared memory only; the second block pass
//            re-reads instead of recomputing.
// Per-lane inputs of a T10 warp group (node coordinates, class id), loaded
// before the CTA stages its class tables so the two dependent global loads
// (conn -> x) overlap the table copy instead of stalling the group start.
struct T10Pre {
  double xa[3];
  int ce;
  int32_t fd;  // force scratch position of (e, a)
};
// CLS: class mode (the class id is loaded); table mode never touches A.cls
// (a compile-time switch: a run-time null test here changed the scheduling of
// the store loop and cost 7 % of the element kernel).
template <bool CLS>
__device__ __forceinline__ void t10_preload(int64_t grp, const ElArgs& A, T10Pre& p) {
  const int lane = threadIdx.x & 31;
  const int g = lane / 10, a = lane % 10;
  const int64_t e = grp * 3 + g;
  p.xa[0] = p.xa[1] = p.xa[2] = 0.0;
  p.ce = 0;
  p.fd = 0;
  if (lane < 30 && e < A.n_el) {
    p.fd = A.fdest ? A.fdest[e * 10 + a] : (int32_t)(e * 10 + a);
    const int64_t I = A.conn[e * 10 + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) p.xa[i] = A.x[3 * I + i];
    if constexpr (CLS)
      if (a == 0) p.ce = A.cls[e];
  }
}

// Table mode (meshes without geometry classes): the warp's 3 elements' per-(e,q)
// tables (grad N, J0 w; the paper's layout) are staged into rows
// slot = 3 wib + g of the dynamic shared table, so the two-phase groups read
// them exactly like class tables (class id := slot).
template <int NQ>
__device__ __forceinline__ void t10_stage_tables(int64_t grp, const ElArgs& A, double* __restrict__ s_tab) {
  constexpr int NEN = 10, EPW = 3, TABW = 3 * NEN + 1, PER = NQ * 3 * NEN;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t e0 = grp * EPW;
  for (int t = lane; t < EPW * PER; t += 32) {
    const int g = t / PER, r = t - PER * g, q = r / (3 * NEN), c = r - 3 * NEN * q;
    const int64_t e = e0 + g;
    s_tab[((wib * EPW + g) * NQ + q) * TABW + c] = e < A.n_el ? A.gradN[e * PER + r] : 0.0;
  }
  if (lane < EPW * NQ) {
    const int g = lane / NQ, q = lane - NQ * g;
    const int64_t e = e0 + g;
    s_tab[((wib * EPW + g) * NQ + q) * TABW + 3 * NEN] = e < A.n_el ? A.J0w[e * NQ + q] : 0.0;
  }
  __syncwarp();
}

// The same staging issued as cp.async (8-byte copies, no wait here): the
// tables stream in while the lanes load their node coordinates; the group
// waits (cp.async.wait_all) right before phase A.
__device__ __forceinline__ void pf_cp8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
template <int NQ>
__device__ __forceinline__ void t10_stage_tables_async(int64_t grp, const ElArgs& A, double* __restrict__ s_tab) {
  constexpr int NEN = 10, EPW = 3, TABW = 3 * NEN + 1, PER = NQ * 3 * NEN;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t e0 = grp * EPW;
  const int nv = (int)min((int64_t)EPW, A.n_el - e0);  // valid elements of the group
  for (int t = lane; t < nv * PER; t += 32) {
    const int g = t / PER, r = t - PER * g, q = r / (3 * NEN), c = r - 3 * NEN * q;
    pf_cp8(&s_tab[((wib * EPW + g) * NQ + q) * TABW + c], A.gradN + (e0 + g) * PER + r);
  }
  if (lane < nv * NQ) {
    const int g = lane / NQ, q = lane - NQ * g;
    pf_cp8(&s_tab[((wib * EPW + g) * NQ + q) * TABW + 3 * NEN], A.J0w + (e0 + g) * NQ + q);
  }
}

// Min (affine) layout for straight-sided T10 without geometry classes
// (SURVEY §8(d) "min layout"; P:312-320 with J constant per element): 13 fp64
// per element, the barycentric gradients grad_X z_i (i = 0..3) and J0 = det J.
// The warp's 3 elements' tables are generated in shared memory, rows slot =
// 3 wib + g as in table mode:
//   corner i: grad N_i = (4 z_i - 1) grad z_i,
//   edge (a,b): grad N = 4 (z_a grad z_b + z_b grad z_a),  J0 w_q = J0 * w_q
// (the T10 basis of reading Q2 at the rule's barycentric points).
template <int NQ>
__device__ __forceinline__ void t10_rule_point(int q, double z[4], double& w) {
  if constexpr (NQ == 5) {  // Keast (reading Q1): centroid -2/15, then z_p = 1/2 at point p + 1
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] = q == 0 ? 0.25 : (i == q - 1 ? 0.5 : 1.0 / 6.0);
    w = q == 0 ? -2.0 / 15.0 : 3.0 / 40.0;
  } else {  // 4-point degree-2 rule: z_p = (5 + 3 sqrt 5)/20 at point p, (5 - sqrt 5)/20 elsewhere
    const double r5 = 2.2360679774997896964;
    const double alpha = 0.25 + 0.15 * r5, beta = 0.25 - 0.05 * r5;
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] = i == q ? alpha : beta;
    w = 1.0 / 24.0;
  }
}

// Load half: lane (element g, point q) of the warp's 3 x NQ fetches its
// element's 13 values (issued before the conn -> x loads so both overlap).
struct T10Aff {
  double gz[4][3];
  double J0;
};
template <int NQ>
__device__ __forceinline__ void t10_affine_load(int64_t grp, const ElArgs& A, T10Aff& f) {
  constexpr int EPW = 3;
  const int lane = threadIdx.x & 31;
  const int g = lane / NQ;
  const int64_t e = grp * EPW + g;
  const bool ok = lane < EPW * NQ && e < A.n_el;
  const double* a = A.aff + 13 * (ok ? e : 0);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) f.gz[i][k] = ok ? a[3 * i + k] : 0.0;
  f.J0 = ok ? a[12] : 0.0;
}
// Expand half: the lane's table row (grad N_a of the 10 nodes, J0 w_q).
template <int NQ, bool JW = false>  // JW: f.J0 already holds J0 w_q (jinv layout)
__device__ __forceinline__ void t10_affine_expand(const T10Aff& f, double* __restrict__ s_tab) {
  constexpr int NEN = 10, EPW = 3, TABW = 3 * NEN + 1;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (lane < EPW * NQ) {
    const int g = lane / NQ, q = lane - NQ * g;
    double z[4], w;
    t10_rule_point<NQ>(q, z, w);
    double* t = s_tab + ((wib * EPW + g) * NQ + q) * TABW;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 3; ++k) t[3 * i + k] = (4.0 * z[i] - 1.0) * f.gz[i][k];
    const int ea[6] = {0, 1, 2, 0, 1, 2}, eb[6] = {1, 2, 0, 3, 3, 3};
#pragma unroll
    for (int m = 0; m < 6; ++m)
#pragma unroll
      for (int k = 0; k < 3; ++k) t[3 * (4 + m) + k] = 4.0 * (z[ea[m]] * f.gz[eb[m]][k] + z[eb[m]] * f.gz[ea[m]][k]);
    t[3 * NEN] = JW ? f.J0 : f.J0 * w;
  }
  __syncwarp();
}
// Curved T10 ("jinv" layout, 10 fp64 per (e,q)): lane (element g, point q)
// loads J^-1 and J0 w_q of its point; grad_X z_{j+1} = row j of J^-1 and
// grad_X z_0 = -(their sum) at that point, so t10_affine_expand<NQ, true>
// rebuilds the same table row (grad N = d N / d xi J^-1).
template <int NQ>
__device__ __forceinline__ void t10_jinv_load(int64_t grp, const ElArgs& A, T10Aff& f) {
  constexpr int EPW = 3;
  const int lane = threadIdx.x & 31;
  const int g = lane / NQ, q = lane - NQ * (lane / NQ);
  const int64_t e = grp * EPW + g;
  const bool ok = lane < EPW * NQ && e < A.n_el;
  const double* p = A.jinv + 10 * ((ok ? e : 0) * NQ + (ok ? q : 0));
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) f.gz[1 + j][k] = ok ? p[3 * j + k] : 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) f.gz[0][k] = -(f.gz[1][k] + f.gz[2][k] + f.gz[3][k]);
  f.J0 = ok ? p[9] : 0.0;  // J0 w_q
}
template <int NQ>
__device__ __forceinline__ void t10_stage_jinv(int64_t grp, const ElArgs& A, double* __restrict__ s_tab) {
  T10Aff f;
  t10_jinv_load<NQ>(grp, A, f);
  t10_affine_expand<NQ, true>(f, s_tab);
}
template <int NQ>
__device__ __forceinline__ void t10_stage_affine(int64_t grp, const ElArgs& A, double* __restrict__ s_tab) {
  T10Aff f;
  t10_affine_load<NQ>(grp, A, f);
  t10_affine_expand<NQ>(f, s_tab);
}

#ifndef TLFEA_T10_2PH_NPASS
#define TLFEA_T10_2PH_NPASS 2  // config 3: 2 passes at 3 CTAs/SM (166 registers) 9.96 ms; 3 passes at 4 CTAs 10.72; 1 pass 12.97
#endif
#ifndef TLFEA_T10_2PH_MINB
#define TLFEA_T10_2PH_MINB 3
#endif
template <int NQ, bool KV = false, bool TA = false>
__device__ __forceinline__ void element_group_t10svk(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab,
                                                     const T10Pre& pre) {
  constexpr int NEN = 10, GROUP = 10, EPW = 3, NUB = 55, NB = 6, TABW = 3 * NEN + 1;
  constexpr int NPASS = TLFEA_T10_2PH_NPASS;
  constexpr int NBP = (NB + NPASS - 1) / NPASS;
  constexpr int KQ = KV ? 27 : 21;  // per (element, q): F (9), S (6), F F^T (6) [, S + S_v (6)]
  __shared__ double s_ga[kWarps][NQ][3][kLD];
  __shared__ double s_k[kWarps][EPW][NQ][KQ];
  __shared__ double s_x[kWarps][EPW][3 * NEN];
  __shared__ double s_v[kWarps][KV ? EPW : 1][KV ? 3 * NEN : 1];
  __shared__ double s_part[kWarps][9][kLD];
  __shared__ int32_t s_dst[kWarps][EPW * NUB];
  __shared__ int32_t s_pos[kWarps][32];
  __shared__ int32_t s_cls[kWarps][EPW];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const int32_t* __restrict__ dest = A.dest;
  double* __restrict__ Kscr = A.Kscr;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = lane < EPW * GROUP;
  const int g = lane_active ? lane / GROUP : 0;
  const int a = lane_active ? lane % GROUP : 0;
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < n_el;
  const int gbase = g * GROUP;
  const bool write = dest;
  if (write) {
    const int64_t e0 = grp * EPW, lim = (n_el - e0) * NUB;
    for (int t = lane; t < EPW * NUB; t += 32)
      if (t < lim) pf_cp4(&s_dst[wib][t], dest + e0 * NUB + t);
  }
  if (lane_active) {
#pragma unroll
    for (int i = 0; i < 3; ++i) s_x[wib][g][3 * a + i] = pre.xa[i];
    if (a == 0) s_cls[wib][g] = pre.ce;
    if constexpr (KV) {
      double va[3] = {0, 0, 0};
      if (valid) {
        const int64_t I = A.conn[e * NEN + a];
#pragma unroll
        for (int i = 0; i < 3; ++i) va[i] = A.v[3 * I + i];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) s_v[wib][g][3 * a + i] = va[i];
    }
  }
  __syncwarp();
  if constexpr (TA) {  // table mode: the staged per-element tables have landed
    pf_wait();
    __syncwarp();
  }
  // ---- phase A: two lanes per (element, q), each owning 5 of the 10 nodes
  // (EPW * NQ * 2 = 30 lanes for Keast-5): partial F over its nodes, the halves
  // exchanged by one shuffle; lane h = 0 then stores F and S, lane h = 1 F F^T,
  // and each lane writes g_b = F grad N_b for its own nodes.
  static_assert(EPW * NQ * 2 <= 32, "phase A: two lanes per (element, q)");
  {
    const bool act = lane < EPW * NQ * 2;
    const int pr = act ? lane >> 1 : 0, hf = lane & 1;
    const int ge = pr / NQ, q = pr - NQ * (pr / NQ);
    const double* t = s_tab + (s_cls[wib][ge] * NQ + q) * TABW;
    const double* xs = s_x[wib][ge];
    double F[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
    for (int bb = 0; bb < NEN / 2; ++bb) {
      const int b = hf * (NEN / 2) + bb;
      const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xi = xs[3 * b + i];
        F[3 * i] = fma(xi, n0, F[3 * i]);
        F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
        F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
      }
    }
    // F = (nodes 0-4) + (nodes 5-9), the same order on both lanes
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const double o = __shfl_xor_sync(0xffffffffu, F[r], 1);
      F[r] = hf ? o + F[r] : F[r] + o;
    }
    double Fd[9];  // Kelvin-Voigt: Fdot = sum_a v_a (x) grad N_a (reading Q9)
    if constexpr (KV) {
#pragma unroll
      for (int r = 0; r < 9; ++r) Fd[r] = 0.0;
#pragma unroll
      for (int bb = 0; bb < NEN / 2; ++bb) {
        const int b = hf * (NEN / 2) + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double vi = s_v[wib][ge][3 * b + i];
          Fd[3 * i] = fma(vi, n0, Fd[3 * i]);
          Fd[3 * i + 1] = fma(vi, n1, Fd[3 * i + 1]);
          Fd[3 * i + 2] = fma(vi, n2, Fd[3 * i + 2]);
        }
      }
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const double o = __shfl_xor_sync(0xffffffffu, Fd[r], 1);
        Fd[r] = hf ? o + Fd[r] : Fd[r] + o;
      }
    }
    if (act) {
      double* kq = s_k[wib][ge][q];
      if (hf == 0) {
        double S[6];
        svk_S(F, mat.lam, mat.mu, S);
#pragma unroll
        for (int r = 0; r < 9; ++r) kq[r] = F[r];
#pragma unroll
        for (int r = 0; r < 6; ++r) kq[9 + r] = S[r];
        if constexpr (KV) {  // the force takes S + S_v; the tangent the elastic part only (reading Q8)
          double Sv[6];
          kv_S(F, Fd, mat.eta, mat.lamd, Sv);
#pragma unroll
          for (int r = 0; r < 6; ++r) kq[21 + r] = S[r] + Sv[r];
        }
      } else {
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int i, k;
          voigt_pair(vv, i, k);
          kq[15 + vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
        }
      }
#pragma unroll
      for (int bb = 0; bb < NEN / 2; ++bb) {
        const int b = hf * (NEN / 2) + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          s_ga[wib][q][i][ge * GROUP + b] = F[3 * i] * n0 + F[3 * i + 1] * n1 + F[3 * i + 2] * n2;
      }
    }
  }
  __syncwarp();
  // ---- phase B: one lane per (element, node a)
  const int ce = s_cls[wib][g];
  double fa[3] = {0, 0, 0};
  double K[NBP][9];
#pragma unroll 1
  for (int pass = 0; pass < NPASS; ++pass) {
#pragma unroll
    for (int j = 0; j < NBP; ++j)
#pragma unroll
      for (int r = 0; r < 9; ++r) K[j][r] = 0.0;
#pragma unroll kQUnroll
    for (int q = 0; q < NQ; ++q) {
      const double* t = s_tab + (ce * NQ + q) * TABW;
      const double* kq = s_k[wib][g][q];
      const double gN[3] = {t[3 * a], t[3 * a + 1], t[3 * a + 2]};
      const double w = t[3 * NEN];
      double S[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) S[r] = kq[9 + r];
      double tw[3];  // w S grad N_a
#pragma unroll
      for (int I = 0; I < 3; ++I) tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
      if (pass == 0) {
        if constexpr (KV) {
          double tt[3];  // w (S + S_v) grad N_a
#pragma unroll
          for (int I = 0; I < 3; ++I)
            tt[I] = w * (kq[21 + vidx(I, 0)] * gN[0] + kq[21 + vidx(I, 1)] * gN[1] + kq[21 + vidx(I, 2)] * gN[2]);
#pragma unroll
          for (int i = 0; i < 3; ++i)
            fa[i] = fma(kq[3 * i], tt[0], fma(kq[3 * i + 1], tt[1], fma(kq[3 * i + 2], tt[2], fa[i])));
        } else {
#pragma unroll
          for (int i = 0; i < 3; ++i)
            fa[i] = fma(kq[3 * i], tw[0], fma(kq[3 * i + 1], tw[1], fma(kq[3 * i + 2], tw[2], fa[i])));
        }
      }
      const double lw = mat.lam * w, mw = mat.mu * w;
      double gl[3], gm[3], gNm[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double gai = s_ga[wib][q][i][lane];
        gl[i] = lw * gai;
        gm[i] = mw * gai;
        gNm[i] = mw * gN[i];
      }
      double B[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) B[r] = kq[15 + r];
#pragma unroll
      for (int jj = 0; jj < NBP; ++jj) {
        const int j = pass * NBP + jj;
        const int b = j < NB ? partner<0>(a, 0, j) : -1;
        if (b < 0) continue;
        double* Kj = K[jj];
        const int lb = gbase + b;
        const double gb[3] = {s_ga[wib][q][0][lb], s_ga[wib][q][1][lb], s_ga[wib][q][2][lb]};
        const double nb[3] = {t[3 * b], t[3 * b + 1], t[3 * b + 2]};
        const double s = fma(tw[0], nb[0], fma(tw[1], nb[1], tw[2] * nb[2]));
        const double d = fma(gNm[0], nb[0], fma(gNm[1], nb[1], gNm[2] * nb[2]));
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double acc = fma(gl[i], gb[k], fma(gb[i], gm[k], fma(d, B[vidx(i, k)], Kj[3 * i + k])));
            Kj[3 * i + k] = (i == k) ? acc + s : acc;
          }
      }
    }
    if (valid && pass == 0) {
      double* fo = A.fscr + (int64_t)pre.fd * 3;
      if (TLFEA_CHECK) TL_FCHK(fo);
      fo[0] = fa[0];
      fo[1] = fa[1];
      fo[2] = fa[2];
    }
    {
      // warp-staged block stores, as in element_group
      constexpr int NLB = EPW * GROUP, NIT = (NLB + 2) / 3;
      const int bi = lane / 9, rr = lane - 9 * (lane / 9);
      if (write && pass == 0) {
        pf_wait();
        __syncwarp();
      }
#pragma unroll
      for (int jj = 0; jj < NBP; ++jj) {
        const int j = pass * NBP + jj;
        const int b = (valid && j < NB) ? partner<0>(a, 0, j) : -1;
        int32_t pos = -1;
        if (b >= 0) {
          const double* Kj = K[jj];
          const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
          bool tr = a > b;
          pos = (int32_t)(e * NUB + ub);
          if (dest) {
            const int32_t dd = s_dst[wib][g * NUB + ub];
            pos = dd >> 1;
            tr = tr != ((dd & 1) != 0);
          }
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) s_part[wib][tr ? 3 * k + i : 3 * i + k][lane] = Kj[3 * i + k];
        }
        s_pos[wib][lane] = pos;
        __syncwarp();
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          const int blk = 3 * it + bi;
          if (lane < 27 && blk < NLB) {
            const int32_t p = s_pos[wib][blk];
            if (p >= 0) k_store(Kscr + (int64_t)p * 9 + rr, s_part[wib][rr][blk]);
          }
        }
        __syncwarp();
      }
    }
  }
}

// T10 + Mooney-Rivlin (optionally Kelvin-Voigt) + geometry classes, two
// phases. Phase A, two lanes per (element, q): F (and Fdot) over 5 nodes each
// plus one shuffle, the MR state, S, S + S_v, and the symmetric 6x6 Voigt
// tangent (w-scaled, 21 entries; each lane builds 3 of the 6 columns) into
// shared memory. Phase B, one lane per node a: B_a (6x3) from F and grad N_a,
// C B_a, then K_ab = s_ab I + B_a^T C B_b (Eq. tangent_block, reading Q6/Q8)
// and f_a += F (w S_tot grad N_a). The lane-per-node kernel evaluated the MR
// state and S on all 10 lanes of an element and the tangent columns on 6.
__host__ __device__ __forceinline__ int cs_idx(int v, int w) {  // v <= w
  return v * 6 - (v * (v - 1)) / 2 + (w - v);
}

template <int NQ, bool KV>
__device__ __forceinline__ void element_group_t10mr(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab,
                                                    bool table_mode = false) {
  constexpr int NEN = 10, GROUP = 10, EPW = 3, NUB = 55, NB = 6, TABW = 3 * NEN + 1, KQ = 42;
  static_assert(EPW * NQ * 2 <= 32, "phase A: two lanes per (element, q)");
  __shared__ double s_k[kWarps][EPW][NQ][KQ];  // F (9), S (6), S + S_v (6), w C (21, upper Voigt)
  __shared__ double s_x[kWarps][EPW][3 * NEN];
  __shared__ double s_v[kWarps][KV ? EPW : 1][KV ? 3 * NEN : 1];
  __shared__ double s_node[kWarps][18][kLD];  // B_a per lane; reused as the store staging
  __shared__ int32_t s_dst[kWarps][EPW * NUB];
  __shared__ int32_t s_pos[kWarps][32];
  __shared__ int32_t s_cls[kWarps][EPW];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const int32_t* __restrict__ dest = A.dest;
  double* __restrict__ Kscr = A.Kscr;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = lane < EPW * GROUP;
  const int g = lane_active ? lane / GROUP : 0;
  const int a = lane_active ? lane % GROUP : 0;
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < n_el;
  const int gbase = g * GROUP;
  const bool write = dest;
  if (write) {
    const int64_t e0 = grp * EPW, lim = (n_el - e0) * NUB;
    for (int t = lane; t < EPW * NUB; t += 32)
      if (t < lim) pf_cp4(&s_dst[wib][t], dest + e0 * NUB + t);
  }
  int32_t fd = 0;
  if (lane_active) {
    double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
    int ce = 0;
    if (valid) {
      fd = A.fdest ? A.fdest[e * NEN + a] : (int32_t)(e * NEN + a);
      const int64_t I = A.conn[e * NEN + a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xa[i] = A.x[3 * I + i];
        if (KV) va[i] = A.v[3 * I + i];
      }
      if (a == 0) ce = table_mode ? wib * EPW + g : A.cls[e];
    }
    if (table_mode) ce = wib * EPW + g;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      s_x[wib][g][3 * a + i] = xa[i];
      if (KV) s_v[wib][g][3 * a + i] = va[i];
    }
    if (a == 0) s_cls[wib][g] = ce;
  }
  __syncwarp();
  {  // ---- phase A
    const bool act = lane < EPW * NQ * 2;
    const int pr = act ? lane >> 1 : 0, hf = lane & 1;
    const int ge = pr / NQ, q = pr - NQ * (pr / NQ);
    const double* t = s_tab + (s_cls[wib][ge] * NQ + q) * TABW;
    double F[9], Fd[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = Fd[r] = 0.0;
#pragma unroll
    for (int bb = 0; bb < NEN / 2; ++bb) {
      const int b = hf * (NEN / 2) + bb;
      const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xi = s_x[wib][ge][3 * b + i];
        F[3 * i] = fma(xi, n0, F[3 * i]);
        F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
        F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        if (KV) {
          const double vi = s_v[wib][ge][3 * b + i];
          Fd[3 * i] = fma(vi, n0, Fd[3 * i]);
          Fd[3 * i + 1] = fma(vi, n1, Fd[3 * i + 1]);
          Fd[3 * i + 2] = fma(vi, n2, Fd[3 * i + 2]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const double o = __shfl_xor_sync(0xffffffffu, F[r], 1);
      F[r] = hf ? o + F[r] : F[r] + o;
      if (KV) {
        const double od = __shfl_xor_sync(0xffffffffu, Fd[r], 1);
        Fd[r] = hf ? od + Fd[r] : Fd[r] + od;
      }
    }
    MRState ms;
    mr_state(F, ms);
    const double w = t[3 * NEN];
    if (act) {
      double* kq = s_k[wib][ge][q];
      if (hf == 0) {
        if (grp * EPW + ge < n_el && !(ms.J > 0.0)) atomicMin(A.err, (unsigned long long)((grp * EPW + ge) * 64 + q));
        double S[6];
        mr_S(ms, mat.C10, mat.C01, mat.kappa, S);
#pragma unroll
        for (int r = 0; r < 9; ++r) kq[r] = F[r];
#pragma unroll
        for (int r = 0; r < 6; ++r) kq[9 + r] = S[r];
        double Sv[6] = {0, 0, 0, 0, 0, 0};
        if (KV) kv_S(F, Fd, mat.eta, mat.lamd, Sv);
#pragma unroll
        for (int r = 0; r < 6; ++r) kq[15 + r] = S[r] + Sv[r];
      }
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {
        const int col = 3 * hf + cc;
        double cv[6];
        mr_Cv_column_dispatch(ms, mat.C10, mat.C01, mat.kappa, col, cv);
#pragma unroll
        for (int vv = 0; vv < 6; ++vv)
          if (vv <= col) kq[21 + cs_idx(vv, col)] = w * cv[vv];
      }
    }
  }
  __syncwarp();
  // ---- phase B (one pass: 6 blocks per lane)
  const int ce = s_cls[wib][g];
  double fa[3] = {0, 0, 0};
  double K[NB][9];
#pragma unroll
  for (int j = 0; j < NB; ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) K[j][r] = 0.0;
#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    const double* t = s_tab + (ce * NQ + q) * TABW;
    const double* kq = s_k[wib][g][q];
    const double gN[3] = {t[3 * a], t[3 * a + 1], t[3 * a + 2]};
    const double w = t[3 * NEN];
    double F[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = kq[r];
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
      for (int i = 0; i < 3; ++i) s_node[wib][3 * vv + i][lane] = Ba[vv][i];
    double tw[3], tt[3];
#pragma unroll
    for (int I = 0; I < 3; ++I) {
      tw[I] = w * (kq[9 + vidx(I, 0)] * gN[0] + kq[9 + vidx(I, 1)] * gN[1] + kq[9 + vidx(I, 2)] * gN[2]);
      tt[I] = w * (kq[15 + vidx(I, 0)] * gN[0] + kq[15 + vidx(I, 1)] * gN[1] + kq[15 + vidx(I, 2)] * gN[2]);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) fa[i] = fma(F[3 * i], tt[0], fma(F[3 * i + 1], tt[1], fma(F[3 * i + 2], tt[2], fa[i])));
    double CB[6][3];
#pragma unroll
    for (int vv = 0; vv < 6; ++vv)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double sacc = 0.0;
#pragma unroll
        for (int ww = 0; ww < 6; ++ww)
          sacc = fma(kq[21 + (vv <= ww ? cs_idx(vv, ww) : cs_idx(ww, vv))], Ba[ww][i], sacc);
        CB[vv][i] = sacc;
      }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = partner<0>(a, 0, j);
      if (b < 0) continue;
      double* Kj = K[j];
      const int lb = gbase + b;
      const double sv = fma(tw[0], t[3 * b], fma(tw[1], t[3 * b + 1], tw[2] * t[3 * b + 2]));
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double bb[6];
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) bb[vv] = s_node[wib][3 * vv + k][lb];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double acc = Kj[3 * i + k];
#pragma unroll
          for (int vv = 0; vv < 6; ++vv) acc = fma(CB[vv][i], bb[vv], acc);
          Kj[3 * i + k] = (i == k) ? acc + sv : acc;
        }
      }
    }
    __syncwarp();
  }
  if (valid) {
    double* fo = A.fscr + (int64_t)fd * 3;
    if (TLFEA_CHECK) TL_FCHK(fo);
    fo[0] = fa[0];
    fo[1] = fa[1];
    fo[2] = fa[2];
  }
  // warp-staged block stores (staging in s_node rows 0..8)
  constexpr int NLB = EPW * GROUP, NIT = (NLB + 2) / 3;
  const int bi = lane / 9, rr = lane - 9 * (lane / 9);
  if (write) {
    pf_wait();
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int b = (valid && j < NB) ? partner<0>(a, 0, j) : -1;
    int32_t pos = -1;
    if (b >= 0) {
      const double* Kj = K[j];
      const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
      bool tr = a > b;
      pos = (int32_t)(e * NUB + ub);
      if (dest) {
        const int32_t dd = s_dst[wib][g * NUB + ub];
        pos = dd >> 1;
        tr = tr != ((dd & 1) != 0);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) s_node[wib][tr ? 3 * k + i : 3 * i + k][lane] = Kj[3 * i + k];
    }
    s_pos[wib][lane] = pos;
    __syncwarp();
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int blk = 3 * it + bi;
      if (lane < 27 && blk < NLB) {
        const int32_t p = s_pos[wib][blk];
        if (p >= 0) k_store(Kscr + (int64_t)p * 9 + rr, s_node[wib][rr][blk]);
      }
    }
    __syncwarp();
  }
}

// Force-only counterpart (tlfea_force_only, the AdamW inner evaluation): phase A,
// one lane per (element, q), forms w P = w F S (Eq. F_assembly, reading Q5, J0 w
// folded in) once; phase B, one lane per (element, node a), contracts
// f_a = sum_q (w P) grad N_a (Eq. fint_local). The lane-per-node kernel reduced
// F and evaluated S on all 10 lanes of an element at every q.
template <int NQ, bool TA = false>
__device__ __forceinline__ void element_group_t10svk_force(int64_t grp, const ElArgs& A,
                                                           const double* __restrict__ s_tab, const T10Pre& pre) {
  constexpr int NEN = 10, GROUP = 10, EPW = 3, TABW = 3 * NEN + 1;
  __shared__ double s_x[kWarps][EPW][3 * NEN];
  __shared__ double s_pw[kWarps][EPW][NQ][9];
  __shared__ int32_t s_cls[kWarps][EPW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = lane < EPW * GROUP;
  const int g = lane_active ? lane / GROUP : 0;
  const int a = lane_active ? lane % GROUP : 0;
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < A.n_el;
  if (lane_active) {
#pragma unroll
    for (int i = 0; i < 3; ++i) s_x[wib][g][3 * a + i] = pre.xa[i];
    if (a == 0) s_cls[wib][g] = pre.ce;
  }
  __syncwarp();
  if constexpr (TA) {
    pf_wait();
    __syncwarp();
  }
  if (lane < EPW * NQ) {
    const int ge = lane / NQ, q = lane - NQ * (lane / NQ);
    const double* t = s_tab + (s_cls[wib][ge] * NQ + q) * TABW;
    const double* xs = s_x[wib][ge];
    double F[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
    for (int b = 0; b < NEN; ++b) {
      const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xi = xs[3 * b + i];
        F[3 * i] = fma(xi, n0, F[3 * i]);
        F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
        F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
      }
    }
    double S[6];
    svk_S(F, A.mat.lam, A.mat.mu, S);
    const double w = t[3 * NEN];
    double* pw = s_pw[wib][ge][q];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int J = 0; J < 3; ++J)
        pw[3 * i + J] = w * (F[3 * i] * sget(S, 0, J) + F[3 * i + 1] * sget(S, 1, J) + F[3 * i + 2] * sget(S, 2, J));
  }
  __syncwarp();
  if (!valid) return;
  const int ce = s_cls[wib][g];
  double fa[3] = {0, 0, 0};
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double* t = s_tab + (ce * NQ + q) * TABW + 3 * a;
    const double* pw = s_pw[wib][g][q];
    const double n0 = t[0], n1 = t[1], n2 = t[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) fa[i] = fma(pw[3 * i], n0, fma(pw[3 * i + 1], n1, fma(pw[3 * i + 2], n2, fa[i])));
  }
  double* fo = A.fscr + (int64_t)pre.fd * 3;
  if (TLFEA_CHECK) TL_FCHK(fo);
  fo[0] = fa[0];
  fo[1] = fa[1];
  fo[2] = fa[2];
}

// Force-only T10 SVK with geometry classes, wide groups (the AdamW inner
// evaluation, Alg. 2; Eq. F_assembly / fint_local as above): a warp
// holds EPW = 32 / NQ elements so that phase A (one lane per (element, q):
// F, S, w P = w F S) runs on every lane instead of 12 of 32; phase B walks the
// EPW x 10 (element, node) tasks in rounds of 32 lanes. kFW warps per CTA
// amortize the class-table copy over kFW * EPW elements; the element range
// need not be tile aligned (element = e_begin + warp * EPW + g).
constexpr int kFW = 8;
#ifndef TLFEA_FORCE_WIDE
#define TLFEA_FORCE_WIDE 1
#endif
#ifndef TLFEA_FW_PERSIST
#define TLFEA_FW_PERSIST 1  // persistent warps, next group's inputs prefetched
#endif
#ifndef TLFEA_FW_MINB
#define TLFEA_FW_MINB 3  // 5-point rule (6 elements per warp): 80 registers; config 5 0.577 ms vs 0.574 at 2, 0.64 at 4 (spills)
#endif
#ifndef TLFEA_FW_MINB4
#define TLFEA_FW_MINB4 2  // 4-point rule (8 elements per warp, 3 node rounds): 3 CTAs/SM spill 80 B
#endif
template <int NQ>
struct FwIdx {  // one group's indices: node ids, force destinations, class id
  static constexpr int NT = (32 / NQ) * 10, NR = (NT + 31) / 32;
  int32_t node[NR];
  int32_t fd[NR];
  int32_t ce;
};
template <int NQ>
__device__ __forceinline__ void fw_load_idx(const ElArgs& A, int64_t e0, FwIdx<NQ>& in) {
  constexpr int NEN = 10, EPW = 32 / NQ;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < FwIdx<NQ>::NR; ++r) {
    const int t = lane + 32 * r;
    const int64_t e = e0 + t / NEN;
    in.node[r] = -1;
    in.fd[r] = -1;
    if (t < FwIdx<NQ>::NT && e < A.n_el) {
      const int64_t ea = e * NEN + t % NEN;
      in.fd[r] = A.fdest ? A.fdest[ea] : (int32_t)ea;
      in.node[r] = A.conn[ea];
    }
  }
  in.ce = (lane < EPW && e0 + lane < A.n_el) ? A.cls[e0 + lane] : 0;
}
template <int NQ>
__device__ __forceinline__ void fw_load_x(const ElArgs& A, const FwIdx<NQ>& in, double (*x)[3]) {
#pragma unroll
  for (int r = 0; r < FwIdx<NQ>::NR; ++r) {
    x[r][0] = x[r][1] = x[r][2] = 0.0;
    if (in.node[r] >= 0) {
      const int64_t I = in.node[r];
#pragma unroll
      for (int i = 0; i < 3; ++i) x[r][i] = A.x[3 * I + i];
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(kFW * 32, NQ == 4 ? TLFEA_FW_MINB4 : TLFEA_FW_MINB) k_force_t10svk_wide(ElArgs A, int64_t e_begin) {
  constexpr int NEN = 10, EPW = 32 / NQ, NT = EPW * NEN, NR = (NT + 31) / 32, TABW = 3 * NEN + 1;
  extern __shared__ double s_tab[];  // [n_cls][NQ][3 NEN + 1]
  __shared__ double s_x[kFW][EPW][3 * NEN];
  __shared__ double s_pw[kFW][EPW][NQ][9];
  __shared__ int32_t s_cls[kFW][EPW];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n_el = A.n_el, stride = (int64_t)gridDim.x * kFW * EPW;
  int64_t e0 = e_begin + ((int64_t)blockIdx.x * kFW + wib) * EPW;
  // software pipeline: group k computes while group k+1's coordinates and
  // group k+2's indices are in flight (the coordinate loads depend on the
  // indices, so they are issued one group apart)
  FwIdx<NQ> cur, nxt;
  double xr[NR][3];
  fw_load_idx<NQ>(A, e0, cur);
  if (TLFEA_FW_PERSIST) fw_load_idx<NQ>(A, e0 + stride, nxt);
  fw_load_x<NQ>(A, cur, xr);
  {
    const int tot = A.n_cls * NQ * TABW;
    constexpr int U = 8;
    for (int t = threadIdx.x; t < tot; t += U * blockDim.x) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = t + u * (int)blockDim.x < tot ? A.cls_tab[t + u * blockDim.x] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t + u * (int)blockDim.x < tot) s_tab[t + u * blockDim.x] = v[u];
    }
  }
  __syncthreads();
  for (; e0 < n_el; e0 += stride) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int t = lane + 32 * r;
      if (t < NT)
#pragma unroll
        for (int i = 0; i < 3; ++i) s_x[wib][t / NEN][3 * (t % NEN) + i] = xr[r][i];
    }
    if (lane < EPW) s_cls[wib][lane] = cur.ce;
    int32_t fd[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) fd[r] = cur.fd[r];
    __syncwarp();
    if (TLFEA_FW_PERSIST) {
      cur = nxt;
      fw_load_x<NQ>(A, cur, xr);
      fw_load_idx<NQ>(A, e0 + 2 * stride, nxt);
    }
    if (lane < EPW * NQ) {  // phase A: F, S, w P = w F S at (element ge, point q)
      const int ge = lane / NQ, q = lane - NQ * ge;
      const double* t = s_tab + (s_cls[wib][ge] * NQ + q) * TABW;
      const double* xs = s_x[wib][ge];
      double F[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
      for (int b = 0; b < NEN; ++b) {
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xi = xs[3 * b + i];
          F[3 * i] = fma(xi, n0, F[3 * i]);
          F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
          F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        }
      }
      double S[6];
      svk_S(F, A.mat.lam, A.mat.mu, S);
      const double w = t[3 * NEN];
      double* pw = s_pw[wib][ge][q];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int J = 0; J < 3; ++J)
          pw[3 * i + J] = w * (F[3 * i] * sget(S, 0, J) + F[3 * i + 1] * sget(S, 1, J) + F[3 * i + 2] * sget(S, 2, J));
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NR; ++r) {  // phase B: f_a = sum_q (w P)_q grad N_a(q)
      const int t = lane + 32 * r;
      if (fd[r] < 0) continue;
      const int g = t / NEN, a = t % NEN, ce = s_cls[wib][g];
      double fa[3] = {0, 0, 0};
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double* tq = s_tab + (ce * NQ + q) * TABW + 3 * a;
        const double* pw = s_pw[wib][g][q];
        const double n0 = tq[0], n1 = tq[1], n2 = tq[2];
#pragma unroll
        for (int i = 0; i < 3; ++i) fa[i] = fma(pw[3 * i], n0, fma(pw[3 * i + 1], n1, fma(pw[3 * i + 2], n2, fa[i])));
      }
      double* fo = A.fscr + (int64_t)fd[r] * 3;
      if (TLFEA_CHECK) TL_FCHK(fo);
      fo[0] = fa[0];
      fo[1] = fa[1];
      fo[2] = fa[2];
    }
    __syncwarp();
    if (!TLFEA_FW_PERSIST) break;
  }
}


// ------------------------------------------ T10 SVK force only, affine form
// Straight-sided T10 (every mesh with the affine min layout, and congruent
// meshes whose classes are straight-sided): grad N is linear in the
// barycentric coordinates z, so with the four constant gradients grad z_k
// (SURVEY §8(d) min layout, P:312-320 with J constant) the element needs no
// per-point tables:
//   F(z) = sum_k z_k G_k,  G_k = 4 (x_k (x) grad z_k + sum_{j != k} x_kj (x) grad z_j) - C,
//   C = sum_i x_i (x) grad z_i   (x_kj: the mid-edge node of edge (k, j); sum z = 1)
// is the T10 deformation gradient of Eq. F_assembly at any point, and
// with wP_q = J0 w_q F_q S_q (reading Q5), Q_i = sum_q z_qi wP_q, R = sum_q wP_q:
//   corner i: f_i = sum_q wP_q grad N_i(z_q) = (4 Q_i - R) grad z_i,
//   edge (a,b): f = 4 (Q_a grad z_b + Q_b grad z_a)          (Eq. fint_local).
// The rules' points are permutations, so F_q and Q_i cost a few FMAs each
// (Keast-5: F_0 = T/4, F_q = T/6 + G_{q-1}/3 with T = sum_k G_k; 4-point:
// F_q = beta T + (alpha - beta) G_q). One thread per element, all in registers:
// no shared-memory traffic (the two-phase kernels above are bound by it).
#ifndef TLFEA_FORCE_AFF
#define TLFEA_FORCE_AFF 1
#endif
#ifndef TLFEA_INR_CLOSED
#define TLFEA_INR_CLOSED 1  // AdamW element inertia: closed-form T10 mass (mass_rule 0) instead of the class rows
#endif
#ifndef TLFEA_FA_MINB
#define TLFEA_FA_MINB 3  // config 5: 0.263 ms at 3 CTAs/SM (166 registers) vs 0.283 at 4 (128, spills), 0.320 at 2
#endif
constexpr int kFABlock = 128;
// INR (the AdamW gradient, classes only): each element also adds its inertia
// (1/h) sum_b m_ab (v - v_n)_b (Eq. residual P:101-113 element by element, the
// class element mass of setup) to its nodal forces, so the gradient gather
// sums the force scratch without the mass-row SpMV.
template <int NQ, bool CLS, bool INR = false>
__global__ void __launch_bounds__(kFABlock, TLFEA_FA_MINB) k_force_t10_aff(ElArgs A, int64_t e_begin,
                                                                           const double* __restrict__ cls_aff) {
  extern __shared__ double s_aff[];  // CLS: [n_cls][13] (INR: then [n_cls][100] element masses)
  if (CLS) {
    for (int t = threadIdx.x; t < A.n_cls * 13; t += blockDim.x) s_aff[t] = cls_aff[t];
    if (INR)
      for (int t = threadIdx.x; t < A.n_cls * 100; t += blockDim.x) s_aff[A.n_cls * 13 + t] = A.cls_mass[t];
    __syncthreads();
  }
  const int64_t e = e_begin + (int64_t)blockIdx.x * kFABlock + threadIdx.x;
  if (e >= A.n_el) return;
  const double* af = CLS ? s_aff + 13 * A.cls[e] : A.aff + 13 * e;
  double gz[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) gz[i][k] = af[3 * i + k];
  const double J0 = af[12];
  int32_t nd[10];
#pragma unroll
  for (int a = 0; a < 10; ++a) nd[a] = A.conn[e * 10 + a];
  double x[10][3];
#pragma unroll
  for (int a = 0; a < 10; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) x[a][i] = A.x[3 * (int64_t)nd[a] + i];
  // edge node of (k, j) in the local order of reading Q2: 4 (0,1) 5 (1,2) 6 (2,0) 7 (0,3) 8 (1,3) 9 (2,3)
  constexpr int EDGE[4][4] = {{-1, 4, 6, 7}, {4, -1, 5, 8}, {6, 5, -1, 9}, {7, 8, 9, -1}};
  double C[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = x[0][r] * gz[0][c] + x[1][r] * gz[1][c] + x[2][r] * gz[2][c] + x[3][r] * gz[3][c];
  double G[4][9], T[9];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double h = x[k][r] * gz[k][c];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j != k) h = fma(x[EDGE[k][j]][r], gz[j][c], h);
        G[k][3 * r + c] = fma(4.0, h, -C[3 * r + c]);
      }
#pragma unroll
  for (int r = 0; r < 9; ++r) T[r] = (G[0][r] + G[1][r]) + (G[2][r] + G[3][r]);
  const double lam = A.mat.lam, mu = A.mat.mu;
  // wP at one point: J0 w F S
  auto wP_at = [&](const double F[9], double jw, double out[9]) {
    double S[6];
    svk_S(F, lam, mu, S);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int J = 0; J < 3; ++J)
        out[3 * i + J] = jw * (F[3 * i] * sget(S, 0, J) + F[3 * i + 1] * sget(S, 1, J) + F[3 * i + 2] * sget(S, 2, J));
  };
  double P4[4][9], base[9], R[9];  // per-permutation-point wP, and the parts shared by all Q_i
  double ca, cr;                   // Q_i = base + ca P4[i];  4 Q_i - R = 4 base - R + 4 ca P4[i]
  if constexpr (NQ == 5) {  // Keast (reading Q1): centroid w = -2/15; z_{q-1} = 1/2, others 1/6, w = 3/40
    double F[9], P0[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = 0.25 * T[r];
    wP_at(F, J0 * (-2.0 / 15.0), P0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = fma(1.0 / 3.0, G[k][r], T[r] * (1.0 / 6.0));
      wP_at(F, J0 * (3.0 / 40.0), P4[k]);
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const double U = (P4[0][r] + P4[1][r]) + (P4[2][r] + P4[3][r]);
      base[r] = fma(0.25, P0[r], U * (1.0 / 6.0));
      R[r] = P0[r] + U;
    }
    ca = 1.0 / 3.0;
  } else {  // 4-point degree 2: z_q = alpha at q, beta elsewhere, w = 1/24
    const double r5 = 2.2360679774997896964;
    const double alpha = 0.25 + 0.15 * r5, beta = 0.25 - 0.05 * r5;
    double F[9];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = fma(alpha - beta, G[k][r], beta * T[r]);
      wP_at(F, J0 * (1.0 / 24.0), P4[k]);
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      R[r] = (P4[0][r] + P4[1][r]) + (P4[2][r] + P4[3][r]);
      base[r] = beta * R[r];
    }
    ca = alpha - beta;
  }
  (void)cr;
  double f[10][3];
#pragma unroll
  for (int i = 0; i < 4; ++i)  // corners: (4 Q_i - R) grad z_i
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) s = fma(fma(4.0, fma(ca, P4[i][3 * r + c], base[3 * r + c]), -R[3 * r + c]), gz[i][c], s);
      f[i][r] = s;
    }
  constexpr int EA[6] = {0, 1, 2, 0, 1, 2}, EB[6] = {1, 2, 0, 3, 3, 3};
#pragma unroll
  for (int m = 0; m < 6; ++m)  // edges: 4 (Q_a grad z_b + Q_b grad z_a)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double qa = fma(ca, P4[EA[m]][3 * r + c], base[3 * r + c]);
        const double qb = fma(ca, P4[EB[m]][3 * r + c], base[3 * r + c]);
        s = fma(qa, gz[EB[m]][c], fma(qb, gz[EA[m]][c], s));
      }
      f[4 + m][r] = 4.0 * s;
    }
  if constexpr (INR) {
    double dv[10][3];
#pragma unroll
    for (int b = 0; b < 10; ++b)
#pragma unroll
      for (int i = 0; i < 3; ++i) dv[b][i] = A.v[3 * (int64_t)nd[b] + i];  // v - v_n (the AdamW update wrote it)
#if TLFEA_INR_CLOSED
    if (A.mass_closed) {
      // the exact consistent mass of a straight-sided T10 (reading Q4):
      // m_ab = rho V / 420 C_ab, C = {corner-corner 6 | 1; corner-edge -4 on the
      // edge, else -6; edge-edge 32 | 16 sharing a vertex | 8 opposite}, so with
      // S_c, S_e the corner / edge sums of v - v_n:
      //   corner i: 5 dv_i + S_c - 6 S_e + 2 (sum of the edges at i)
      //   edge (a,b): 2 (dv_a + dv_b) - 6 S_c + 16 S_e + 16 dv_m - 8 dv_opposite
      const double sc = A.mat.rho0 * J0 / 2520.0 * A.inv_h;  // rho V / 420 / h, V = J0 / 6
      constexpr int EA2[6] = {0, 1, 2, 0, 1, 2}, EB2[6] = {1, 2, 0, 3, 3, 3}, OPP[6] = {9, 7, 8, 5, 6, 4};
      constexpr int AT[4][3] = {{4, 6, 7}, {4, 5, 8}, {5, 6, 9}, {7, 8, 9}};  // edges at corner i
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double Sc = (dv[0][i] + dv[1][i]) + (dv[2][i] + dv[3][i]);
        const double Se = ((dv[4][i] + dv[5][i]) + (dv[6][i] + dv[7][i])) + (dv[8][i] + dv[9][i]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double r = 5.0 * dv[c][i] + Sc - 6.0 * Se + 2.0 * ((dv[AT[c][0]][i] + dv[AT[c][1]][i]) + dv[AT[c][2]][i]);
          f[c][i] = fma(r, sc, f[c][i]);
        }
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          const double r = 2.0 * (dv[EA2[m]][i] + dv[EB2[m]][i]) - 6.0 * Sc + 16.0 * Se + 16.0 * dv[4 + m][i] -
                           8.0 * dv[OPP[m]][i];
          f[4 + m][i] = fma(r, sc, f[4 + m][i]);
        }
      }
    } else
#endif
    {
    const double* me = s_aff + A.n_cls * 13 + 100 * A.cls[e];
#pragma unroll
    for (int a = 0; a < 10; ++a) {
      double r[3] = {0, 0, 0};
#pragma unroll
      for (int b = 0; b < 10; ++b) {
        const double mab = me[10 * a + b];
#pragma unroll
        for (int i = 0; i < 3; ++i) r[i] = fma(mab, dv[b][i], r[i]);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) f[a][i] = fma(r[i], A.inv_h, f[a][i]);
    }
    }
  }
#pragma unroll
  for (int a = 0; a < 10; ++a) {
    const int64_t fp = A.fdest ? (int64_t)A.fdest[e * 10 + a] : e * 10 + a;
    double* fo = A.fscr + 3 * fp;
    if (TLFEA_CHECK) TL_FCHK(fo);
    fo[0] = f[a][0];
    fo[1] = f[a][1];
    fo[2] = f[a][2];
  }
}


// ------------------------------------ force only, one lane per point
// ANCF3443 (16 coefficients, 48 points), ANCF3243 (8, 12) and T10 with
// Mooney-Rivlin or Kelvin-Voigt (10, 4 or 5: 6-8 elements per warp) force only
// (tlfea_force_only, the AdamW inner evaluation, Alg. 2): one lane
// per (element, quadrature point) computes F (and Fdot) = sum_a (x_a, v_a) (x)
// grad N_a (Eq. F_assembly), the stress (SVK / MR, + Kelvin-Voigt) and
// accumulates its point's f_a += w P grad N_a for all the element's
// coefficients (Eq. fint_local); the partials are summed over the element's
// lanes through shared memory in ascending lane order (deterministic). The
// lane-per-coefficient group reduced F through shared memory and evaluated
// the stress on every lane at every point.
#ifndef TLFEA_FORCE_LPQ
#define TLFEA_FORCE_LPQ 1
#endif
template <int ELEM, int NQ, int MODEL, bool KV, bool CLS>
__global__ void __launch_bounds__(kWarps * 32) k_force_lpq(ElArgs A, int64_t e_begin) {
  constexpr int NEN = Geo<ELEM>::NEN, TABW = 3 * NEN + 1, ND = 3 * NEN, LDF = ND + 1;
  constexpr int EPW = NQ >= 32 ? 1 : 32 / NQ, NR = (NQ + 31) / 32;
  extern __shared__ double s_dyn[];  // [kWarps][32][LDF] lane partials, then (CLS) [n_cls][NQ][TABW]
  __shared__ double s_x[kWarps][EPW][ND];
  __shared__ double s_v[kWarps][KV ? EPW : 1][KV ? ND : 1];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* s_f = s_dyn + (size_t)wib * 32 * LDF;
  const double* s_tab = s_dyn + (size_t)kWarps * 32 * LDF;
  if (CLS) {
    double* st = s_dyn + (size_t)kWarps * 32 * LDF;
    for (int t = threadIdx.x; t < A.n_cls * NQ * TABW; t += blockDim.x) st[t] = A.cls_tab[t];
  }
  const int64_t e0 = e_begin + ((int64_t)blockIdx.x * kWarps + wib) * EPW;
  for (int t = lane; t < EPW * NEN; t += 32) {
    const int g = t / NEN, a = t - NEN * g;
    const int64_t e = e0 + g;
    double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
    if (e < A.n_el) {
      const int64_t I = A.conn[e * NEN + a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xa[i] = A.x[3 * I + i];
        if (KV) va[i] = A.v[3 * I + i];
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      s_x[wib][g][3 * a + i] = xa[i];
      if (KV) s_v[wib][g][3 * a + i] = va[i];
    }
  }
  __syncthreads();
  const int g = NQ >= 32 ? 0 : lane / NQ;
  const int64_t e = e0 + g;
  const bool act = (NQ >= 32 || lane < EPW * NQ) && e < A.n_el;
  const int ce = (CLS && act) ? A.cls[e] : 0;
  double f[ND];
#pragma unroll
  for (int r = 0; r < ND; ++r) f[r] = 0.0;
#pragma unroll
  for (int rnd = 0; rnd < NR; ++rnd) {
    const int q = NQ >= 32 ? lane + 32 * rnd : lane - NQ * g;
    if (!act || q >= NQ) continue;
    const double* gN;
    double w;
    if (CLS) {
      gN = s_tab + (ce * NQ + q) * TABW;
      w = gN[ND];
    } else {
      gN = A.gradN + (e * NQ + q) * ND;
      w = A.J0w[e * NQ + q];
    }
    double F[9], Fd[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = Fd[r] = 0.0;
#pragma unroll
    for (int b = 0; b < NEN; ++b) {
      const double n0 = gN[3 * b], n1 = gN[3 * b + 1], n2 = gN[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xi = s_x[wib][g][3 * b + i];
        F[3 * i] = fma(xi, n0, F[3 * i]);
        F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
        F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        if (KV) {
          const double vi = s_v[wib][g][3 * b + i];
          Fd[3 * i] = fma(vi, n0, Fd[3 * i]);
          Fd[3 * i + 1] = fma(vi, n1, Fd[3 * i + 1]);
          Fd[3 * i + 2] = fma(vi, n2, Fd[3 * i + 2]);
        }
      }
    }
    double S[6];
    if (MODEL == 0) {
      svk_S(F, A.mat.lam, A.mat.mu, S);
    } else {
      MRState ms;
      mr_state(F, ms);
      if (!(ms.J > 0.0)) atomicMin(A.err, (unsigned long long)(e * 64 + q));
      mr_S(ms, A.mat.C10, A.mat.C01, A.mat.kappa, S);
    }
    if (KV) {
      double Sv[6];
      kv_S(F, Fd, A.mat.eta, A.mat.lamd, Sv);
#pragma unroll
      for (int r = 0; r < 6; ++r) S[r] += Sv[r];
    }
    double P[9];  // w F S
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int J = 0; J < 3; ++J)
        P[3 * i + J] = w * (F[3 * i] * sget(S, 0, J) + F[3 * i + 1] * sget(S, 1, J) + F[3 * i + 2] * sget(S, 2, J));
#pragma unroll
    for (int b = 0; b < NEN; ++b) {
      const double n0 = gN[3 * b], n1 = gN[3 * b + 1], n2 = gN[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) f[3 * b + i] = fma(P[3 * i], n0, fma(P[3 * i + 1], n1, fma(P[3 * i + 2], n2, f[3 * b + i])));
    }
  }
#pragma unroll
  for (int r = 0; r < ND; ++r) s_f[lane * LDF + r] = f[r];
  __syncwarp();
  // f of (element g2, value r) = sum over the element's lanes in ascending order
  for (int t = lane; t < EPW * ND; t += 32) {
    const int g2 = t / ND, r = t - ND * g2;
    const int64_t e2 = e0 + g2;
    if (e2 >= A.n_el) continue;
    const int l0 = NQ >= 32 ? 0 : g2 * NQ, l1 = NQ >= 32 ? 32 : l0 + NQ;
    double sum = 0.0;
    for (int l = l0; l < l1; ++l) sum += s_f[l * LDF + r];
    const int a = r / 3, i = r - 3 * a;
    const int64_t fp = A.fdest ? (int64_t)A.fdest[e2 * NEN + a] : e2 * NEN + a;
    if (TLFEA_CHECK) tl_chk(A.fscr + 3 * fp + i, 1, __LINE__);
    A.fscr[3 * fp + i] = sum;
  }
}

#ifndef TLFEA_ANCF_NPASS
#define TLFEA_ANCF_NPASS 1  // block passes (each re-runs phase A per chunk)
#endif
#ifndef TLFEA_ANCF_MINB
#define TLFEA_ANCF_MINB 3  // config 4: 1.312 ms at 3 CTAs/SM (168 registers, 28 B spill) vs 1.347 at 2
#endif
// ANCF3443 plate element (16 coefficients, GL 4x4x3 = 48 points), SVK, no KV,
// geometry classes: the two-phase scheme of element_group_t10svk with one
// element per warp and the quadrature points in chunks of QC = 8.
//   phase A (per chunk): lanes (q, s), four per point, each owning 4 of the 16
//            coefficients: partial F, two shuffles, then S (s = 0) or F F^T
//            (s = 1) and g_b = F grad N_b of its coefficients into shared memory;
//   phase B (per chunk): lanes (node a, half) accumulate their 4-5 upper blocks
//            over the chunk's points (and f_a on half 0) from shared memory.
// The lane-per-node kernel evaluated the per-point kinematics on all 32 lanes
// (fp64 pipe 62 % busy on config 4, ~40 % of it kinematics).
template <int NQ>
__device__ __forceinline__ void element_group_ancf_svk(int64_t e, const ElArgs& A, const double* __restrict__ s_tab) {
  constexpr int NEN = 16, NUB = 136, NB = 5, TABW = 3 * NEN + 1, QC = 8, LPQ = 4, NPL = NEN / LPQ, LDG = NEN + 1;
  static_assert(NQ % QC == 0 && QC * LPQ == 32, "quadrature points in whole chunks, one lane group per point");
  __shared__ double s_ga[kWarps][QC][3][LDG];
  __shared__ double s_k[kWarps][QC][21];  // F (9), S (6), F F^T (6)
  __shared__ double s_x[kWarps][3 * NEN];
  __shared__ double s_part[kWarps][9][kLD];
  __shared__ int32_t s_dst[kWarps][NUB];
  __shared__ int32_t s_pos[kWarps][32];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const int32_t* __restrict__ dest = A.dest;
  double* __restrict__ Kscr = A.Kscr;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int a = lane & 15, half = lane >> 4;
  const bool valid = e < n_el;
  if (!valid) return;  // warp-uniform (one element per warp)
  const bool write = dest;
  if (write) {
    for (int t = lane; t < NUB; t += 32) pf_cp4(&s_dst[wib][t], dest + e * NUB + t);
  }
  const int ce = A.cls[e];
  if (half == 0) {
    const int64_t I = A.conn[e * NEN + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) s_x[wib][3 * a + i] = A.x[3 * I + i];
  }
  const int32_t fd = (half == 0) ? (A.fdest ? A.fdest[e * NEN + a] : (int32_t)(e * NEN + a)) : 0;
  __syncwarp();
  constexpr int NPASS = TLFEA_ANCF_NPASS, NBP = (NB + NPASS - 1) / NPASS;
  double fa[3] = {0, 0, 0};
  double K[NBP][9];
  if (write) {
    pf_wait();
    __syncwarp();
  }
#pragma unroll 1
  for (int pass = 0; pass < NPASS; ++pass) {
#pragma unroll
  for (int j = 0; j < NBP; ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) K[j][r] = 0.0;
#pragma unroll 1
  for (int q0 = 0; q0 < NQ; q0 += QC) {
    // ---- phase A: LPQ = 4 lanes per point, NPL = 4 coefficients each
    {
      const int qq = lane / LPQ, sub = lane % LPQ;
      const double* t = s_tab + (ce * NQ + q0 + qq) * TABW;
      double F[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
      for (int bb = 0; bb < NPL; ++bb) {
        const int b = sub * NPL + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xi = s_x[wib][3 * b + i];
          F[3 * i] = fma(xi, n0, F[3 * i]);
          F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
          F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        }
      }
      // F = (p0 + p1) + (p2 + p3), the same bits on all four lanes
#pragma unroll
      for (int m = 1; m < LPQ; m <<= 1)
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          const double o = __shfl_xor_sync(0xffffffffu, F[r], m);
          F[r] = (sub & m) ? o + F[r] : F[r] + o;
        }
      double* kq = s_k[wib][qq];
      if (sub == 0) {
        double S[6];
        svk_S(F, mat.lam, mat.mu, S);
#pragma unroll
        for (int r = 0; r < 9; ++r) kq[r] = F[r];
#pragma unroll
        for (int r = 0; r < 6; ++r) kq[9 + r] = S[r];
      } else if (sub == 1) {
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int i, k;
          voigt_pair(vv, i, k);
          kq[15 + vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
        }
      }
#pragma unroll
      for (int bb = 0; bb < NPL; ++bb) {
        const int b = sub * NPL + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) s_ga[wib][qq][i][b] = F[3 * i] * n0 + F[3 * i + 1] * n1 + F[3 * i + 2] * n2;
      }
    }
    __syncwarp();
    // ---- phase B
#pragma unroll 1
    for (int qq = 0; qq < QC; ++qq) {
      const double* t = s_tab + (ce * NQ + q0 + qq) * TABW;
      const double* kq = s_k[wib][qq];
      const double gN[3] = {t[3 * a], t[3 * a + 1], t[3 * a + 2]};
      const double w = t[3 * NEN];
      double S[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) S[r] = kq[9 + r];
      double tw[3];
#pragma unroll
      for (int I = 0; I < 3; ++I) tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
      if (half == 0 && pass == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
          fa[i] = fma(kq[3 * i], tw[0], fma(kq[3 * i + 1], tw[1], fma(kq[3 * i + 2], tw[2], fa[i])));
      }
      const double lw = mat.lam * w, mw = mat.mu * w;
      double gl[3], gm[3], gNm[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double gai = s_ga[wib][qq][i][a];
        gl[i] = lw * gai;
        gm[i] = mw * gai;
        gNm[i] = mw * gN[i];
      }
      double B[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) B[r] = kq[15 + r];
#pragma unroll
      for (int jj = 0; jj < NBP; ++jj) {
        const int j = pass * NBP + jj;
        const int b = j < NB ? partner<1>(a, half, j) : -1;
        if (b < 0) continue;
        double* Kj = K[jj];
        const double gb[3] = {s_ga[wib][qq][0][b], s_ga[wib][qq][1][b], s_ga[wib][qq][2][b]};
        const double nb[3] = {t[3 * b], t[3 * b + 1], t[3 * b + 2]};
        const double sv = fma(tw[0], nb[0], fma(tw[1], nb[1], tw[2] * nb[2]));
        const double d = fma(gNm[0], nb[0], fma(gNm[1], nb[1], gNm[2] * nb[2]));
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double acc = fma(gl[i], gb[k], fma(gb[i], gm[k], fma(d, B[vidx(i, k)], Kj[3 * i + k])));
            Kj[3 * i + k] = (i == k) ? acc + sv : acc;
          }
      }
    }
    __syncwarp();
  }
  if (half == 0 && pass == 0) {
    double* fo = A.fscr + (int64_t)fd * 3;
    if (TLFEA_CHECK) TL_FCHK(fo);
    fo[0] = fa[0];
    fo[1] = fa[1];
    fo[2] = fa[2];
  }
  // warp-staged block stores, as in element_group
  constexpr int NLB = 32, NIT = (NLB + 2) / 3;
  const int bi = lane / 9, rr = lane - 9 * (lane / 9);
#pragma unroll
  for (int jj = 0; jj < NBP; ++jj) {
    const int j = pass * NBP + jj;
    const int b = j < NB ? partner<1>(a, half, j) : -1;
    int32_t pos = -1;
    if (b >= 0) {
      const double* Kj = K[jj];
      const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
      bool tr = a > b;
      pos = (int32_t)(e * NUB + ub);
      if (dest) {
        const int32_t dd = s_dst[wib][ub];
        pos = dd >> 1;
        tr = tr != ((dd & 1) != 0);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) s_part[wib][tr ? 3 * k + i : 3 * i + k][lane] = Kj[3 * i + k];
    }
    s_pos[wib][lane] = pos;
    __syncwarp();
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int blk = 3 * it + bi;
      if (lane < 27 && blk < NLB) {
        const int32_t p = s_pos[wib][blk];
        if (p >= 0) k_store(Kscr + (int64_t)p * 9 + rr, s_part[wib][rr][blk]);
      }
    }
    __syncwarp();
  }
  }  // pass
}

// ANCF3243 beam (8 coefficients, GL 3x2x2 = 12 points), SVK, no KV, geometry
// classes: the two-phase scheme with 4 elements per warp and the points in
// chunks of QC = 4: phase A on lanes (element, point, half) — two lanes per
// (element, point), 4 coefficients each — then phase B on lanes (element,
// node a) over the chunk's points. One block pass (4-5 blocks per lane).
template <int NQ>
__device__ __forceinline__ void element_group_beam_svk(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab) {
  constexpr int NEN = 8, GROUP = 8, EPW = 4, NUB = 36, NB = 5, TABW = 3 * NEN + 1, QC = 4;
  static_assert(NQ % QC == 0 && EPW * QC * 2 == 32, "one lane pair per (element, point) of a chunk");
  __shared__ double s_ga[kWarps][QC][3][kLD];
  __shared__ double s_k[kWarps][EPW][QC][21];
  __shared__ double s_x[kWarps][EPW][3 * NEN];
  __shared__ double s_part[kWarps][9][kLD];
  __shared__ int32_t s_dst[kWarps][EPW * NUB];
  __shared__ int32_t s_pos[kWarps][32];
  __shared__ int32_t s_cls[kWarps][EPW];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const int32_t* __restrict__ dest = A.dest;
  double* __restrict__ Kscr = A.Kscr;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane / GROUP, a = lane % GROUP, gbase = g * GROUP;
  const int64_t e = grp * EPW + g;
  const bool valid = e < n_el;
  const bool write = dest;
  if (write) {
    const int64_t e0 = grp * EPW, lim = (n_el - e0) * NUB;
    for (int t = lane; t < EPW * NUB; t += 32)
      if (t < lim) pf_cp4(&s_dst[wib][t], dest + e0 * NUB + t);
  }
  {
    double xa[3] = {0, 0, 0};
    int ce = 0;
    if (valid) {
      const int64_t I = A.conn[e * NEN + a];
#pragma unroll
      for (int i = 0; i < 3; ++i) xa[i] = A.x[3 * I + i];
      if (a == 0) ce = A.cls[e];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) s_x[wib][g][3 * a + i] = xa[i];
    if (a == 0) s_cls[wib][g] = ce;
  }
  const int32_t fd = valid ? (A.fdest ? A.fdest[e * NEN + a] : (int32_t)(e * NEN + a)) : 0;
  __syncwarp();
  const int ce = s_cls[wib][g];
  double fa[3] = {0, 0, 0};
  double K[NB][9];
#pragma unroll
  for (int j = 0; j < NB; ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) K[j][r] = 0.0;
#pragma unroll 1
  for (int q0 = 0; q0 < NQ; q0 += QC) {
    {  // ---- phase A
      const int pr = lane >> 1, hf = lane & 1;
      const int ge = pr / QC, qq = pr - QC * (pr / QC);
      const double* t = s_tab + (s_cls[wib][ge] * NQ + q0 + qq) * TABW;
      const double* xs = s_x[wib][ge];
      double F[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
      for (int bb = 0; bb < NEN / 2; ++bb) {
        const int b = hf * (NEN / 2) + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xi = xs[3 * b + i];
          F[3 * i] = fma(xi, n0, F[3 * i]);
          F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
          F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        }
      }
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const double o = __shfl_xor_sync(0xffffffffu, F[r], 1);
        F[r] = hf ? o + F[r] : F[r] + o;
      }
      double* kq = s_k[wib][ge][qq];
      if (hf == 0) {
        double S[6];
        svk_S(F, mat.lam, mat.mu, S);
#pragma unroll
        for (int r = 0; r < 9; ++r) kq[r] = F[r];
#pragma unroll
        for (int r = 0; r < 6; ++r) kq[9 + r] = S[r];
      } else {
#pragma unroll
        for (int vv = 0; vv < 6; ++vv) {
          int i, k;
          voigt_pair(vv, i, k);
          kq[15 + vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
        }
      }
#pragma unroll
      for (int bb = 0; bb < NEN / 2; ++bb) {
        const int b = hf * (NEN / 2) + bb;
        const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          s_ga[wib][qq][i][ge * GROUP + b] = F[3 * i] * n0 + F[3 * i + 1] * n1 + F[3 * i + 2] * n2;
      }
    }
    __syncwarp();
#pragma unroll 1
    for (int qq = 0; qq < QC; ++qq) {  // ---- phase B
      const double* t = s_tab + (ce * NQ + q0 + qq) * TABW;
      const double* kq = s_k[wib][g][qq];
      const double gN[3] = {t[3 * a], t[3 * a + 1], t[3 * a + 2]};
      const double w = t[3 * NEN];
      double S[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) S[r] = kq[9 + r];
      double tw[3];
#pragma unroll
      for (int I = 0; I < 3; ++I) tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
#pragma unroll
      for (int i = 0; i < 3; ++i)
        fa[i] = fma(kq[3 * i], tw[0], fma(kq[3 * i + 1], tw[1], fma(kq[3 * i + 2], tw[2], fa[i])));
      const double lw = mat.lam * w, mw = mat.mu * w;
      double gl[3], gm[3], gNm[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double gai = s_ga[wib][qq][i][lane];
        gl[i] = lw * gai;
        gm[i] = mw * gai;
        gNm[i] = mw * gN[i];
      }
      double B[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) B[r] = kq[15 + r];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int b = partner<2>(a, 0, j);
        if (b < 0) continue;
        double* Kj = K[j];
        const int lb = gbase + b;
        const double gb[3] = {s_ga[wib][qq][0][lb], s_ga[wib][qq][1][lb], s_ga[wib][qq][2][lb]};
        const double nb[3] = {t[3 * b], t[3 * b + 1], t[3 * b + 2]};
        const double sv = fma(tw[0], nb[0], fma(tw[1], nb[1], tw[2] * nb[2]));
        const double d = fma(gNm[0], nb[0], fma(gNm[1], nb[1], gNm[2] * nb[2]));
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double acc = fma(gl[i], gb[k], fma(gb[i], gm[k], fma(d, B[vidx(i, k)], Kj[3 * i + k])));
            Kj[3 * i + k] = (i == k) ? acc + sv : acc;
          }
      }
    }
    __syncwarp();
  }
  if (valid) {
    double* fo = A.fscr + (int64_t)fd * 3;
    if (TLFEA_CHECK) TL_FCHK(fo);
    fo[0] = fa[0];
    fo[1] = fa[1];
    fo[2] = fa[2];
  }
  constexpr int NLB = 32, NIT = (NLB + 2) / 3;
  const int bi = lane / 9, rr = lane - 9 * (lane / 9);
  if (write) {
    pf_wait();
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const int b = valid ? partner<2>(a, 0, j) : -1;
    int32_t pos = -1;
    if (b >= 0) {
      const double* Kj = K[j];
      const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
      bool tr = a > b;
      pos = (int32_t)(e * NUB + ub);
      if (dest) {
        const int32_t dd = s_dst[wib][g * NUB + ub];
        pos = dd >> 1;
        tr = tr != ((dd & 1) != 0);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) s_part[wib][tr ? 3 * k + i : 3 * i + k][lane] = Kj[3 * i + k];
    }
    s_pos[wib][lane] = pos;
    __syncwarp();
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int blk = 3 * it + bi;
      if (lane < 27 && blk < NLB) {
        const int32_t p = s_pos[wib][blk];
        if (p >= 0) k_store(Kscr + (int64_t)p * 9 + rr, s_part[wib][rr][blk]);
      }
    }
    __syncwarp();
  }
}

#ifndef TLFEA_MR_MINB
#define TLFEA_MR_MINB 2  // config 2: 0.509 ms at 2 CTAs/SM (248 registers); 3 CTAs spill 380 B, 0.575 ms
#endif
#ifndef TLFEA_MR_2PH
#define TLFEA_MR_2PH 1  // T10 Mooney-Rivlin (+KV) class-mode tangent eval through element_group_t10mr
#endif
#ifndef TLFEA_BEAM_2PH
#define TLFEA_BEAM_2PH 1  // ANCF3243 SVK class-mode tangent eval through element_group_beam_svk
#endif
#ifndef TLFEA_BEAM_MINB
#define TLFEA_BEAM_MINB 3  // config 6: 1.19 ms (168 registers, 20 B spill) vs 1.24 at 2 CTAs, 1.40 lane-per-node
#endif
#ifndef TLFEA_ANCF_2PH
#define TLFEA_ANCF_2PH 1  // ANCF3443 SVK class-mode tangent eval through element_group_ancf_svk
#endif
#ifndef TLFEA_T10_2PH
#define TLFEA_T10_2PH 1  // T10 SVK class-mode tangent eval through element_group_t10svk
#endif

#ifndef TLFEA_T10_FMINB
#define TLFEA_T10_FMINB 6  // T10 SVK force-only (two-phase) CTAs per SM: 80 registers, no spills (config 5: 0.674 ms vs 0.784 at 4, 0.676 at 8)
#endif
template <int ELEM, int MODEL, int NPASS, bool KV, bool TAN, bool CLS>
__host__ __device__ constexpr int el_minb_k() {
  return (ELEM == 0 && MODEL == 0 && !KV && !TAN)                         ? TLFEA_T10_FMINB
         : (TLFEA_T10_2PH && ELEM == 0 && MODEL == 0 && TAN && (CLS || !KV)) ? TLFEA_T10_2PH_MINB
         : (TLFEA_ANCF_2PH && ELEM == 1 && MODEL == 0 && !KV && TAN && CLS) ? TLFEA_ANCF_MINB
         : (TLFEA_BEAM_2PH && ELEM == 2 && MODEL == 0 && !KV && TAN && CLS) ? TLFEA_BEAM_MINB
         : (TLFEA_MR_2PH && ELEM == 0 && MODEL == 1 && TAN)                 ? TLFEA_MR_MINB
                                                                            : el_minb<ELEM, MODEL, NPASS>();
}

// AFF: table mode with the tables generated from the affine (min) layout.
// JNV: table mode with the tables generated from the per-(e,q) J^-1 layout (curved T10).
template <int ELEM, int NQ, int MODEL, bool KV, bool TAN, bool CLS, int NPASS, bool AFF = false, bool JNV = false>
__global__ void __launch_bounds__(kWarps * 32, el_minb_k<ELEM, MODEL, NPASS, KV, TAN, CLS>()) k_element(ElArgs A) {
  extern __shared__ double s_tab[];  // CLS: [n_cls][NQ][3 NEN + 1]
  // (SVK in table mode measured slower two-phase: config 3 without classes 13.97 vs 12.61 ms, force only
  // 1.20 vs 1.11 ms — staging the per-(e,q) tables serializes the group start; MR gains: 0.59 vs 0.71 ms)
  constexpr bool T2PH = TLFEA_T10_2PH && ELEM == 0 && MODEL == 0 && !KV;  // tangent or force only
  constexpr bool A2PH = TLFEA_ANCF_2PH && ELEM == 1 && MODEL == 0 && !KV && TAN && CLS;
  constexpr bool B2PH = TLFEA_BEAM_2PH && ELEM == 2 && MODEL == 0 && !KV && TAN && CLS;
  constexpr bool M2PH = TLFEA_MR_2PH && ELEM == 0 && MODEL == 1 && TAN;
  constexpr bool V2PH = TLFEA_T10_2PH && ELEM == 0 && MODEL == 0 && KV && TAN && CLS;  // SVK + Kelvin-Voigt
  const int64_t grp = A.g0 + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);  // this warp's element group
  T10Pre pre;
  if constexpr (T2PH && !CLS && !AFF && !JNV) t10_stage_tables_async<NQ>(grp, A, s_tab);
  T10Aff aff;
  if constexpr (T2PH && AFF) t10_affine_load<NQ>(grp, A, aff);
  if constexpr (T2PH && JNV) t10_jinv_load<NQ>(grp, A, aff);
  if constexpr (T2PH) t10_preload<CLS>(grp, A, pre);
  if constexpr (T2PH && AFF) t10_affine_expand<NQ>(aff, s_tab);
  if constexpr (T2PH && JNV) t10_affine_expand<NQ, true>(aff, s_tab);
  if (CLS) {
    // all loads of a thread in flight at once (one L2 round trip, not one per element)
    const int tot = A.n_cls * NQ * (Geo<ELEM>::NEN * 3 + 1);
    constexpr int U = 8;
    for (int t = threadIdx.x; t < tot; t += U * blockDim.x) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = t + u * (int)blockDim.x < tot ? A.cls_tab[t + u * blockDim.x] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t + u * (int)blockDim.x < tot) s_tab[t + u * blockDim.x] = v[u];
    }
    __syncthreads();
  }
  if constexpr (T2PH) {
    if constexpr (!CLS) pre.ce = (threadIdx.x >> 5) * 3 + (threadIdx.x & 31) / 10;  // staged slot
    // (affine tables are written synchronously: no cp.async wait before phase A)
    if constexpr (TAN)
      element_group_t10svk<NQ, false, !CLS && !AFF && !JNV>(grp, A, s_tab, pre);
    else
      element_group_t10svk_force<NQ, !CLS && !AFF && !JNV>(grp, A, s_tab, pre);
  } else if constexpr (A2PH) {
    element_group_ancf_svk<NQ>(grp, A, s_tab);
  } else if constexpr (B2PH) {
    element_group_beam_svk<NQ>(grp, A, s_tab);
  } else if constexpr (V2PH) {
    T10Pre pv;
    t10_preload<CLS>(grp, A, pv);
    element_group_t10svk<NQ, true>(grp, A, s_tab, pv);
  } else if constexpr (M2PH) {
    if constexpr (!CLS && AFF)
      t10_stage_affine<NQ>(grp, A, s_tab);
    else if constexpr (!CLS && JNV)
      t10_stage_jinv<NQ>(grp, A, s_tab);
    else if constexpr (!CLS)
      t10_stage_tables<NQ>(grp, A, s_tab);
    element_group_t10mr<NQ, KV>(grp, A, s_tab, !CLS);
  } else
    element_group<ELEM, NQ, MODEL, KV, TAN, CLS, NPASS, TLFEA_DEST_ASYNC != 0>(grp, A, s_tab);
}


// ------------------------------------------------- consistent KV tangent
// SURVEY §8(f) NEXT-4 (options.kv_consistent_tangent): H = dg/dv of the
// velocity residual (Eq. residual, x = q_n + h v, reading Q9) with
// Kelvin-Voigt damping, H = M/h + h (K^el + K^vx + K^vv / h), where per
// quadrature point (w = J0 w_q, g = F grad N, gd = Fdot grad N, d_ab =
// grad N_a . grad N_b, s^v_ab = grad N_a . S_v grad N_b):
//   K^vv_ab = w (eta g_b g_a^T + eta d_ab F F^T + lam_d g_a g_b^T)   (dP_v/dFdot)
//   K^vx_ab = w (s^v_ab I + eta d_ab F Fdot^T + eta g_b gd_a^T + lam_d g_a gd_b^T)
// (dP_v/dF at fixed Fdot; DESIGN.md §9a derives both). K^vv and K^el are
// symmetric, K^vx is not, so every element pair (a, b), a <= b, yields two
// blocks: lane a accumulates KA = K_ab and KB = K_ba for each of its partners.
// The gather-sorted scratch slot of an element upper block holds 18 values:
// the contribution to the unit's H(I,J) then to H(J,I), each in its own
// orientation (no transposes). One lane per element node as in element_group
// (T10: 3 elements per warp, ANCF3443: 2 lanes per node, beam: 4 elements per
// warp); three block passes keep the 2 x 9 accumulators per partner in
// registers. A variant path: it is not tuned like the symmetric kernels.
template <int ELEM, int NQ, int MODEL, bool CLS>
__device__ __forceinline__ void element_group_kvc(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab) {
  using G = Geo<ELEM>;
  constexpr int NEN = G::NEN, GROUP = G::GROUP, EPW = G::EPW, NUB = G::NUB, NB = G::NB;
  constexpr int TABW = NEN * 3 + 1;
  constexpr int NPASS = 3, NBP = (NB + NPASS - 1) / NPASS;
  constexpr bool MULTI = ELEM != 1;
  __shared__ double s_part[kWarps][18][kLD];
  __shared__ double s_F[kWarps][EPW][18];
  __shared__ double s_node[kWarps][9][kLD];  // g, gd, grad N per lane
  __shared__ double s_C[kWarps][EPW][MODEL == 1 ? 36 : 1];
  __shared__ int32_t s_pos[kWarps][32];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = MULTI ? (lane < EPW * GROUP) : true;
  const int g = (MULTI && lane_active) ? lane / GROUP : 0;
  const int a = MULTI ? (lane_active ? lane % GROUP : 0) : (lane & 15);
  const int half = MULTI ? 0 : (lane >> 4);
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < n_el;
  const int gbase = g * GROUP;
  const double ih = A.inv_h;

  double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
  int ce = 0;
  if (valid) {
    const int64_t I = A.conn[e * NEN + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      xa[i] = A.x[3 * I + i];
      va[i] = A.v[3 * I + i];
    }
    if (CLS) ce = A.cls[e];
  }
  double fa[3] = {0, 0, 0};
  double KA[NBP][9], KB[NBP][9];
#pragma unroll 1
  for (int pass = 0; pass < NPASS; ++pass) {
#pragma unroll
    for (int j = 0; j < NBP; ++j)
#pragma unroll
      for (int r = 0; r < 9; ++r) KA[j][r] = KB[j][r] = 0.0;
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
      double gN[3] = {0, 0, 0}, w = 0.0;
      if (valid) {
        if (CLS) {
          const double* t = s_tab + (ce * NQ + q) * TABW;
          gN[0] = t[3 * a];
          gN[1] = t[3 * a + 1];
          gN[2] = t[3 * a + 2];
          w = t[3 * NEN];
        } else {
          const double* src = A.gradN + ((e * NQ + q) * NEN + a) * 3;
          gN[0] = src[0];
          gN[1] = src[1];
          gN[2] = src[2];
          w = A.J0w[e * NQ + q];
        }
      }
      // F, Fdot = sum_a (x_a, v_a) (x) grad N_a over the element's lanes
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int J = 0; J < 3; ++J) {
          s_part[wib][3 * i + J][lane] = xa[i] * gN[J];
          s_part[wib][9 + 3 * i + J][lane] = va[i] * gN[J];
        }
      __syncwarp();
      if (MULTI) {
        if (lane_active) {
          for (int comp = a; comp < 18; comp += GROUP) {
            const double* p = &s_part[wib][comp][gbase];
            double sum = 0.0;
#pragma unroll
            for (int b = 0; b < NEN; ++b) sum += p[b];
            s_F[wib][g][comp] = sum;
          }
        }
      } else {
        const int comp = lane & 15;
        if (comp < 9) {
          const double* p = &s_part[wib][9 * half + comp][0];
          double sum = 0.0;
#pragma unroll
          for (int b = 0; b < 16; ++b) sum += p[b];
          s_F[wib][0][9 * half + comp] = sum;
        }
      }
      __syncwarp();
      double F[9], Fd[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        F[r] = s_F[wib][g][r];
        Fd[r] = s_F[wib][g][9 + r];
      }
      double S[6], Sv[6];
      MRState ms;
      if (MODEL == 0) {
        svk_S(F, mat.lam, mat.mu, S);
      } else {
        mr_state(F, ms);
        if (valid && !(ms.J > 0.0) && a == 0 && half == 0) atomicMin(A.err, (unsigned long long)(e * 64 + q));
        mr_S(ms, mat.C10, mat.C01, mat.kappa, S);
      }
      kv_S(F, Fd, mat.eta, mat.lamd, Sv);
      double tw[3], twv[3];  // w S grad N_a, w S_v grad N_a
#pragma unroll
      for (int I = 0; I < 3; ++I) {
        tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
        twv[I] = w * (sget(Sv, I, 0) * gN[0] + sget(Sv, I, 1) * gN[1] + sget(Sv, I, 2) * gN[2]);
      }
      if (pass == 0) {  // f_a += F (w (S + S_v) grad N_a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
          fa[i] = fma(F[3 * i], tw[0] + twv[0], fma(F[3 * i + 1], tw[1] + twv[1], fma(F[3 * i + 2], tw[2] + twv[2], fa[i])));
      }
      double ga[3], gda[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        ga[i] = F[3 * i] * gN[0] + F[3 * i + 1] * gN[1] + F[3 * i + 2] * gN[2];
        gda[i] = Fd[3 * i] * gN[0] + Fd[3 * i + 1] * gN[1] + Fd[3 * i + 2] * gN[2];
      }
      double B[6], Cd[9];  // F F^T (Voigt), F Fdot^T
#pragma unroll
      for (int vv = 0; vv < 6; ++vv) {
        int i, k;
        voigt_pair(vv, i, k);
        B[vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) Cd[3 * i + k] = F[3 * i] * Fd[3 * k] + F[3 * i + 1] * Fd[3 * k + 1] + F[3 * i + 2] * Fd[3 * k + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        s_node[wib][i][lane] = ga[i];
        s_node[wib][3 + i][lane] = gda[i];
        s_node[wib][6 + i][lane] = gN[i];
      }
      double CB[MODEL == 1 ? 6 : 1][3];
      if (MODEL == 1) {
        if (lane_active && (MULTI || half == 0)) {
          const int col = MULTI ? a : lane;
          if (col < 6) {
            double cc[6];
            mr_Cv_column_dispatch(ms, mat.C10, mat.C01, mat.kappa, col, cc);
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) s_C[wib][g][6 * vv + col] = w * cc[vv];
          }
        }
      }
      __syncwarp();
      if constexpr (MODEL == 1) {
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
          for (int i = 0; i < 3; ++i) {
            double sacc = 0.0;
#pragma unroll
            for (int ww = 0; ww < 6; ++ww) sacc = fma(s_C[wib][g][6 * vv + ww], Ba[ww][i], sacc);
            CB[vv][i] = sacc;
          }
      }
      // symmetric part coefficients: SVK folds K^vv / h into the Lame pair
      const double lwe = MODEL == 0 ? w * (mat.lam + mat.lamd * ih) : w * mat.lamd * ih;
      const double mwe = MODEL == 0 ? w * (mat.mu + mat.eta * ih) : w * mat.eta * ih;
      const double ew = w * mat.eta, ldw = w * mat.lamd;
#pragma unroll
      for (int jj = 0; jj < NBP; ++jj) {
        const int j = pass * NBP + jj;
        const int b = j < NB ? partner<ELEM>(a, half, j) : -1;
        if (b < 0) continue;
        const int lb = gbase + b;
        double gb[3], gdb[3], nb[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          gb[i] = s_node[wib][i][lb];
          gdb[i] = s_node[wib][3 + i][lb];
          nb[i] = s_node[wib][6 + i][lb];
        }
        const double s = tw[0] * nb[0] + tw[1] * nb[1] + tw[2] * nb[2];
        const double sv = twv[0] * nb[0] + twv[1] * nb[1] + twv[2] * nb[2];
        const double dd = gN[0] * nb[0] + gN[1] * nb[1] + gN[2] * nb[2];
        double E[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k)
            E[3 * i + k] = lwe * ga[i] * gb[k] + mwe * gb[i] * ga[k] + mwe * dd * B[vidx(i, k)] + (i == k ? s : 0.0);
        if constexpr (MODEL == 1) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double bb[6];
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) {
              int I, J;
              voigt_pair(vv, I, J);
              bb[vv] = (I == J) ? F[3 * k + I] * nb[I] : F[3 * k + I] * nb[J] + F[3 * k + J] * nb[I];
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double acc = 0.0;
#pragma unroll
              for (int vv = 0; vv < 6; ++vv) acc = fma(CB[vv][i], bb[vv], acc);
              E[3 * i + k] += acc;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double c = ew * dd * Cd[3 * i + k] + (i == k ? sv : 0.0);
            KA[jj][3 * i + k] += E[3 * i + k] + c + ew * gb[i] * gda[k] + ldw * ga[i] * gdb[k];
            KB[jj][3 * i + k] += E[3 * k + i] + c + ew * ga[i] * gdb[k] + ldw * gb[i] * gda[k];
          }
      }
      __syncwarp();
    }
    if (valid && pass == 0 && (MULTI || half == 0)) {
      const int64_t fp = A.fdest ? (int64_t)A.fdest[e * NEN + a] : e * NEN + a;
      double* fo = A.fscr + fp * 3;
      if (TLFEA_CHECK) TL_FCHK(fo);
      fo[0] = fa[0];
      fo[1] = fa[1];
      fo[2] = fa[2];
    }
    // blocks -> 18-value scratch slots: [H(I,J) part | H(J,I) part]
    constexpr int NLB = MULTI ? EPW * GROUP : 32;
    constexpr int NIT = (NLB + 2) / 3;
    const int bi = lane / 9, rr = lane - 9 * (lane / 9);
#pragma unroll
    for (int jj = 0; jj < NBP; ++jj) {
      const int j = pass * NBP + jj;
      const int b = (valid && j < NB) ? partner<ELEM>(a, half, j) : -1;
      int32_t pos = -1;
      bool flip = false;
      if (b >= 0) {
        const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
        const int32_t d = A.dest[e * NUB + ub];
        pos = d >> 1;
        // KA = K_ab; the unit's (I,J) block is K_{lo,hi} unless the dest bit flips it
        flip = a != b && ((a > b) != ((d & 1) != 0));
      }
      s_pos[wib][lane] = pos;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        if (b >= 0) {
#pragma unroll
          for (int r = 0; r < 9; ++r) s_part[wib][r][lane] = (flip != (part == 1)) ? KB[jj][r] : KA[jj][r];
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          const int blk = 3 * it + bi;
          if (lane < 27 && blk < NLB) {
            const int32_t p = s_pos[wib][blk];
            if (p >= 0) k_store(A.Kscr + (int64_t)p * 18 + 9 * part + rr, s_part[wib][rr][blk]);
          }
        }
        __syncwarp();
      }
    }
  }
}


// T10 two-phase consistent-KV tangent (SVK or MR). Phase A, two lanes per
// (element, q): F and Fdot over 5 nodes each plus one shuffle, then S (the
// elastic stress), S_v (reading Q7) and, for Mooney-Rivlin, the w-scaled 6x6
// Voigt tangent (3 columns per lane), once per (element, q) into shared
// memory. Phase B, one lane per (element, node a), in T10KVC_NPASS passes over
// its partners: g, gd of both nodes from F, Fdot and the gradients, the
// elastic block plus K^vv / h and K^vx for K_ab and K_ba (as element_group_kvc)
// and f_a. The lane-per-node kernel (element_group_kvc) recomputed the F
// reduction, the MR state and the MR tangent on every lane in every pass.
#ifndef TLFEA_T10KVC_2PH
#define TLFEA_T10KVC_2PH 1
#endif
#ifndef TLFEA_T10KVC_NPASS
#define TLFEA_T10KVC_NPASS 3
#endif
template <int NQ, int MODEL>
__device__ __forceinline__ void element_group_t10kvc(int64_t grp, const ElArgs& A, const double* __restrict__ s_tab,
                                                     bool table_mode) {
  constexpr int NEN = 10, GROUP = 10, EPW = 3, NUB = 55, NB = 6, TABW = 3 * NEN + 1;
  constexpr int KQ = MODEL == 1 ? 51 : 30;  // F (9), Fd (9), S (6), S_v (6) [, w C (21, upper Voigt)]
  constexpr int NPASS = TLFEA_T10KVC_NPASS, NBP = (NB + NPASS - 1) / NPASS;
  static_assert(EPW * NQ * 2 <= 32, "phase A: two lanes per (element, q)");
  __shared__ double s_k[kWarps][EPW][NQ][KQ];
  __shared__ double s_x[kWarps][EPW][3 * NEN];
  __shared__ double s_v[kWarps][EPW][3 * NEN];
  __shared__ double s_st[kWarps][9][kLD];  // store staging
  __shared__ int32_t s_pos[kWarps][32];
  __shared__ int32_t s_cls[kWarps][EPW];
  const int64_t n_el = A.n_el;
  const MatDev& mat = A.mat;
  const double ih = A.inv_h;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool lane_active = lane < EPW * GROUP;
  const int g = lane_active ? lane / GROUP : 0;
  const int a = lane_active ? lane % GROUP : 0;
  const int64_t e = grp * EPW + g;
  const bool valid = lane_active && e < n_el;
  int32_t fd = 0;
  if (lane_active) {
    double xa[3] = {0, 0, 0}, va[3] = {0, 0, 0};
    int ce = 0;
    if (valid) {
      fd = A.fdest ? A.fdest[e * NEN + a] : (int32_t)(e * NEN + a);
      const int64_t I = A.conn[e * NEN + a];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xa[i] = A.x[3 * I + i];
        va[i] = A.v[3 * I + i];
      }
      if (!table_mode && a == 0) ce = A.cls[e];
    }
    if (table_mode) ce = wib * EPW + g;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      s_x[wib][g][3 * a + i] = xa[i];
      s_v[wib][g][3 * a + i] = va[i];
    }
    if (a == 0) s_cls[wib][g] = ce;
  }
  __syncwarp();
  {  // ---- phase A
    const bool act = lane < EPW * NQ * 2;
    const int pr = act ? lane >> 1 : 0, hf = lane & 1;
    const int ge = pr / NQ, q = pr - NQ * (pr / NQ);
    const double* t = s_tab + (s_cls[wib][ge] * NQ + q) * TABW;
    double F[9], Fd[9];
#pragma unroll
    for (int r = 0; r < 9; ++r) F[r] = Fd[r] = 0.0;
#pragma unroll
    for (int bb = 0; bb < NEN / 2; ++bb) {
      const int b = hf * (NEN / 2) + bb;
      const double n0 = t[3 * b], n1 = t[3 * b + 1], n2 = t[3 * b + 2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double xi = s_x[wib][ge][3 * b + i], vi = s_v[wib][ge][3 * b + i];
        F[3 * i] = fma(xi, n0, F[3 * i]);
        F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
        F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        Fd[3 * i] = fma(vi, n0, Fd[3 * i]);
        Fd[3 * i + 1] = fma(vi, n1, Fd[3 * i + 1]);
        Fd[3 * i + 2] = fma(vi, n2, Fd[3 * i + 2]);
      }
    }
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const double o = __shfl_xor_sync(0xffffffffu, F[r], 1), od = __shfl_xor_sync(0xffffffffu, Fd[r], 1);
      F[r] = hf ? o + F[r] : F[r] + o;
      Fd[r] = hf ? od + Fd[r] : Fd[r] + od;
    }
    const double w = t[3 * NEN];
    MRState ms;
    if (MODEL == 1) mr_state(F, ms);
    if (act) {
      double* kq = s_k[wib][ge][q];
      if (hf == 0) {
        double S[6], Sv[6];
        if (MODEL == 0) {
          svk_S(F, mat.lam, mat.mu, S);
        } else {
          if (grp * EPW + ge < n_el && !(ms.J > 0.0)) atomicMin(A.err, (unsigned long long)((grp * EPW + ge) * 64 + q));
          mr_S(ms, mat.C10, mat.C01, mat.kappa, S);
        }
        kv_S(F, Fd, mat.eta, mat.lamd, Sv);
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          kq[r] = F[r];
          kq[9 + r] = Fd[r];
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          kq[18 + r] = S[r];
          kq[24 + r] = Sv[r];
        }
      }
      if constexpr (MODEL == 1) {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          const int col = 3 * hf + cc;
          double cv[6];
          mr_Cv_column_dispatch(ms, mat.C10, mat.C01, mat.kappa, col, cv);
#pragma unroll
          for (int vv = 0; vv < 6; ++vv)
            if (vv <= col) kq[30 + cs_idx(vv, col)] = w * cv[vv];
        }
      }
    }
  }
  __syncwarp();
  // ---- phase B
  const int ce = s_cls[wib][g];
  double fa[3] = {0, 0, 0};
  const double lwe = MODEL == 0 ? mat.lam + mat.lamd * ih : mat.lamd * ih;  // x w below
  const double mwe = MODEL == 0 ? mat.mu + mat.eta * ih : mat.eta * ih;
#pragma unroll 1
  for (int pass = 0; pass < NPASS; ++pass) {
    double KA[NBP][9], KB[NBP][9];
#pragma unroll
    for (int j = 0; j < NBP; ++j)
#pragma unroll
      for (int r = 0; r < 9; ++r) KA[j][r] = KB[j][r] = 0.0;
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
      const double* t = s_tab + (ce * NQ + q) * TABW;
      const double* kq = s_k[wib][g][q];
      const double gN[3] = {t[3 * a], t[3 * a + 1], t[3 * a + 2]};
      const double w = t[3 * NEN];
      double F[9], Fd[9], S[6], Sv[6];
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        F[r] = kq[r];
        Fd[r] = kq[9 + r];
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        S[r] = kq[18 + r];
        Sv[r] = kq[24 + r];
      }
      double tw[3], twv[3], ga[3], gda[3];
#pragma unroll
      for (int I = 0; I < 3; ++I) {
        tw[I] = w * (sget(S, I, 0) * gN[0] + sget(S, I, 1) * gN[1] + sget(S, I, 2) * gN[2]);
        twv[I] = w * (sget(Sv, I, 0) * gN[0] + sget(Sv, I, 1) * gN[1] + sget(Sv, I, 2) * gN[2]);
        ga[I] = F[3 * I] * gN[0] + F[3 * I + 1] * gN[1] + F[3 * I + 2] * gN[2];
        gda[I] = Fd[3 * I] * gN[0] + Fd[3 * I + 1] * gN[1] + Fd[3 * I + 2] * gN[2];
      }
      if (pass == 0) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
          fa[i] = fma(F[3 * i], tw[0] + twv[0], fma(F[3 * i + 1], tw[1] + twv[1], fma(F[3 * i + 2], tw[2] + twv[2], fa[i])));
      }
      double B[6], Cd[9];  // F F^T (Voigt), F Fdot^T
#pragma unroll
      for (int vv = 0; vv < 6; ++vv) {
        int i, k;
        voigt_pair(vv, i, k);
        B[vv] = F[3 * i] * F[3 * k] + F[3 * i + 1] * F[3 * k + 1] + F[3 * i + 2] * F[3 * k + 2];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
          Cd[3 * i + k] = F[3 * i] * Fd[3 * k] + F[3 * i + 1] * Fd[3 * k + 1] + F[3 * i + 2] * Fd[3 * k + 2];
      double CB[MODEL == 1 ? 6 : 1][3];
      if constexpr (MODEL == 1) {
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
          for (int i = 0; i < 3; ++i) {
            double sacc = 0.0;
#pragma unroll
            for (int ww = 0; ww < 6; ++ww)
              sacc = fma(kq[30 + (vv <= ww ? cs_idx(vv, ww) : cs_idx(ww, vv))], Ba[ww][i], sacc);
            CB[vv][i] = sacc;
          }
      }
      const double lw = lwe * w, mw = mwe * w, ew = w * mat.eta, ldw = w * mat.lamd;
#pragma unroll
      for (int jj = 0; jj < NBP; ++jj) {
        const int j = pass * NBP + jj;
        const int b = j < NB ? partner<0>(a, 0, j) : -1;
        if (b < 0) continue;
        const double nb[3] = {t[3 * b], t[3 * b + 1], t[3 * b + 2]};
        double gb[3], gdb[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          gb[i] = F[3 * i] * nb[0] + F[3 * i + 1] * nb[1] + F[3 * i + 2] * nb[2];
          gdb[i] = Fd[3 * i] * nb[0] + Fd[3 * i + 1] * nb[1] + Fd[3 * i + 2] * nb[2];
        }
        const double sab = tw[0] * nb[0] + tw[1] * nb[1] + tw[2] * nb[2];
        const double sv = twv[0] * nb[0] + twv[1] * nb[1] + twv[2] * nb[2];
        const double dd = gN[0] * nb[0] + gN[1] * nb[1] + gN[2] * nb[2];
        double E[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k)
            E[3 * i + k] = lw * ga[i] * gb[k] + mw * gb[i] * ga[k] + mw * dd * B[vidx(i, k)] + (i == k ? sab : 0.0);
        if constexpr (MODEL == 1) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            double bb[6];
#pragma unroll
            for (int vv = 0; vv < 6; ++vv) {
              int I, J;
              voigt_pair(vv, I, J);
              bb[vv] = (I == J) ? F[3 * k + I] * nb[I] : F[3 * k + I] * nb[J] + F[3 * k + J] * nb[I];
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double acc = 0.0;
#pragma unroll
              for (int vv = 0; vv < 6; ++vv) acc = fma(CB[vv][i], bb[vv], acc);
              E[3 * i + k] += acc;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double c = ew * dd * Cd[3 * i + k] + (i == k ? sv : 0.0);
            KA[jj][3 * i + k] += E[3 * i + k] + c + ew * gb[i] * gda[k] + ldw * ga[i] * gdb[k];
            KB[jj][3 * i + k] += E[3 * k + i] + c + ew * ga[i] * gdb[k] + ldw * gb[i] * gda[k];
          }
      }
    }
    if (valid && pass == 0) {
      double* fo = A.fscr + (int64_t)fd * 3;
      if (TLFEA_CHECK) TL_FCHK(fo);
      fo[0] = fa[0];
      fo[1] = fa[1];
      fo[2] = fa[2];
    }
    // blocks -> 18-value scratch slots: [H(I,J) part | H(J,I) part]
    constexpr int NLB = EPW * GROUP, NIT = (NLB + 2) / 3;
    const int bi = lane / 9, rr = lane - 9 * (lane / 9);
#pragma unroll
    for (int jj = 0; jj < NBP; ++jj) {
      const int j = pass * NBP + jj;
      const int b = (valid && j < NB) ? partner<0>(a, 0, j) : -1;
      int32_t pos = -1;
      bool flip = false;
      if (b >= 0) {
        const int ub = a <= b ? ublk(NEN, a, b) : ublk(NEN, b, a);
        const int32_t d = A.dest[e * NUB + ub];
        pos = d >> 1;
        flip = a != b && ((a > b) != ((d & 1) != 0));
      }
      s_pos[wib][lane] = pos;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        if (b >= 0) {
#pragma unroll
          for (int r = 0; r < 9; ++r) s_st[wib][r][lane] = (flip != (part == 1)) ? KB[jj][r] : KA[jj][r];
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          const int blk = 3 * it + bi;
          if (lane < 27 && blk < NLB) {
            const int32_t p = s_pos[wib][blk];
            if (p >= 0) k_store(A.Kscr + (int64_t)p * 18 + 9 * part + rr, s_st[wib][rr][blk]);
          }
        }
        __syncwarp();
      }
    }
  }
}

template <int NQ, int MODEL, bool CLS, bool AFF>
__global__ void __launch_bounds__(kWarps * 32, 2) k_element_t10kvc(ElArgs A) {
  extern __shared__ double s_tab[];  // CLS: [n_cls][NQ][31]; else the warp's staged tables
  const int64_t grp = A.g0 + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if constexpr (CLS) {
    const int tot = A.n_cls * NQ * 31;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) s_tab[t] = A.cls_tab[t];
    __syncthreads();
  } else if constexpr (AFF) {
    t10_stage_affine<NQ>(grp, A, s_tab);
  } else {
    t10_stage_tables<NQ>(grp, A, s_tab);
  }
  element_group_t10kvc<NQ, MODEL>(grp, A, s_tab, !CLS);
}

template <int ELEM, int NQ, int MODEL, bool CLS>
__global__ void __launch_bounds__(kWarps * 32, 2) k_element_kvc(ElArgs A) {
  extern __shared__ double s_tab[];  // CLS: [n_cls][NQ][3 NEN + 1]
  if (CLS) {
    const int tot = A.n_cls * NQ * (Geo<ELEM>::NEN * 3 + 1);
    for (int t = threadIdx.x; t < tot; t += blockDim.x) s_tab[t] = A.cls_tab[t];
    __syncthreads();
  }
  const int64_t grp = A.g0 + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  element_group_kvc<ELEM, NQ, MODEL, CLS>(grp, A, s_tab);
}


// ------------------------------------------------------------------ gather

// v3: TMA bulk copies (cp.async.bulk global->shared, mbarrier completion),
// double-buffered per warp: one elected lane moves the next window of the
// contiguous scratch range while the warp sums the current one.
constexpr int kG3Warps = 4;  // H gather warps per CTA (the fused kernel needs kElWarps == 4)
#ifndef TLFEA_G3WB
#define TLFEA_G3WB 64
#endif
constexpr int kG3WB = TLFEA_G3WB;            // blocks per window
constexpr int kG3Buf = kG3WB * 9 + 2;        // doubles per buffer (+16 B alignment slack)

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}

struct GatherArgs {
  int64_t n_units;
  const int32_t* unit_ptr;
  const int32_t* u_off;
  const int32_t* u_offT;
  const int32_t* u_deg;
  const double* u_m;
  const double* Kscr;
  double h;
  double* H;
  int upper;  // UPPER H storage (u_deg = L | diagonal << 16, no transposed copy)
};

// Per-warp TMA staging: two windows and their mbarriers. `wk` counts the
// windows this warp has consumed so far (buffer wk & 1, phase (wk >> 1) & 1),
// so the barriers can be reused across work items of a persistent kernel.
struct G3Warp {
  double* buf[2];
  uint64_t* bar;
  uint32_t wk;
};

// The 32 consecutive units u0 .. u0+31 on one warp.
__device__ __forceinline__ void gather_units_warp(int64_t u0, const GatherArgs& A, G3Warp& W) {
  const int lane = threadIdx.x & 31;
  const int64_t n_units = A.n_units;
  const int32_t* __restrict__ unit_ptr = A.unit_ptr;
  const double* __restrict__ Kscr = A.Kscr;
  const double h = A.h;
  double* __restrict__ H = A.H;
  if (u0 >= n_units) return;
  const int64_t u = u0 + lane;
  const bool valid = u < n_units;
  const int64_t uend = min(u0 + 32, n_units);
  const int64_t P0 = unit_ptr[u0], P1 = unit_ptr[uend];
  int32_t my0 = 0, my1 = 0, off = 0, offT = -1, dg = 0;
  double m = 0.0;
  if (valid) {
    my0 = unit_ptr[u];
    my1 = unit_ptr[u + 1];
    off = A.u_off[u];
    offT = A.u_offT[u];
    dg = A.u_deg[u];
    m = A.u_m[u];
  }
  const int nwin = (int)((P1 - P0 + kG3WB - 1) / kG3WB);
  const uint32_t wk0 = W.wk;
  auto issue = [&](int k) {
    const int64_t w0 = P0 + (int64_t)k * kG3WB, w1 = min(w0 + (int64_t)kG3WB, P1);
    const uintptr_t a = (uintptr_t)(Kscr + w0 * 9) & ~(uintptr_t)15;
    const uintptr_t b = ((uintptr_t)(Kscr + w1 * 9) + 15) & ~(uintptr_t)15;
    const uint32_t wi = wk0 + k;
    if (TLFEA_CHECK) {
      tl_chk(Kscr + w0 * 9, 0, __LINE__);
      tl_chk(Kscr + w1 * 9 - 1, 0, __LINE__);
    }
    bulk_load(W.buf[wi & 1], (const void*)a, (unsigned)(b - a), &W.bar[wi & 1]);
  };
  if (lane == 0 && nwin > 0) issue(0);
  double acc[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) acc[r] = 0.0;
  for (int k = 0; k < nwin; ++k) {
    if (lane == 0 && k + 1 < nwin) issue(k + 1);
    const uint32_t wi = wk0 + k;
    mbar_wait(&W.bar[wi & 1], (wi >> 1) & 1);
    const int64_t w0 = P0 + (int64_t)k * kG3WB, w1 = min(w0 + (int64_t)kG3WB, P1);
    const int delta = (int)(((uintptr_t)(Kscr + w0 * 9) & 15) >> 3);  // 0 or 1 double
    const double* buf = W.buf[wi & 1] + delta;
    const int64_t a0 = max((int64_t)my0, w0), a1 = min((int64_t)my1, w1);
    for (int64_t t = a0; t < a1; ++t) {
      const double* sb = buf + (t - w0) * 9;
#pragma unroll
      for (int r = 0; r < 9; ++r) acc[r] += sb[r];
    }
    __syncwarp();
  }
  W.wk = wk0 + nwin;
  // Warp-cooperative stores: the 32 unit blocks (h K + M/h) are staged in the
  // drained TMA window, then lane t % 32 writes value t = 3 u + f of DOF row d
  // of unit u. Consecutive units of one row I have consecutive block offsets,
  // so a direct store instruction covers 256 contiguous bytes (per-lane 72-byte
  // blocks touched 24 sectors per instruction); the transposed (J,I) blocks keep
  // each unit's 24-byte row piece on three adjacent lanes. Config 3 gather:
  // 7.55 vs 7.98 ms.
  double* st = W.buf[0];
  const double mh = m / h;
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int f = 0; f < 3; ++f) st[lane * 9 + 3 * d + f] = fma(h, acc[3 * d + f], d == f ? mh : 0.0);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int t = 32 * k + lane, sl = t / 3, f = t - 3 * (t / 3);
    const int32_t o = __shfl_sync(0xffffffffu, off, sl), oT = __shfl_sync(0xffffffffu, offT, sl);
    const int32_t dgl = __shfl_sync(0xffffffffu, dg, sl);
    const bool vl = u0 + sl < n_units;
    if (A.upper) {
      // UPPER storage (common.cuh): entry (d, f) at off + f + d (2 + 3 L) - d (d-1)/2,
      // the diagonal block keeps f >= d only; no transposed copy
      const int L = dgl & 0xffff;
      const bool diag = (dgl >> 16) != 0;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (vl && (!diag || f >= d)) {
          if (TLFEA_CHECK) tl_chk(&H[o + f + d * (2 + 3 * L) - d * (d - 1) / 2], 2, __LINE__);
          H[o + f + d * (2 + 3 * L) - d * (d - 1) / 2] = st[sl * 9 + 3 * d + f];
        }
    } else {
      const int dl = dgl & 0xffff, dT = dgl >> 16;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        if (vl) h_store(H + 3 * (int64_t)o + 3 * d * dl + f, st[sl * 9 + 3 * d + f]);
        if (vl && oT >= 0) h_store(H + 3 * (int64_t)oT + 3 * d * dT + f, st[sl * 9 + 3 * f + d]);
      }
    }
  }
}


__device__ __forceinline__ void g3_init(double (*s_buf)[2][kG3Buf], uint64_t (*s_bar)[2], G3Warp& W) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (lane == 0) {
    mbar_init(&s_bar[wib][0], 1);
    mbar_init(&s_bar[wib][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  W.buf[0] = s_buf[wib][0];
  W.buf[1] = s_buf[wib][1];
  W.bar = s_bar[wib];
  W.wk = 0;
}

#ifdef TLFEA_G3_MINB
__global__ void __launch_bounds__(kG3Warps * 32, TLFEA_G3_MINB) k_gather_units_v3(GatherArgs A) {
#else
__global__ void __launch_bounds__(kG3Warps * 32) k_gather_units_v3(GatherArgs A) {
#endif
  __shared__ __align__(16) double s_buf[kG3Warps][2][kG3Buf];
  __shared__ __align__(8) uint64_t s_bar[kG3Warps][2];
  G3Warp W;
  g3_init(s_buf, s_bar, W);
  gather_units_warp(((int64_t)blockIdx.x * kG3Warps + (threadIdx.x >> 5)) * 32, A, W);
}


// Consistent KV tangent gather (NEXT-4): as gather_units_warp, but each
// scratch slot holds 18 values (the unit's H(I,J) part, then its H(J,I) part,
// both in their own orientation) and the two blocks are written untransposed.
constexpr int kG3WB2 = kG3WB / 2;  // 18-value blocks per window (same buffer)
__device__ __forceinline__ void gather_units_warp_kvc(int64_t u0, const GatherArgs& A, G3Warp& W) {
  const int lane = threadIdx.x & 31;
  const int64_t n_units = A.n_units;
  const double* __restrict__ Kscr = A.Kscr;
  double* __restrict__ H = A.H;
  if (u0 >= n_units) return;
  const int64_t u = u0 + lane;
  const bool valid = u < n_units;
  const int64_t uend = min(u0 + 32, n_units);
  const int64_t P0 = A.unit_ptr[u0], P1 = A.unit_ptr[uend];
  int32_t my0 = 0, my1 = 0, off = 0, offT = -1, dg = 0;
  double m = 0.0;
  if (valid) {
    my0 = A.unit_ptr[u];
    my1 = A.unit_ptr[u + 1];
    off = A.u_off[u];
    offT = A.u_offT[u];
    dg = A.u_deg[u];
    m = A.u_m[u];
  }
  const int nwin = (int)((P1 - P0 + kG3WB2 - 1) / kG3WB2);
  const uint32_t wk0 = W.wk;
  auto issue = [&](int k) {
    const int64_t w0 = P0 + (int64_t)k * kG3WB2, w1 = min(w0 + (int64_t)kG3WB2, P1);
    const uint32_t wi = wk0 + k;  // 144-byte slots: always 16-byte aligned
    if (TLFEA_CHECK) {
      tl_chk(Kscr + w0 * 18, 0, __LINE__);
      tl_chk(Kscr + w1 * 18 - 1, 0, __LINE__);
    }
    bulk_load(W.buf[wi & 1], (const void*)(Kscr + w0 * 18), (unsigned)((w1 - w0) * 144), &W.bar[wi & 1]);
  };
  if (lane == 0 && nwin > 0) issue(0);
  double acc[18];
#pragma unroll
  for (int r = 0; r < 18; ++r) acc[r] = 0.0;
  for (int k = 0; k < nwin; ++k) {
    if (lane == 0 && k + 1 < nwin) issue(k + 1);
    const uint32_t wi = wk0 + k;
    mbar_wait(&W.bar[wi & 1], (wi >> 1) & 1);
    const int64_t w0 = P0 + (int64_t)k * kG3WB2, w1 = min(w0 + (int64_t)kG3WB2, P1);
    const double* buf = W.buf[wi & 1];
    const int64_t a0 = max((int64_t)my0, w0), a1 = min((int64_t)my1, w1);
    for (int64_t t = a0; t < a1; ++t) {
      const double* sb = buf + (t - w0) * 18;
#pragma unroll
      for (int r = 0; r < 18; ++r) acc[r] += sb[r];
    }
    __syncwarp();
  }
  W.wk = wk0 + nwin;
  // warp-cooperative stores as in gather_units_warp (18 staged values per unit)
  const double h = A.h, mh = m / h;
  double* st = W.buf[0];
#pragma unroll
  for (int r = 0; r < 18; ++r) st[lane * 18 + r] = fma(h, acc[r], (r % 9) % 4 == 0 ? mh : 0.0);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int t = 32 * k + lane, sl = t / 3, f = t - 3 * (t / 3);
    const int32_t o = __shfl_sync(0xffffffffu, off, sl), oT = __shfl_sync(0xffffffffu, offT, sl);
    const int32_t dgl = __shfl_sync(0xffffffffu, dg, sl);
    const bool vl = u0 + sl < n_units;
    const int dl = dgl & 0xffff, dT = dgl >> 16;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (vl) h_store(H + 3 * (int64_t)o + 3 * d * dl + f, st[sl * 18 + 3 * d + f]);
      if (vl && oT >= 0) h_store(H + 3 * (int64_t)oT + 3 * d * dT + f, st[sl * 18 + 9 + 3 * d + f]);
    }
  }
}

__global__ void __launch_bounds__(kG3Warps * 32) k_gather_units_kvc(GatherArgs A) {
  __shared__ __align__(16) double s_buf[kG3Warps][2][kG3Buf];
  __shared__ __align__(8) uint64_t s_bar[kG3Warps][2];
  G3Warp W;
  g3_init(s_buf, s_bar, W);
  gather_units_warp_kvc(((int64_t)blockIdx.x * kG3Warps + (threadIdx.x >> 5)) * 32, A, W);
}


// ------------------------------------------- small meshes: one launch
// For small T10 SVK meshes with geometry classes (the paper's low ladder
// rungs, BASELINE config 1) the three launches of tlfea_eval are bound by
// kernel boundaries, not by work. k_eval_small runs the same device code in
// one cooperative launch: the class-mode two-phase element groups (grid-
// stride over warp groups), a grid-wide barrier, then the TMA unit gather of
// H and the per-DOF f / g gather (grid-stride). Results are bitwise those of
// the three-kernel path (same arithmetic, same summation orders).
#ifndef TLFEA_SMALL_MAX_EL
#define TLFEA_SMALL_MAX_EL 3000  // ladder: faster up to ~1k elements (RES0-RES4), even at 4.5k, slower at 18k
#endif
template <int NQ>
__global__ void __launch_bounds__(kWarps * 32, TLFEA_T10_2PH_MINB) k_eval_small(ElArgs A, GatherArgs G, FArgs F) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double s_dyn[];  // class tables, then the gather windows + mbarriers
  const int wib = threadIdx.x >> 5;
  {
    const int tot = A.n_cls * NQ * 31;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) s_dyn[t] = A.cls_tab[t];
    __syncthreads();
  }
  const int64_t ngrp = (A.n_el + 2) / 3;
  for (int64_t base = (int64_t)blockIdx.x * kWarps; base < ngrp; base += (int64_t)gridDim.x * kWarps) {
    const int64_t grp = base + wib;
    T10Pre pre;
    t10_preload<true>(grp, A, pre);
    element_group_t10svk<NQ, false, false>(grp, A, s_dyn, pre);
  }
  // the scratch written through the generic proxy is read by TMA (async proxy)
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  cg::this_grid().sync();
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // s_dyn: class tables -> TMA windows
  __syncthreads();
  G3Warp W;
  {
    double* bufs = s_dyn + (size_t)wib * 2 * kG3Buf;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_dyn + (size_t)kWarps * 2 * kG3Buf) + 2 * wib;
    if ((threadIdx.x & 31) == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    W.buf[0] = bufs;
    W.buf[1] = bufs + kG3Buf;
    W.bar = bars;
    W.wk = 0;
  }
  for (int64_t ug = (int64_t)blockIdx.x * kWarps + wib; ug * 32 < G.n_units; ug += (int64_t)gridDim.x * kWarps) {
    gather_units_warp(ug * 32, G, W);
    // the next group's first TMA window lands in the buffer this group's
    // cooperative stores just read through the generic proxy (WAR across proxies)
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 3 * F.n_own;
       t += (int64_t)gridDim.x * blockDim.x)
    gather_f_dof_one(t, F);
}

// ------------------------------------------------------------- launchers

static ElArgs el_args(const Context* c, const double* x, const double* v) {
  ElArgs A;
  A.n_el = c->n_el;
  A.conn = c->conn;
  A.gradN = c->gradN;
  A.J0w = c->J0w;
  A.cls = c->cls;
  A.cls_tab = c->cls_tab;
  A.n_cls = c->n_cls;
  A.aff = c->aff;
  A.jinv = c->jinv;
  A.g0 = 0;
  A.x = x;
  A.v = v;
  A.mat = c->mat;
  A.fscr = c->fscr;
  A.Kscr = c->Kscr;
  A.dest = c->dest;
  A.fdest = c->fdest;
  A.err = c->err_flag;
  A.inv_h = c->eval_inv_h;
  A.cls_mass = c->cls_mass;
  A.mass_closed = (c->mass_rule == 0 && c->affine) ? 1 : 0;
  return A;
}

template <int ELEM, int NQ, int MODEL, bool KV, bool TAN>
static tlfea_status launch_el(Context* c, const double* x, const double* v, cudaStream_t s, int64_t e_begin,
                              int64_t e_end) {
  using G = Geo<ELEM>;
  const int64_t per_cta = (int64_t)kWarps * G::EPW;
  if (e_end <= e_begin) return TLFEA_OK;
  if constexpr (ELEM == 0 && MODEL == 0 && !KV && !TAN && TLFEA_FORCE_AFF) {
    if ((c->n_cls > 0 && c->cls_aff) || (c->n_cls == 0 && c->aff)) {
      ElArgs A = el_args(c, x, v);
      A.n_el = e_end;
      const unsigned grid = (unsigned)((e_end - e_begin + kFABlock - 1) / kFABlock);
      if (c->n_cls > 0 && c->inr) {  // the AdamW gradient with element-level inertia (v holds v - v_n)
        const size_t smem = sizeof(double) * c->n_cls * (13 + 100);
        k_force_t10_aff<NQ, true, true><<<grid, kFABlock, smem, s>>>(A, e_begin, c->cls_aff);
      } else if (c->n_cls > 0) {
        const size_t smem = sizeof(double) * c->n_cls * 13;
        k_force_t10_aff<NQ, true><<<grid, kFABlock, smem, s>>>(A, e_begin, c->cls_aff);
      } else {
        k_force_t10_aff<NQ, false><<<grid, kFABlock, 0, s>>>(A, e_begin, nullptr);
      }
      TL_CHECK_LAUNCH();
      return TLFEA_OK;
    }
  }
  if constexpr (ELEM == 0 && MODEL == 0 && !KV && !TAN && TLFEA_FORCE_WIDE) {
    if (c->n_cls > 0) {
      const int64_t per = (int64_t)kFW * (32 / NQ);
      const size_t smem = sizeof(double) * c->n_cls * NQ * (G::NEN * 3 + 1);
      ElArgs A = el_args(c, x, v);
      A.n_el = e_end;
      auto kern = k_force_t10svk_wide<NQ>;
      TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem, kFW * 32));
      int64_t grid = (e_end - e_begin + per - 1) / per;
      if (TLFEA_FW_PERSIST) {  // one resident wave of persistent CTAs
        int dev = 0, nsm = 0, occ = 0;
        TL_CUDA(cudaGetDevice(&dev));
        TL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        TL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFW * 32, smem));
        grid = std::min<int64_t>(grid, (int64_t)nsm * std::max(occ, 1));
      }
      kern<<<(unsigned)grid, kFW * 32, smem, s>>>(A, e_begin);
      TL_CHECK_LAUNCH();
      return TLFEA_OK;
    }
  }
  // force only, one lane per point: ANCF, and T10 with Mooney-Rivlin or Kelvin-Voigt
  // (T10 SVK without damping has the affine and two-phase kernels)
  if constexpr ((ELEM != 0 || MODEL != 0 || KV) && !TAN && TLFEA_FORCE_LPQ) {
    constexpr int EPWq = NQ >= 32 ? 1 : 32 / NQ;
    const int64_t per = (int64_t)kWarps * EPWq;
    ElArgs A = el_args(c, x, v);
    A.n_el = e_end;
    const unsigned grid = (unsigned)((e_end - e_begin + per - 1) / per);
    const size_t smem = sizeof(double) * ((size_t)kWarps * 32 * (3 * G::NEN + 1) +
                                          (c->n_cls > 0 ? (size_t)c->n_cls * NQ * (3 * G::NEN + 1) : 0));
    auto kern = c->n_cls > 0 ? k_force_lpq<ELEM, NQ, MODEL, KV, true> : k_force_lpq<ELEM, NQ, MODEL, KV, false>;
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
    kern<<<grid, kWarps * 32, smem, s>>>(A, e_begin);
    TL_CHECK_LAUNCH();
    return TLFEA_OK;
  }
  if (e_begin % per_cta != 0) return fail(TLFEA_E_INVALID, "internal: element range not tile aligned");
  const unsigned grid = (unsigned)((e_end - e_begin + per_cta - 1) / per_cta);
  ElArgs A = el_args(c, x, v);
  A.n_el = e_end;
  A.g0 = e_begin / G::EPW;
  if (c->n_cls > 0) {
    const size_t smem = sizeof(double) * c->n_cls * NQ * (G::NEN * 3 + 1);
    auto kern = k_element<ELEM, NQ, MODEL, KV, TAN, true, el_npass<ELEM, MODEL>()>;
    if constexpr (ELEM == 0 && MODEL == 0 && !KV && TAN) TL_TRY_LAUNCH(ensure_carveout((const void*)kern));
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
    kern<<<grid, kWarps * 32, smem, s>>>(A);
  } else {
    // the T10 two-phase groups stage each warp's element tables in dynamic shared memory
    constexpr bool stage = ELEM == 0 && ((TLFEA_MR_2PH && MODEL == 1 && TAN) || (TLFEA_T10_2PH && MODEL == 0 && !KV));
    const size_t smem = stage ? sizeof(double) * kWarps * G::EPW * NQ * (G::NEN * 3 + 1) : 0;
    if constexpr (stage) {
      if (c->aff) {  // tables generated from the affine (min) layout
        auto kern = k_element<ELEM, NQ, MODEL, KV, TAN, false, el_npass<ELEM, MODEL>(), true>;
        if constexpr (MODEL == 0 && !KV && TAN) TL_TRY_LAUNCH(ensure_carveout((const void*)kern));
        TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
        kern<<<grid, kWarps * 32, smem, s>>>(A);
        TL_CHECK_LAUNCH();
        return TLFEA_OK;
      }
      if (c->jinv) {  // tables generated from the per-(e,q) J^-1 layout (curved T10)
        auto kern = k_element<ELEM, NQ, MODEL, KV, TAN, false, el_npass<ELEM, MODEL>(), false, true>;
        if constexpr (MODEL == 0 && !KV && TAN) TL_TRY_LAUNCH(ensure_carveout((const void*)kern));
        TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
        kern<<<grid, kWarps * 32, smem, s>>>(A);
        TL_CHECK_LAUNCH();
        return TLFEA_OK;
      }
    }
    auto kern = k_element<ELEM, NQ, MODEL, KV, TAN, false, el_npass<ELEM, MODEL>()>;
    if constexpr (ELEM == 0 && MODEL == 0 && !KV && TAN) TL_TRY_LAUNCH(ensure_carveout((const void*)kern));
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
    kern<<<grid, kWarps * 32, smem, s>>>(A);
  }
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

// Consistent KV tangent (NEXT-4): k_element_kvc, class tables or per-(e,q) tables.
template <int ELEM, int NQ, int MODEL>
static tlfea_status launch_el_kvc(Context* c, const double* x, const double* v, cudaStream_t s, int64_t e_begin,
                                  int64_t e_end) {
  using G = Geo<ELEM>;
  const int64_t per_cta = (int64_t)kWarps * G::EPW;
  if (e_end <= e_begin) return TLFEA_OK;
  if (e_begin % per_cta != 0) return fail(TLFEA_E_INVALID, "internal: element range not tile aligned");
  if (!c->dest) return fail(TLFEA_E_INVALID, "internal: consistent KV tangent needs the gather-sorted scratch");
  const unsigned grid = (unsigned)((e_end - e_begin + per_cta - 1) / per_cta);
  ElArgs A = el_args(c, x, v);
  A.n_el = e_end;
  A.g0 = e_begin / G::EPW;
  if constexpr (ELEM == 0 && TLFEA_T10KVC_2PH) {  // the two-phase T10 group
    if (c->n_cls > 0) {
      const size_t smem = sizeof(double) * c->n_cls * NQ * 31;
      auto kern = k_element_t10kvc<NQ, MODEL, true, false>;
      TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
      kern<<<grid, kWarps * 32, smem, s>>>(A);
    } else {
      const size_t smem = sizeof(double) * kWarps * 3 * NQ * 31;
      auto kern = c->aff ? k_element_t10kvc<NQ, MODEL, false, true> : k_element_t10kvc<NQ, MODEL, false, false>;
      TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
      kern<<<grid, kWarps * 32, smem, s>>>(A);
    }
    TL_CHECK_LAUNCH();
    return TLFEA_OK;
  }
  if (c->n_cls > 0) {
    const size_t smem = sizeof(double) * c->n_cls * NQ * (G::NEN * 3 + 1);
    auto kern = k_element_kvc<ELEM, NQ, MODEL, true>;
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
    kern<<<grid, kWarps * 32, smem, s>>>(A);
  } else {
    k_element_kvc<ELEM, NQ, MODEL, false><<<grid, kWarps * 32, 0, s>>>(A);
  }
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

template <int ELEM, int NQ, int MODEL>
static tlfea_status launch_el_kv(Context* c, const double* x, const double* v, bool tan, cudaStream_t s, int64_t e0,
                                 int64_t e1) {
  const bool kv = c->mat.kv && v != nullptr;
  if (tan && c->kvc) {
    if (!v) return fail(TLFEA_E_INVALID, "consistent KV tangent: NULL v");
    return launch_el_kvc<ELEM, NQ, MODEL>(c, x, v, s, e0, e1);
  }
  if (tan)
    return kv ? launch_el<ELEM, NQ, MODEL, true, true>(c, x, v, s, e0, e1)
              : launch_el<ELEM, NQ, MODEL, false, true>(c, x, v, s, e0, e1);
  return kv ? launch_el<ELEM, NQ, MODEL, true, false>(c, x, v, s, e0, e1)
            : launch_el<ELEM, NQ, MODEL, false, false>(c, x, v, s, e0, e1);
}

template <int ELEM, int NQ>
static tlfea_status launch_el_model(Context* c, const double* x, const double* v, bool tan, cudaStream_t s, int64_t e0,
                                    int64_t e1) {
  if (c->mat.model == TLFEA_SVK) return launch_el_kv<ELEM, NQ, 0>(c, x, v, tan, s, e0, e1);
  return launch_el_kv<ELEM, NQ, 1>(c, x, v, tan, s, e0, e1);
}

// Local elements [e_begin, e_end) (e_end < 0: all); e_begin a multiple of
// the element-kernel CTA tile.
// TLFEA_CHECK: register the launch's buffers for the device bounds checks
static tlfea_status check_ranges(const Context* c, const double* H, cudaStream_t s) {
  if (!TLFEA_CHECK) return TLFEA_OK;
  const size_t kb = (size_t)c->n_el * n_ublk_of(c->nen) * (c->kvc ? 18 : 9);
  const double* r[6] = {c->Kscr, c->Kscr + kb, c->fscr, c->fscr + (size_t)c->n_el * c->nen * 3,
                        H, H ? H + c->nnz_H : nullptr};
  TL_CUDA(cudaMemcpyToSymbolAsync(g_rng, r, sizeof(r), 0, cudaMemcpyHostToDevice, s));
  return TLFEA_OK;
}

tlfea_status launch_element_kernel(Context* c, const double* x, const double* v, bool tangent, cudaStream_t s,
                                   int64_t e_begin, int64_t e_end) {
  if (e_end < 0) e_end = c->n_el;
  TL_TRY(check_ranges(c, nullptr, s));
  if (c->element == TLFEA_T10) {
    if (c->nq == 4) return launch_el_model<0, 4>(c, x, v, tangent, s, e_begin, e_end);
    return launch_el_model<0, 5>(c, x, v, tangent, s, e_begin, e_end);
  }
  if (c->element == TLFEA_ANCF3243) return launch_el_model<2, 12>(c, x, v, tangent, s, e_begin, e_end);
  return launch_el_model<1, 48>(c, x, v, tangent, s, e_begin, e_end);
}

// k_force_t10_aff with element-level inertia serves this context (AdamW gradient)
bool force_inertia_capable(const Context* c) {
  return TLFEA_FORCE_AFF && c->element == TLFEA_T10 && c->mat.model == TLFEA_SVK && !c->mat.kv && c->nranks == 1 &&
         c->n_cls > 0 && c->cls_aff && c->cls_mass;
}

static GatherArgs gather_args(const Context* c, double h, double* H) {
  GatherArgs A;
  A.n_units = c->n_units;
  A.unit_ptr = c->unit_ptr;
  A.u_off = c->u_off;
  A.u_offT = c->u_offT;
  A.u_deg = c->u_deg;
  A.u_m = c->u_m;
  A.Kscr = c->Kscr;
  A.h = h;
  A.H = H;
  A.upper = c->upper;
  return A;
}

tlfea_status launch_gather_H(Context* c, double h, double* H, cudaStream_t s) {
  if (c->n_units == 0) return TLFEA_OK;
  TL_TRY(check_ranges(c, H, s));
  const int64_t per = (int64_t)kG3Warps * 32;
  if (c->kvc) {
    k_gather_units_kvc<<<(unsigned)((c->n_units + per - 1) / per), kG3Warps * 32, 0, s>>>(gather_args(c, h, H));
    TL_CHECK_LAUNCH();
    return TLFEA_OK;
  }
  k_gather_units_v3<<<(unsigned)((c->n_units + per - 1) / per), kG3Warps * 32, 0, s>>>(gather_args(c, h, H));
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

}  // namespace tlfea

namespace tlfea {

bool eval_small_ok(const Context* c) {
  return TLFEA_SMALL_MAX_EL > 0 && TLFEA_T10_2PH && c->element == TLFEA_T10 && c->mat.model == TLFEA_SVK &&
         !c->mat.kv && !c->kvc && c->nranks == 1 && c->n_cls > 0 && c->dest && c->n_el <= TLFEA_SMALL_MAX_EL &&
         c->n_units > 0;
}

template <int NQ>
static tlfea_status launch_small_t(Context* c, const double* x, const double* v, const double* vn, const double* fext,
                                   double h, double* g, double* H, double* fint, cudaStream_t s) {
  ElArgs A = el_args(c, x, v);
  GatherArgs G = gather_args(c, h, H);
  FArgs F;
  F.n_own = c->n_own;
  F.node_ptr = c->node_ptr;
  F.fscr = c->fscr;
  F.fpart_in = nullptr;
  F.own_nodes = c->own_nodes;
  F.rowptr_c = c->rowptr_c;
  F.cols_c = c->cols_c;
  F.M = c->M;
  F.fff = c->fff;
  F.v = v;
  F.vn = vn;
  F.fext = fext;
  F.h = h;
  F.mode = 0;
  F.g = g;
  F.fint = fint;
  auto kern = k_eval_small<NQ>;
  const size_t smem = std::max(sizeof(double) * c->n_cls * NQ * 31,
                               sizeof(double) * kWarps * 2 * kG3Buf + sizeof(uint64_t) * kWarps * 2);
  TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)kern, smem));
  TL_TRY(check_ranges(c, H, s));
  int dev = 0, nsm = 0, occ = 0;
  TL_CUDA(cudaGetDevice(&dev));
  TL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  TL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, smem));
  const int64_t need = std::max(((c->n_el + 2) / 3 + kWarps - 1) / kWarps,
                                (c->n_units / 32 + kWarps) / kWarps);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * std::max(occ, 1)));
  void* args[] = {&A, &G, &F};
  TL_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kWarps * 32), args, smem, s));
  count_launch();
  return TLFEA_OK;
}

tlfea_status launch_eval_small(Context* c, const double* x, const double* v, const double* vn, const double* fext,
                               double h, double* g, double* H, double* fint, cudaStream_t s) {
  if (c->nq == 4) return launch_small_t<4>(c, x, v, vn, fext, h, g, H, fint, s);
  return launch_small_t<5>(c, x, v, vn, fext, h, g, H, fint, s);
}

}  // namespace tlfea
