// tile.cu — the one-kernel eval of libtlfea (B200 / sm_100a, fp64):
// Stage 1 + Stage 2 (force, tangent) + the deterministic CSR assembly of
// H = M/h + h K and of the residual g, with no element scratch in HBM.
//
// PAPER.md §4.3-4.4 computes per element and scatters every 3x3 block with
// atomicAdd; the paper names "blockwise accumulation,
// or two-pass scatter/reduction" as the way out. The two-kernel path
// of element.cu is that two-pass reduction: every element block crosses HBM
// twice (the gather-sorted scratch). Here the reduction is blockwise per CTA
// and the scratch disappears:
//
//   * Setup cuts the owned nodes into spatial tiles (aligned 4x4x4 blocks of
//     a Morton order of the reference coordinates, <= kTileMaxEl touching
//     elements). A tile owns the H gather units {(I,J),(J,I)}, I <= J, whose
//     row node I it holds (the units of element.cu).
//   * Phase A (per tile): the CTA stages x of every element touching the tile
//     and evaluates, once per (element, q), F = sum_a x_a (x) grad N_a
//     (Eq. F_assembly) and the SVK S (reading Q5) into shared memory.
//   * Phase B: one lane per unit sums its element contributions
//       K_ab = sum_q [ (grad N_a . S grad N_b) I + lam G_a G_b^T + mu G_b G_a^T
//                      + mu (grad N_a . grad N_b) F F^T ] J0 w_q,
//     G_a = F grad N_a (Eq. tangent_block), in ascending element
//     order, and writes h K + M_IJ/h I to (I,J) and its transpose to (J,I)
//     (Eq. hessian). The lane of a diagonal unit (I,I) also sums the
//     nodal force f_I = sum_e sum_q F (S grad N_a) J0 w_q (Eq. fint_local/global
//     P:408-423) and writes f_int and the residual g (Eq. residual).
//   Every H / f / g value is summed by one thread in a fixed order: results
//   are bitwise reproducible run to run, with no float atomics.
//
// Each element is staged by every tile it touches (about 2.5 tiles per
// element on Kuhn boxes): the kinematics are recomputed instead of stored.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "material.cuh"

namespace tlfea {

// ------------------------------------------------------------- the kernel

struct TileArgs {
  const int32_t* t_rec_ptr;  // [n_tiles+1] staged element records of each tile
  const uint16_t* t_rec;     // [visits][12]: 10 local node indices, class id, pad
  const int32_t* t_node_ptr; // [n_tiles+1] nodes of each tile (owned first, then halo)
  const int32_t* t_node;     // global coefficient ids
  const int32_t* t_warp_ptr; // [n_tiles+1] warp items of each tile
  const int32_t* w_ent;      // [n_items] first entry of the item's interleaved step list
  const int32_t* w_info;     // [n_items] steps | diagonal lanes << 16 | (parts - 1) << 17 | units per lane << 24
  const uint64_t* ent;       // (step, lane) at w_ent + 32 step + lane: slot | (a_j << 4 | b_j) << (8 + 8 j)
  const int32_t* l_lane;     // [n_items*32] part (0 head) | diagonal unit in slot 0 << 8; -1 empty lane
  const int32_t* l_off;      // [n_items][KU][32] H offset of (I,J) of unit slot j, -1 none
  const int32_t* l_aux;      // offT of (J,I) (-1 none); diagonal unit: the owned row i
  const int32_t* l_deg;      // deg I | deg J << 16
  const double* l_m;         // M_IJ
  const double* cls_tab;     // [n_cls][NQ][31]
  int n_cls;
  int n_tiles;
  const double* x;
  const double* fext;
  const double* fff;
  double lam, mu, h;
  double* H;
  double* g;
  double* fint;
};

// One warp item's metadata, loaded one item ahead of its use.
struct ItemPre {
  int info;
  int lane_info;
  const uint64_t* ent;  // this lane's step column
  uint64_t en0;         // its first step
};

__device__ __forceinline__ void item_load(const TileArgs& A, int w, ItemPre& p) {
  const int lane = threadIdx.x & 31;
  p.info = A.w_info[w];
  p.lane_info = A.l_lane[w * 32 + lane];
  p.ent = A.ent + A.w_ent[w] + lane;
  p.en0 = p.ent[0];  // the step array carries 32 padding entries
}

// One warp item of phase B. A lane holds NU units (I_j, J_j) that share the
// same contributing elements; each step is one element: its per-(element, q)
// kinematics are read once and serve all NU blocks
//   K_ab += (grad N_a . S grad N_b) I + lam G_a G_b^T + mu G_b G_a^T
//           + mu (grad N_a . grad N_b) F F^T,  all times J0 w_q
// (Eq. tangent_block, G_a = F grad N_a). DIAG: the item has lanes
// whose slot 0 is a diagonal unit (I,I); those also sum the nodal force
// f_I = sum F (S grad N_a) J0 w_q (Eq. fint_local/global P:408-423).
template <int NQ, bool DIAG, int NU>
__device__ __forceinline__ void tile_item(const TileArgs& A, int w, const ItemPre& P, const double* s_tab,
                                          const double* s_kin, const uint16_t* s_rec) {
  constexpr int TABW = 31, KS = 15;
  const int lane = threadIdx.x & 31;
  const int steps = P.info & 0xffff, maxpart = ((P.info >> 17) & 0x7f) + 1;
  const int part = P.lane_info < 0 ? -1 : (P.lane_info & 0xff);
  const bool dlane = DIAG && P.lane_info >= 0 && ((P.lane_info >> 8) & 1);
  double acc[NU][9], f[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < NU; ++j)
#pragma unroll
    for (int r = 0; r < 9; ++r) acc[j][r] = 0.0;
  uint64_t en_next = P.en0;
  const double lam = A.lam, mu = A.mu;
#pragma unroll 1
  for (int st = 0; st < steps; ++st) {
    const uint64_t en = en_next;
    if (st + 1 < steps) en_next = P.ent[32 * (st + 1)];  // one step ahead
    const int s = (int)(en & 0xff);
    if (s == 0xff) continue;
    const double* tb0 = s_tab + s_rec[12 * s + 10] * NQ * TABW;
    const double* k0 = s_kin + s * NQ * KS;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double* tb = tb0 + q * TABW;
      const double* k = k0 + q * KS;
      const double w = tb[30];
      double F[9], S[6];
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = k[r];
#pragma unroll
      for (int r = 0; r < 6; ++r) S[r] = k[9 + r];
      double B[6];  // F F^T (Voigt), shared by the lane's blocks
#pragma unroll
      for (int v = 0; v < 6; ++v) {
        int i, kk;
        voigt_pair(v, i, kk);
        B[v] = F[3 * i] * F[3 * kk] + F[3 * i + 1] * F[3 * kk + 1] + F[3 * i + 2] * F[3 * kk + 2];
      }
      const double lw = lam * w, mw = mu * w;
#pragma unroll
      for (int j = 0; j < NU; ++j) {
        const unsigned ab = (unsigned)(en >> (8 + 8 * j)) & 0xffu;
        if (ab == 0xffu) continue;
        const int a = ab >> 4, b = ab & 15;
        const double na[3] = {tb[3 * a], tb[3 * a + 1], tb[3 * a + 2]};
        const double nb[3] = {tb[3 * b], tb[3 * b + 1], tb[3 * b + 2]};
        double Ga[3], Gb[3], ta[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          Ga[i] = F[3 * i] * na[0] + F[3 * i + 1] * na[1] + F[3 * i + 2] * na[2];
          Gb[i] = F[3 * i] * nb[0] + F[3 * i + 1] * nb[1] + F[3 * i + 2] * nb[2];
          ta[i] = w * (sget(S, i, 0) * na[0] + sget(S, i, 1) * na[1] + sget(S, i, 2) * na[2]);
        }
        if (DIAG && j == 0 && dlane) {  // f_a += F (w S grad N_a)   (Eq. fint_local)
#pragma unroll
          for (int i = 0; i < 3; ++i)
            f[i] = fma(F[3 * i], ta[0], fma(F[3 * i + 1], ta[1], fma(F[3 * i + 2], ta[2], f[i])));
        }
        const double sab = ta[0] * nb[0] + ta[1] * nb[1] + ta[2] * nb[2];
        const double dab = mw * (na[0] * nb[0] + na[1] * nb[1] + na[2] * nb[2]);
        double gl[3], gm[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          gl[i] = lw * Ga[i];
          gm[i] = mw * Gb[i];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            double r = fma(gl[i], Gb[kk], fma(gm[i], Ga[kk], fma(dab, B[vidx(i, kk)], acc[j][3 * i + kk])));
            acc[j][3 * i + kk] = (i == kk) ? r + sab : r;
          }
      }
    }
  }
  if (maxpart > 1) {  // parts of a split lane job: head += part 1 + part 2 ... (fixed order)
    for (int k = 1; k < maxpart; ++k) {
      const int pk = __shfl_down_sync(0xffffffffu, part, k);
      const bool take = lane + k < 32 && pk == k;
#pragma unroll
      for (int j = 0; j < NU; ++j)
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          const double o = __shfl_down_sync(0xffffffffu, acc[j][r], k);
          if (take) acc[j][r] += o;
        }
      if constexpr (DIAG) {
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double o = __shfl_down_sync(0xffffffffu, f[r], k);
          if (take) f[r] += o;
        }
      }
    }
  }
  if (part != 0) return;
  const double h = A.h;
#pragma unroll
  for (int j = 0; j < NU; ++j) {
    const int li = (w * kTileKU + j) * 32 + lane;
    const int32_t off = A.l_off[li];
    if (off < 0) continue;
    const int32_t aux = A.l_aux[li], dg = A.l_deg[li];
    const double mh = A.l_m[li] / h;
    const int deg = dg & 0xffff, degT = dg >> 16;
    double* out = A.H + off;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int ff = 0; ff < 3; ++ff) out[3 * d * deg + ff] = fma(h, acc[j][3 * d + ff], d == ff ? mh : 0.0);
    if (DIAG && j == 0 && dlane) {
      // owned row i = aux: f_int, and the force part of the residual g
      // (k_mass_residual wrote (1/h) sum_J M_IJ (v - v_n)_J - f_ext - f_ff)
      const int64_t i = aux;
      if (A.fint) {
#pragma unroll
        for (int d = 0; d < 3; ++d) A.fint[3 * i + d] = f[d];
      }
      if (A.g) {
#pragma unroll
        for (int d = 0; d < 3; ++d) A.g[3 * i + d] += f[d];
      }
    } else if (aux >= 0) {
      double* o2 = A.H + aux;
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int ff = 0; ff < 3; ++ff) o2[3 * d * degT + ff] = fma(h, acc[j][3 * ff + d], d == ff ? mh : 0.0);
    }
  }
}

template <int NQ, bool DIAG, int NU>
__device__ __forceinline__ void tile_item_nu(const TileArgs& A, int w, const ItemPre& P, int nu, const double* s_tab,
                                             const double* s_kin, const uint16_t* s_rec) {
  if constexpr (NU < kTileKU) {
    if (nu > NU) {
      tile_item_nu<NQ, DIAG, NU + 1>(A, w, P, nu, s_tab, s_kin, s_rec);
      return;
    }
  }
  tile_item<NQ, DIAG, NU>(A, w, P, s_tab, s_kin, s_rec);
}

template <int NQ>
__device__ __forceinline__ void tile_item_dispatch(const TileArgs& A, int w, const ItemPre& P, const double* s_tab,
                                                   const double* s_kin, const uint16_t* s_rec) {
  const int nu = (P.info >> 24) & 0xf;
  if ((P.info >> 16) & 1)
    tile_item_nu<NQ, true, 1>(A, w, P, nu, s_tab, s_kin, s_rec);
  else
    tile_item_nu<NQ, false, 1>(A, w, P, nu, s_tab, s_kin, s_rec);
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

// Issue the staging copies of one tile: element records and x of its nodes
// (node ids loaded by the caller, two per thread).
__device__ __forceinline__ void tile_stage(const TileArgs& A, int tile, int64_t I0, int64_t I1, double* s_x,
                                           uint16_t* s_rec) {
  const int r0 = A.t_rec_ptr[tile], ne = A.t_rec_ptr[tile + 1] - r0;
  const int nn = A.t_node_ptr[tile + 1] - A.t_node_ptr[tile];
  const uint2* src = reinterpret_cast<const uint2*>(A.t_rec + 12 * (int64_t)r0);
  uint2* dst = reinterpret_cast<uint2*>(s_rec);
  for (int t = threadIdx.x; t < 3 * ne; t += blockDim.x) cp_async8(dst + t, src + t);
  const int t0 = threadIdx.x, t1 = threadIdx.x + blockDim.x;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (t0 < nn) cp_async8(s_x + 3 * t0 + d, A.x + 3 * I0 + d);
    if (t1 < nn) cp_async8(s_x + 3 * t1 + d, A.x + 3 * I1 + d);
  }
}

__device__ __forceinline__ void tile_node_ids(const TileArgs& A, int tile, int64_t& I0, int64_t& I1) {
  const int n0 = A.t_node_ptr[tile], nn = A.t_node_ptr[tile + 1] - n0;
  const int t0 = threadIdx.x, t1 = threadIdx.x + blockDim.x;
  I0 = t0 < nn ? A.t_node[n0 + t0] : 0;
  I1 = t1 < nn ? A.t_node[n0 + t1] : 0;
}

// Persistent: CTA c runs tiles c, c + gridDim.x, ...; the next tile's records
// and coordinates stream into the other staging buffer (cp.async) during the
// current tile's phase B; phase-B items go to the warps through a shared
// ticket, longest first.
template <int NQ>
__global__ void __launch_bounds__(kTileWarps * 32, 2) k_tile_eval(TileArgs A) {
  constexpr int TABW = 31;       // class table row: grad N (30) + J0 w
  constexpr int KS = 15;         // per (element, q): F (9), S (6)
  static_assert(kTileMaxNode <= 2 * kTileWarps * 32, "two nodes per thread");
  extern __shared__ __align__(16) double sm[];
  const int tabn = A.n_cls * NQ * TABW;
  double* s_tab = sm;
  double* s_kin = sm + ((tabn + 1) & ~1);
  double* s_xb = s_kin + kTileMaxEl * NQ * KS;                               // [2][node][3]
  uint16_t* s_rb = reinterpret_cast<uint16_t*>(s_xb + 2 * 3 * kTileMaxNode);  // [2][slot][12]
  int* s_ticket = reinterpret_cast<int*>(s_rb + 2 * 12 * kTileMaxEl);
  const int lane = threadIdx.x & 31;
  int tile = blockIdx.x;
  if (tile >= A.n_tiles) return;
  for (int t = threadIdx.x; t < tabn; t += blockDim.x) cp_async8(s_tab + t, A.cls_tab + t);
  {
    int64_t I0, I1;
    tile_node_ids(A, tile, I0, I1);
    tile_stage(A, tile, I0, I1, s_xb, s_rb);
  }
#pragma unroll 1
  for (int it = 0; tile < A.n_tiles; ++it, tile += gridDim.x) {
    const int b = it & 1;
    const double* s_x = s_xb + b * 3 * kTileMaxNode;
    const uint16_t* s_rec = s_rb + b * 12 * kTileMaxEl;
    const int next = tile + gridDim.x;
    int64_t J0 = 0, J1 = 0;  // the next tile's node ids, consumed after phase A
    if (next < A.n_tiles) tile_node_ids(A, next, J0, J1);
    const int w0 = A.t_warp_ptr[tile], w1 = A.t_warp_ptr[tile + 1];
    const int ne = A.t_rec_ptr[tile + 1] - A.t_rec_ptr[tile];
    cp_async_commit_wait();
    __syncthreads();
    // ---- phase A: item (slot, q): F (Eq. F_assembly) and S (SVK, reading Q5)
    for (int t = threadIdx.x; t < ne * NQ; t += blockDim.x) {
      const int s = t / NQ, q = t - NQ * s;
      const uint16_t* rc = s_rec + 12 * s;
      const double* tb = s_tab + (rc[10] * NQ + q) * TABW;
      double F[9];
#pragma unroll
      for (int r = 0; r < 9; ++r) F[r] = 0.0;
#pragma unroll
      for (int a = 0; a < 10; ++a) {
        const double n0 = tb[3 * a], n1 = tb[3 * a + 1], n2 = tb[3 * a + 2];
        const double* xa = s_x + 3 * rc[a];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xi = xa[i];
          F[3 * i] = fma(xi, n0, F[3 * i]);
          F[3 * i + 1] = fma(xi, n1, F[3 * i + 1]);
          F[3 * i + 2] = fma(xi, n2, F[3 * i + 2]);
        }
      }
      double S[6];
      svk_S(F, A.lam, A.mu, S);
      double* k = s_kin + (s * NQ + q) * KS;
#pragma unroll
      for (int r = 0; r < 9; ++r) k[r] = F[r];
#pragma unroll
      for (int r = 0; r < 6; ++r) k[9 + r] = S[r];
    }
    if (threadIdx.x == 0) *s_ticket = 0;
    __syncthreads();
    if (next < A.n_tiles)
      tile_stage(A, next, J0, J1, s_xb + (b ^ 1) * 3 * kTileMaxNode, s_rb + (b ^ 1) * 12 * kTileMaxEl);
    // ---- phase B
    auto ticket = [&]() {
      int k = 0;
      if (lane == 0) k = atomicAdd(s_ticket, 1);
      return w0 + __shfl_sync(0xffffffffu, k, 0);
    };
    int w = ticket();
    ItemPre cur;
    if (w < w1) item_load(A, w, cur);
    while (w < w1) {
      const int wn = ticket();
      ItemPre nxt;
      if (wn < w1) item_load(A, wn, nxt);
      tile_item_dispatch<NQ>(A, w, cur, s_tab, s_kin, s_rec);
      cur = nxt;
      w = wn;
    }
  }
}

// The mass part of the residual, one thread per owned DOF t = 3i + d
// (Eq. residual; f_ff reading Q10):
//   g[t] = (1/h) sum_J M_IJ (v - v_n)_{3J+d} - f_ext - f_ff,  f_int[t] = 0;
// k_tile_eval then adds the nodal force of every row with elements.
__global__ void k_mass_residual(int64_t n_own, const int32_t* __restrict__ own_nodes,
                                const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ cols_c,
                                const double* __restrict__ M, const double* __restrict__ v,
                                const double* __restrict__ vn, const double* __restrict__ fext,
                                const double* __restrict__ fff, double h, double* __restrict__ g,
                                double* __restrict__ fint) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 3 * n_own) return;
  const int64_t i = t / 3;
  const int d = (int)(t - 3 * i);
  if (fint) fint[t] = 0.0;
  if (!g) return;
  double m = 0.0;
  const int32_t p0 = rowptr_c[i], p1 = rowptr_c[i + 1];
#pragma unroll 4
  for (int32_t p = p0; p < p1; ++p) {
    const int64_t J = cols_c[p];
    m += M[p] * (v[3 * J + d] - (vn ? vn[3 * J + d] : 0.0));
  }
  const int64_t I = own_nodes[i];
  g[t] = m / h - (fext ? fext[3 * I + d] : 0.0) - fff[t];
}

size_t tile_smem_bytes(int n_cls, int nq) {
  const size_t tabn = (size_t)n_cls * nq * 31;
  return sizeof(double) * (((tabn + 1) & ~(size_t)1) + (size_t)kTileMaxEl * nq * 15 + 6 * (size_t)kTileMaxNode) +
         sizeof(uint16_t) * 24 * kTileMaxEl + sizeof(int);
}

// persistent grid: resident CTAs per SM x SMs (computed once per context)
static unsigned tile_grid(Context* c, const void* kern, size_t smem) {
  if (c->tile_grid == 0) {
    int per_sm = 0, n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, c->device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileWarps * 32, smem);
    c->tile_grid = (int)std::min<int64_t>(std::max(1, per_sm) * (int64_t)std::max(1, n_sm), c->n_tiles);
  }
  return (unsigned)c->tile_grid;
}

tlfea_status launch_tile_eval(Context* c, const double* x, const double* v, const double* vn, const double* fext,
                              double h, double* g, double* H, double* fint, cudaStream_t s) {
  if (c->n_tiles == 0) return TLFEA_OK;
  TileArgs A;
  A.t_rec_ptr = c->t_rec_ptr;
  A.t_rec = c->t_rec;
  A.t_node_ptr = c->t_node_ptr;
  A.t_node = c->t_node;
  A.t_warp_ptr = c->t_warp_ptr;
  A.w_ent = c->w_ent;
  A.w_info = c->w_info;
  A.ent = c->t_ent;
  A.l_lane = c->l_lane;
  A.l_off = c->l_off;
  A.l_aux = c->l_aux;
  A.l_deg = c->l_deg;
  A.l_m = c->l_m;
  A.cls_tab = c->cls_tab;
  A.n_cls = c->n_cls;
  A.n_tiles = (int)c->n_tiles;
  A.x = x;
  A.fext = fext;
  A.fff = c->fff;
  A.lam = c->mat.lam;
  A.mu = c->mat.mu;
  A.h = h;
  A.H = H;
  A.g = g;
  A.fint = fint;
  if (c->n_own > 0) {
    k_mass_residual<<<(unsigned)((3 * c->n_own + 255) / 256), 256, 0, s>>>(
        c->n_own, c->own_nodes, c->rowptr_c, c->cols_c, c->M, v, vn, fext, c->fff, h, g, fint);
    TL_CHECK_LAUNCH();
  }
  const size_t smem = tile_smem_bytes(c->n_cls, c->nq);
  if (c->nq == 4) {
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)k_tile_eval<4>, smem));
    k_tile_eval<4><<<tile_grid(c, (const void*)k_tile_eval<4>, smem), kTileWarps * 32, smem, s>>>(A);
  } else {
    TL_TRY_LAUNCH(ensure_dynamic_smem((const void*)k_tile_eval<5>, smem));
    k_tile_eval<5><<<tile_grid(c, (const void*)k_tile_eval<5>, smem), kTileWarps * 32, smem, s>>>(A);
  }
  TL_CHECK_LAUNCH();
  return TLFEA_OK;
}

// ------------------------------------------------------------- the plan

namespace {

uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffULL;
  v = (v | v << 16) & 0x1f0000ff0000ffULL;
  v = (v | v << 8) & 0x100f00f00f00f00fULL;
  v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
  v = (v | v << 2) & 0x1249249249249249ULL;
  return v;
}

template <class T>
tlfea_status d2h(std::vector<T>& h, const T* d, size_t n) {
  h.resize(n);
  if (n) TL_CUDA(cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost));
  return TLFEA_OK;
}

template <class T>
tlfea_status h2d(Context* c, T** d, const std::vector<T>& h) {
  TL_TRY(c->alloc(d, std::max<size_t>(h.size(), 1)));
  if (!h.empty()) TL_CUDA(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return TLFEA_OK;
}

}  // namespace

// Tiles, their staged elements, and per-warp interleaved contribution lists
// (the blk_ent lists of the units, element ids replaced by tile slots). Runs
// on the host from the device-built pattern / unit arrays. Applies to
// single-rank T10 SVK contexts with geometry classes and FULL H storage;
// anything else keeps the two-kernel path (c->n_tiles = 0).
tlfea_status build_tile_plan(Context* c, const double* X_host) {
  c->n_tiles = 0;
  if (c->element != TLFEA_T10 || c->mat.model != TLFEA_SVK || c->mat.kv || c->nranks != 1 || c->n_cls == 0 ||
      c->upper || c->n_con > 0 || c->n_units == 0 || c->force_tables)
    return TLFEA_OK;
  if ((size_t)c->n_cls * c->nq * 31 > 4096) return TLFEA_OK;
  const int64_t n_own = c->n_own, nnz_c = c->nnz_c, n_units = c->n_units, n_el = c->n_el;
  std::vector<int32_t> own, unit_p, blk_ptr, blk_row, cols, conn, u_off, u_offT, u_deg;
  std::vector<uint32_t> blk_ent;
  std::vector<double> u_m;
  TL_TRY(d2h(own, c->own_nodes, n_own));
  TL_TRY(d2h(unit_p, c->unit_p, n_units));
  TL_TRY(d2h(blk_ptr, c->blk_ptr, nnz_c + 1));
  TL_TRY(d2h(blk_row, c->blk_row, nnz_c));
  TL_TRY(d2h(cols, c->cols_c, nnz_c));
  TL_TRY(d2h(blk_ent, c->blk_ent, (size_t)blk_ptr[nnz_c]));
  TL_TRY(d2h(conn, c->conn, (size_t)n_el * 10));
  TL_TRY(d2h(u_off, c->u_off, n_units));
  TL_TRY(d2h(u_offT, c->u_offT, n_units));
  TL_TRY(d2h(u_deg, c->u_deg, n_units));
  TL_TRY(d2h(u_m, c->u_m, n_units));

  // ---- node tiles: aligned 4x4x4 blocks of a Morton order on a grid of half
  // the smallest element extent (the T10 node spacing of a Kuhn box)
  double lo[3] = {1e300, 1e300, 1e300}, dq[3] = {1e300, 1e300, 1e300};
  for (int64_t i = 0; i < n_own; ++i)
    for (int k = 0; k < 3; ++k) lo[k] = std::min(lo[k], X_host[3 * (int64_t)own[i] + k]);
  for (int64_t e = 0; e < n_el; ++e)
    for (int k = 0; k < 3; ++k) {
      double mn = 1e300, mx = -1e300;
      for (int a = 0; a < 4; ++a) {
        const double v = X_host[3 * (int64_t)conn[e * 10 + a] + k];
        mn = std::min(mn, v);
        mx = std::max(mx, v);
      }
      if (mx > mn) dq[k] = std::min(dq[k], 0.5 * (mx - mn));
    }
  for (int k = 0; k < 3; ++k)
    if (!(dq[k] < 1e300)) dq[k] = 1.0;
  std::vector<uint64_t> code(n_own);
  for (int64_t i = 0; i < n_own; ++i) {
    uint64_t m = 0;
    for (int k = 0; k < 3; ++k) {
      const double r = (X_host[3 * (int64_t)own[i] + k] - lo[k]) / dq[k];
      const uint64_t qk = (uint64_t)std::min(std::max(std::llround(r), 0LL), (long long)0x1fffff);
      m |= spread3(qk) << k;
    }
    code[i] = m;
  }
  std::vector<int32_t> order(n_own);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return code[a] < code[b]; });
  // units of owned row i are contiguous (units ascend in block index)
  std::vector<int64_t> row_u(n_own + 1, 0);
  for (int64_t u = 0; u < n_units; ++u) row_u[blk_row[unit_p[u]] + 1]++;
  for (int64_t i = 0; i < n_own; ++i) row_u[i + 1] += row_u[i];

  std::vector<int32_t> t_rec_ptr{0}, t_node_ptr{0}, t_node, t_warp_ptr{0}, w_ent, w_info, l_off,
      l_aux, l_deg;
  std::vector<uint16_t> t_rec;
  std::vector<uint8_t> hcls;
  TL_TRY(d2h(hcls, c->cls, n_el));
  std::vector<int32_t> node_loc(c->n_coef, -1);  // local index of a node in the tile being emitted
  std::vector<int32_t> halo;
  std::vector<double> l_m;
  std::vector<uint64_t> ent;
  std::vector<int32_t> l_lane;
  std::vector<int32_t> slot_of(n_el, -1);
  std::vector<int32_t> els;

  // Emit the tile of owned rows rows[0..n) if its elements fit; else split in
  // Morton halves. Returns false on an internal limit.
  std::vector<std::pair<int64_t, int64_t>> stack;
  auto elements_of = [&](const int32_t* rows, int64_t n) {
    els.clear();
    for (int64_t k = 0; k < n; ++k)
      for (int64_t u = row_u[rows[k]]; u < row_u[rows[k] + 1]; ++u) {
        const int32_t p = unit_p[u];
        for (int32_t t = blk_ptr[p]; t < blk_ptr[p + 1]; ++t) els.push_back((int32_t)(blk_ent[t] >> 8));
      }
    std::sort(els.begin(), els.end());
    els.erase(std::unique(els.begin(), els.end()), els.end());
  };
  // A tile's lane jobs. Units with the same contributing elements form a
  // group; a lane job holds <= kTileKU units of one group (a diagonal unit, if
  // any, in slot 0) and runs over the group's elements, one element per step.
  // A job with more than kTileCap elements is split into consecutive-lane
  // parts of <= kTileCap steps (summed in part order after the step loop).
  // Jobs sorted by (diagonal, units, steps, elements) and packed into 32-lane
  // warp items (parts never straddle two items); items listed longest first.
  struct Job {
    int diag = 0;
    std::vector<int64_t> units;  // <= kTileKU, diagonal first
    int t0 = 0, t1 = 0;          // element range of the group (steps)
    int part = 0, nparts = 1;
    const std::vector<int32_t>* els = nullptr;  // the group's element list
  };
  struct Item {
    int steps = 0, diag = 0, maxpart = 1, nu = 1;
    std::vector<int> job;  // per lane, -1 empty
  };
  std::vector<Job> jobs;
  std::vector<Item> items;
  std::vector<std::pair<std::vector<int32_t>, int64_t>> ukeys;  // (element list, unit)
  // nodes of the tile: its owned rows' nodes (in the given order), then the
  // other nodes of its elements (ascending); returns the count
  auto nodes_of = [&](const int32_t* rows, int64_t n) -> int64_t {
    for (int64_t k = 0; k < n; ++k) node_loc[own[rows[k]]] = (int32_t)k;
    halo.clear();
    for (int32_t e : els)
      for (int a = 0; a < 10; ++a) {
        const int32_t I = conn[(int64_t)e * 10 + a];
        if (node_loc[I] < 0) {
          node_loc[I] = -2;
          halo.push_back(I);
        }
      }
    std::sort(halo.begin(), halo.end());
    for (size_t k = 0; k < halo.size(); ++k) node_loc[halo[k]] = (int32_t)(n + k);
    return n + (int64_t)halo.size();
  };
  auto clear_nodes = [&](const int32_t* rows, int64_t n) {
    for (int64_t k = 0; k < n; ++k) node_loc[own[rows[k]]] = -1;
    for (int32_t I : halo) node_loc[I] = -1;
  };
  auto emit = [&](const int32_t* rows, int64_t n) -> bool {
    for (size_t s = 0; s < els.size(); ++s) slot_of[els[s]] = (int32_t)s;
    for (int32_t e : els) {
      for (int a = 0; a < 10; ++a) t_rec.push_back((uint16_t)node_loc[conn[(int64_t)e * 10 + a]]);
      t_rec.push_back(hcls[e]);
      t_rec.push_back(0);
    }
    t_rec_ptr.push_back((int32_t)(t_rec.size() / 12));
    for (int64_t k = 0; k < n; ++k) t_node.push_back(own[rows[k]]);
    t_node.insert(t_node.end(), halo.begin(), halo.end());
    t_node_ptr.push_back((int32_t)t_node.size());
    // ---- groups of units with identical element lists
    ukeys.clear();
    for (int64_t k = 0; k < n; ++k)
      for (int64_t u = row_u[rows[k]]; u < row_u[rows[k] + 1]; ++u) {
        const int32_t p = unit_p[u];
        std::vector<int32_t> el;
        for (int32_t t = blk_ptr[p]; t < blk_ptr[p + 1]; ++t) el.push_back((int32_t)(blk_ent[t] >> 8));
        ukeys.push_back({std::move(el), u});
      }
    auto is_diag = [&](int64_t u) { return cols[unit_p[u]] == own[blk_row[unit_p[u]]]; };
    std::sort(ukeys.begin(), ukeys.end(), [&](const auto& x, const auto& y) {
      if (x.first != y.first) return x.first < y.first;
      const int dx = is_diag(x.second), dy = is_diag(y.second);
      return dx != dy ? dx > dy : x.second < y.second;
    });
    jobs.clear();
    for (size_t g0 = 0; g0 < ukeys.size();) {
      size_t g1 = g0 + 1;
      while (g1 < ukeys.size() && ukeys[g1].first == ukeys[g0].first) ++g1;
      std::vector<int64_t> dg, og;
      for (size_t k = g0; k < g1; ++k) (is_diag(ukeys[k].second) ? dg : og).push_back(ukeys[k].second);
      const int c = (int)ukeys[g0].first.size();
      const int np = std::max(1, (c + kTileCap - 1) / kTileCap);
      if (np > 32) return false;
      size_t oi = 0;
      auto add = [&](std::vector<int64_t> us, int diag) {
        for (int k = 0; k < np; ++k) {
          Job J;
          J.diag = diag;
          J.units = us;
          J.t0 = (int)((int64_t)c * k / np);
          J.t1 = (int)((int64_t)c * (k + 1) / np);
          J.part = k;
          J.nparts = np;
          J.els = &ukeys[g0].first;
          jobs.push_back(J);
        }
      };
      for (int64_t d : dg) {
        std::vector<int64_t> us{d};
        while (us.size() < (size_t)kTileKU && oi < og.size()) us.push_back(og[oi++]);
        add(us, 1);
      }
      while (oi < og.size()) {
        std::vector<int64_t> us;
        while (us.size() < (size_t)kTileKU && oi < og.size()) us.push_back(og[oi++]);
        add(us, 0);
      }
      g0 = g1;
    }
    // lane jobs in (diagonal, units, steps, elements) order; the parts of a job stay adjacent
    std::vector<int> heads;
    for (int k = 0; k < (int)jobs.size(); ++k)
      if (jobs[k].part == 0) heads.push_back(k);
    std::stable_sort(heads.begin(), heads.end(), [&](int x, int y) {
      const Job &X = jobs[x], &Y = jobs[y];
      if (X.diag != Y.diag) return X.diag > Y.diag;
      if (X.units.size() != Y.units.size()) return X.units.size() > Y.units.size();
      if (X.els->size() != Y.els->size()) return X.els->size() > Y.els->size();
      return *X.els < *Y.els;
    });
    items.clear();
    {
      Item cur;
      auto flush = [&]() {
        if (cur.job.empty()) return;
        while (cur.job.size() < 32) cur.job.push_back(-1);
        items.push_back(cur);
        cur = Item();
      };
      for (int hd : heads) {
        const int np = jobs[hd].nparts;
        if (cur.job.size() + np > 32 || (!cur.job.empty() && (jobs[cur.job[0]].diag != jobs[hd].diag ||
                                                              (int)jobs[hd].units.size() != cur.nu)))
          flush();
        if (cur.job.empty()) {
          cur.diag = jobs[hd].diag;
          cur.nu = (int)jobs[hd].units.size();
        }
        for (int k = 0; k < np; ++k) {
          cur.job.push_back(hd + k);
          cur.steps = std::max(cur.steps, jobs[hd + k].t1 - jobs[hd + k].t0);
        }
        cur.maxpart = std::max(cur.maxpart, np);
      }
      flush();
    }
    // items longest first (the kernel hands them out through a shared ticket)
    std::vector<int> ord(items.size());
    std::iota(ord.begin(), ord.end(), 0);
    auto cost = [&](int k) { return items[k].steps * (items[k].nu + 1) + (items[k].diag ? 2 : 0); };
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost(a) > cost(b); });
    for (int it : ord) {
      const Item& I = items[it];
      if (ent.size() + 32 * (size_t)I.steps >= (size_t(1) << 31)) return false;
      w_ent.push_back((int32_t)ent.size());
      w_info.push_back(I.steps | I.diag << 16 | (I.maxpart - 1) << 17 | I.nu << 24);
      const size_t base = ent.size();
      ent.resize(base + 32 * (size_t)I.steps, ~0ull);
      const size_t mbase = l_off.size();
      l_off.resize(mbase + 32 * kTileKU, -1);
      l_aux.resize(mbase + 32 * kTileKU, -1);
      l_deg.resize(mbase + 32 * kTileKU, 0);
      l_m.resize(mbase + 32 * kTileKU, 0.0);
      for (int l = 0; l < 32; ++l) {
        const int jb = I.job[l];
        if (jb < 0) {
          l_lane.push_back(-1);
          continue;
        }
        const Job& J = jobs[jb];
        l_lane.push_back(J.part | J.diag << 8);
        for (int t = J.t0; t < J.t1; ++t) {
          const int32_t e = (*J.els)[t];
          uint64_t en = (uint64_t)slot_of[e];
          for (int j = 0; j < kTileKU; ++j) {
            uint64_t ab = 0xff;
            if (j < (int)J.units.size()) {
              // the unit's block (a, b) in element e: blk_ent entries ascend in e
              const int32_t p = unit_p[J.units[j]];
              const uint32_t* be = &blk_ent[blk_ptr[p]];
              ab = be[t] & 0xff;
              if ((int32_t)(be[t] >> 8) != e) return false;
            }
            en |= ab << (8 + 8 * j);
          }
          for (int j = (int)J.units.size(); j < kTileKU; ++j) en |= 0xffull << (8 + 8 * j);
          ent[base + 32 * (size_t)(t - J.t0) + l] = en;
        }
        if (J.part == 0)
          for (int j = 0; j < (int)J.units.size(); ++j) {
            const int64_t u = J.units[j];
            const int32_t p = unit_p[u];
            const size_t mi = mbase + (size_t)j * 32 + l;
            l_off[mi] = u_off[u];
            l_aux[mi] = (J.diag && j == 0) ? blk_row[p] : u_offT[u];
            l_deg[mi] = u_deg[u];
            l_m[mi] = u_m[u];
          }
      }
    }
    t_warp_ptr.push_back((int32_t)w_ent.size());
    for (int32_t e : els) slot_of[e] = -1;
    clear_nodes(rows, n);
    return true;
  };
  // walk the aligned 4x4x4 Morton blocks
  for (int64_t k0 = 0; k0 < n_own;) {
    int64_t k1 = k0 + 1;
    while (k1 < n_own && (code[order[k1]] >> 6) == (code[order[k0]] >> 6)) ++k1;
    stack.push_back({k0, k1});
    while (!stack.empty()) {
      const auto r = stack.back();
      stack.pop_back();
      elements_of(order.data() + r.first, r.second - r.first);
      const int64_t nn = nodes_of(order.data() + r.first, r.second - r.first);
      if ((int64_t)els.size() > kTileMaxEl || nn > kTileMaxNode || r.second - r.first > kTileMaxOwn) {
        clear_nodes(order.data() + r.first, r.second - r.first);
        if (r.second - r.first < 2) return TLFEA_OK;  // one node touches too many elements: keep two kernels
        const int64_t mid = (r.first + r.second) / 2;
        stack.push_back({mid, r.second});
        stack.push_back({r.first, mid});
        continue;
      }
      if (!emit(order.data() + r.first, r.second - r.first)) return TLFEA_OK;
    }
    k0 = k1;
  }
  ent.resize(ent.size() + 32, ~0ull);  // item_load reads a lane's first step unconditionally
  const int64_t nt = (int64_t)t_rec_ptr.size() - 1;
  if (nt >= (int64_t(1) << 31) || (int64_t)w_ent.size() * 32 * kTileKU >= (int64_t(1) << 31)) return TLFEA_OK;
  TL_TRY(h2d(c, &c->t_rec_ptr, t_rec_ptr));
  TL_TRY(h2d(c, &c->t_rec, t_rec));
  TL_TRY(h2d(c, &c->t_node_ptr, t_node_ptr));
  TL_TRY(h2d(c, &c->t_node, t_node));
  TL_TRY(h2d(c, &c->t_warp_ptr, t_warp_ptr));
  TL_TRY(h2d(c, &c->w_ent, w_ent));
  TL_TRY(h2d(c, &c->w_info, w_info));
  TL_TRY(h2d(c, &c->t_ent, ent));
  TL_TRY(h2d(c, &c->l_lane, l_lane));
  TL_TRY(h2d(c, &c->l_off, l_off));
  TL_TRY(h2d(c, &c->l_aux, l_aux));
  TL_TRY(h2d(c, &c->l_deg, l_deg));
  TL_TRY(h2d(c, &c->l_m, l_m));
  c->n_tiles = nt;
  c->n_tile_visits = (int64_t)t_rec.size() / 12;
  return TLFEA_OK;
}

}  // namespace tlfea
