// setup.cu — tlfea_setup: a-1 reference precompute and a-2 fixed-sparsity
// pattern / slot map / mass / f_ff, on the device (§4.1-4.2,
// P:278-379).
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "material.cuh"
#include "shape.cuh"

namespace tlfea {

// ------------------------------------------------------------ error plumbing
static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
tlfea_status fail(tlfea_status st, const std::string& msg) {
  g_err = msg;
  return st;
}
void count_launch(int n) { g_launches += n; }

// Shared-memory carveout (TLFEA_CARVEOUT, percent; -1 = the driver's choice,
// the default). On some boxes of the pool the driver's choice for the T10 SVK
// tangent groups (3 CTAs x ~50 KB per SM) fits only 2 of them: config 3
// element kernel 10.4-10.6 ms instead of ~9.97 ms, where a forced 75 / 100 %
// restored 9.97 ms on such a box. A forced 100 % was not a robust fix: it cost
// the lane-per-point force kernels up to 40 % (200x200 ANCF force only 0.214
// vs 0.154 ms), the beam / Mooney-Rivlin tangent kernels 1-2 %, and on
// another box the curved-mesh T10 group 10.57 vs 10.02 ms; sizing it to the
// register-limited CTA count rounded to too small a configuration (16 ms).
// Left at the driver's choice; recorded as an open item.
#ifndef TLFEA_CARVEOUT
#define TLFEA_CARVEOUT -1
#endif
tlfea_status ensure_dynamic_smem(const void* kernel, size_t bytes, int block_threads) {
  // (set even below 48 KB: static + dynamic above 48 KB needs the opt-in too)
  (void)block_threads;
  if (bytes == 0) return TLFEA_OK;
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> applied;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = applied[{kernel, dev}];
  if (bytes > have) {
    TL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
  return TLFEA_OK;
}
tlfea_status ensure_carveout(const void* kernel) {
  if (TLFEA_CARVEOUT < 0) return TLFEA_OK;
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  bool& d = done[{kernel, dev}];
  if (!d) {
    TL_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, TLFEA_CARVEOUT));
    d = true;
  }
  return TLFEA_OK;
}
const char* last_error() { return g_err.c_str(); }
int64_t launch_count() { return g_launches.load(); }

Context::~Context() {
  nccl_detach(this);
  for (auto& t : timed) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  for (auto& ev : event_pool) cudaEventDestroy(ev);
  for (auto& b : owned) cudaFree(b.p);
}

MatDev make_matdev(const tlfea_material& m) {
  MatDev d{};
  d.model = m.model;
  d.lam = m.E * m.nu / ((1.0 + m.nu) * (1.0 - 2.0 * m.nu));
  d.mu = m.E / (2.0 * (1.0 + m.nu));
  d.C10 = m.C10;
  d.C01 = m.C01;
  d.kappa = m.kappa;
  d.eta = m.eta_damp;
  d.lamd = m.lambda_damp;
  d.kv = (m.eta_damp != 0.0 || m.lambda_damp != 0.0) ? 1 : 0;
  d.rho0 = m.rho0;
  return d;
}

// Temporary device storage for CUB calls (freed on scope exit)
struct Tmp {
  void* p = nullptr;
  size_t bytes = 0;
  ~Tmp() {
    if (p) cudaFree(p);
  }
  tlfea_status get(size_t b) {
    if (b <= bytes) return TLFEA_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t err = cudaMalloc(&p, b ? b : 8);
    if (err != cudaSuccess) {
      cudaGetLastError();
      return fail(TLFEA_E_OOM, "temporary cudaMalloc failed");
    }
    bytes = b;
    return TLFEA_OK;
  }
};

template <class T>
struct TmpArr {
  T* p = nullptr;
  ~TmpArr() {
    if (p) cudaFree(p);
  }
  tlfea_status get(size_t n) {
    cudaError_t err = cudaMalloc(&p, (n ? n : 1) * sizeof(T));
    if (err != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(TLFEA_E_OOM, "temporary cudaMalloc of " + std::to_string(n * sizeof(T)) + " B failed");
    }
    return TLFEA_OK;
  }
};

static inline unsigned grid_for(int64_t n, int block) {
  return (unsigned)std::max<int64_t>(1, (n + block - 1) / block);
}

// ----------------------------------------------------------------- kernels

// a-1: per (e,q): J = sum_a X_a (x) dN_a/dxi, J0 = det J, grad_X N = dN/dxi J^{-1}
// (P:312-320). One thread per (e,q).
__global__ void k_precompute(int element, int64_t n_el, int nq, int nen, const int32_t* __restrict__ conn,
                             const double* __restrict__ X, const double* __restrict__ dims,
                             const double* __restrict__ qxi, const double* __restrict__ qw,
                             double* __restrict__ gradN, double* __restrict__ J0w,
                             unsigned long long* __restrict__ bad, double* __restrict__ jinv = nullptr) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_el * nq) return;
  const int64_t e = t / nq;
  const int q = (int)(t % nq);
  double dN[16][3];
  const double xi[3] = {qxi[3 * q], qxi[3 * q + 1], qxi[3 * q + 2]};
  if (element == TLFEA_T10) {
    t10_shape(xi, nullptr, dN);
  } else if (element == TLFEA_ANCF3443) {
    ancf_shape(xi, dims + 3 * e, nullptr, dN);
  } else {
    beam_shape(xi, dims + 3 * e, nullptr, dN);
  }
  // J = sum_a (X_a - X_o) (x) dN_a/dxi over position coefficients (sum_a dN_a = 0
  // for them), so the element's absolute placement does not enter the rounding:
  // congruent elements get (nearly) bit-identical tables.
  const int64_t Io = conn[e * nen];
  const double o0 = X[3 * Io], o1 = X[3 * Io + 1], o2 = X[3 * Io + 2];
  double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int a = 0; a < nen; ++a) {
    const int64_t I = conn[e * nen + a];
    const bool pos = element == TLFEA_T10 || (a & 3) == 0;
    const double x0 = X[3 * I] - (pos ? o0 : 0.0), x1 = X[3 * I + 1] - (pos ? o1 : 0.0),
                 x2 = X[3 * I + 2] - (pos ? o2 : 0.0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      J[k] += x0 * dN[a][k];
      J[3 + k] += x1 * dN[a][k];
      J[6 + k] += x2 * dN[a][k];
    }
  }
  const double det = det3(J);
  if (!(det > 0.0)) atomicMin(bad, (unsigned long long)e);
  const double r = 1.0 / det;
  double Ji[9];
  Ji[0] = (J[4] * J[8] - J[5] * J[7]) * r;
  Ji[1] = (J[2] * J[7] - J[1] * J[8]) * r;
  Ji[2] = (J[1] * J[5] - J[2] * J[4]) * r;
  Ji[3] = (J[5] * J[6] - J[3] * J[8]) * r;
  Ji[4] = (J[0] * J[8] - J[2] * J[6]) * r;
  Ji[5] = (J[2] * J[3] - J[0] * J[5]) * r;
  Ji[6] = (J[3] * J[7] - J[4] * J[6]) * r;
  Ji[7] = (J[1] * J[6] - J[0] * J[7]) * r;
  Ji[8] = (J[0] * J[4] - J[1] * J[3]) * r;
  double* out = gradN + t * nen * 3;
  for (int a = 0; a < nen; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      out[3 * a + k] = dN[a][0] * Ji[k] + dN[a][1] * Ji[3 + k] + dN[a][2] * Ji[6 + k];
  J0w[t] = det * qw[q];
  if (jinv) {  // the compressed curved-T10 layout: J^-1 (9) and J0 w_q per (e,q)
#pragma unroll
    for (int r = 0; r < 9; ++r) jinv[10 * t + r] = Ji[r];
    jinv[10 * t + 9] = det * qw[q];
  }
}

// Straight-sided T10 test: every mid-edge node at the midpoint of its edge.
__global__ void k_affine_check(int64_t n_el, const int32_t* __restrict__ conn,
                               const double* __restrict__ X, unsigned int* __restrict__ nonaffine) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  const int ea[6] = {0, 1, 2, 0, 1, 2}, eb[6] = {1, 2, 0, 3, 3, 3};
  const int32_t* c = conn + e * 10;
  double h = 0.0, dev = 0.0;
  for (int m = 0; m < 6; ++m)
    for (int k = 0; k < 3; ++k) {
      const double xa = X[3 * (int64_t)c[ea[m]] + k], xb = X[3 * (int64_t)c[eb[m]] + k];
      h = fmax(h, fabs(xa - xb));
      dev = fmax(dev, fabs(X[3 * (int64_t)c[4 + m] + k] - 0.5 * (xa + xb)));
    }
  if (dev > 1e-12 * h) atomicOr(nonaffine, 1u);
}

// Affine (min) layout of a straight-sided T10 (P:312-320 with J constant):
// J = [X1 - X0, X2 - X0, X3 - X0] (columns dX/dxi_c), grad_X z_{c+1} = row c
// of J^-1, grad_X z_0 = -(sum of the others), J0 = det J.
// idx (optional): output row r is element idx[r] (the per-class rows of a
// mesh with geometry classes), else element r.
__global__ void k_affine_layout(int64_t n_el, const int32_t* __restrict__ conn, const double* __restrict__ X,
                                double* __restrict__ aff, const int64_t* __restrict__ idx = nullptr) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  const int32_t* c = conn + (idx ? idx[e] : e) * 10;
  double J[3][3];
  for (int k = 0; k < 3; ++k)
    for (int m = 0; m < 3; ++m) J[k][m] = X[3 * (int64_t)c[m + 1] + k] - X[3 * (int64_t)c[0] + k];
  const double A00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], A01 = J[1][2] * J[2][0] - J[1][0] * J[2][2],
               A02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * A00 + J[0][1] * A01 + J[0][2] * A02;
  const double r = 1.0 / det;
  // inverse: Ji[m][k] = cofactor(k, m) / det
  double Ji[3][3];
  Ji[0][0] = A00 * r;
  Ji[1][0] = A01 * r;
  Ji[2][0] = A02 * r;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
  double* a = aff + 13 * e;
  for (int k = 0; k < 3; ++k) {
    a[3 + k] = Ji[0][k];
    a[6 + k] = Ji[1][k];
    a[9 + k] = Ji[2][k];
    a[k] = -(Ji[0][k] + Ji[1][k] + Ji[2][k]);
  }
  a[12] = det;
}

// Pattern keys: (owned row << 32) | column for every element-local pair whose
// row is owned; non-owned pairs get the sentinel ~0.
__global__ void k_keys(int64_t n_el, int nen, const int32_t* __restrict__ conn,
                       const int32_t* __restrict__ own_idx, unsigned long long* __restrict__ keys) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nen * nen;
  if (t >= n_el * per) return;
  const int64_t e = t / per;
  const int ab = (int)(t % per), a = ab / nen, b = ab % nen;
  const int32_t I = conn[e * nen + a], J = conn[e * nen + b];
  const int32_t r = own_idx[I];
  keys[t] = r >= 0 ? (((unsigned long long)r << 32) | (unsigned)J) : ~0ull;
}

__global__ void k_split_keys(int64_t nnz, const unsigned long long* __restrict__ keys,
                             int32_t* __restrict__ cols, int32_t* __restrict__ row,
                             int32_t* __restrict__ cnt) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int32_t r = (int32_t)(keys[p] >> 32);
  cols[p] = (int32_t)(keys[p] & 0xffffffffu);
  row[p] = r;
  atomicAdd(cnt + r, 1);
}

// DOF lift: row 3i+d holds 3J+e for the sorted coefficient columns J.
// DOF-level positions are 64-bit: H may hold 2^31 or more values (reading Q17)
__global__ void k_lift(int64_t n_own, int64_t nnz_c, const int32_t* __restrict__ rowptr_c,
                       const int32_t* __restrict__ cols_c, const int32_t* __restrict__ blk_row,
                       int64_t* __restrict__ rowptr, int32_t* __restrict__ cols) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n_own) {
    const int64_t b = rowptr_c[p], deg = rowptr_c[p + 1] - b;
    for (int d = 0; d < 3; ++d) rowptr[3 * p + d] = 9 * b + 3 * d * deg;
    if (p == n_own - 1) rowptr[3 * n_own] = 9 * nnz_c;
  }
  if (p >= nnz_c) return;
  const int64_t i = blk_row[p], b = rowptr_c[i], deg = rowptr_c[i + 1] - b, k = p - b;
  const int32_t J = cols_c[p];
  for (int d = 0; d < 3; ++d)
    for (int e = 0; e < 3; ++e) cols[9 * b + 3 * d * deg + 3 * k + e] = 3 * J + e;
}

// UPPER H storage (NEXT-4). Rank of the diagonal block in coefficient row i
// (global coefficient I = own_nodes[i]) = number of columns J < I.
__device__ __forceinline__ int32_t diag_rank(const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ cols_c,
                                             int32_t i, int32_t I) {
  int32_t lo = rowptr_c[i], hi = rowptr_c[i + 1];
  const int32_t b = lo;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cols_c[mid] < I) lo = mid + 1;
    else hi = mid;
  }
  return lo - b;
}

// values of coefficient row i in UPPER storage: 6 (diagonal block, f >= d) + 9 L
__global__ void k_upper_count(int64_t n_own, const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ cols_c,
                              const int32_t* __restrict__ own_nodes, int32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_own) return;
  const int32_t deg = rowptr_c[i + 1] - rowptr_c[i];
  const int32_t L = deg - diag_rank(rowptr_c, cols_c, (int32_t)i, own_nodes[i]) - 1;
  cnt[i] = 6 + 9 * L;
}

__host__ __device__ __forceinline__ int64_t upper_pos(int32_t base, int32_t k, int32_t L, int d, int f) {
  return (int64_t)base + 3 * k + f + d * (2 + 3 * L) - d * (d - 1) / 2;
}

__global__ void k_lift_upper(int64_t n_own, int64_t nnz_c, const int32_t* __restrict__ rowptr_c,
                             const int32_t* __restrict__ cols_c, const int32_t* __restrict__ blk_row,
                             const int32_t* __restrict__ own_nodes, const int32_t* __restrict__ ubase,
                             int64_t* __restrict__ rowptr, int32_t* __restrict__ cols) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n_own) {
    const int32_t deg = rowptr_c[p + 1] - rowptr_c[p];
    const int32_t L = deg - diag_rank(rowptr_c, cols_c, (int32_t)p, own_nodes[p]) - 1;
    for (int d = 0; d < 3; ++d) rowptr[3 * p + d] = ubase[p] + d * (3 + 3 * L) - d * (d - 1) / 2;
    if (p == n_own - 1) rowptr[3 * n_own] = ubase[n_own];
  }
  if (p >= nnz_c) return;
  const int32_t i = blk_row[p], b = rowptr_c[i], deg = rowptr_c[i + 1] - b;
  const int32_t kd = diag_rank(rowptr_c, cols_c, i, own_nodes[i]);
  const int32_t k = (int32_t)p - b - kd;  // rank among J >= I
  if (k < 0) return;                      // lower block: not stored
  const int32_t L = deg - kd - 1, J = cols_c[p];
  for (int d = 0; d < 3; ++d)
    for (int f = (k == 0 ? d : 0); f < 3; ++f) cols[upper_pos(ubase[i], k, L, d, f)] = 3 * J + f;
}

__device__ __forceinline__ int32_t find_in_row(const int32_t* __restrict__ rowptr_c,
                                               const int32_t* __restrict__ cols_c, int32_t r,
                                               int32_t J) {
  int32_t lo = rowptr_c[r], hi = rowptr_c[r + 1];
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cols_c[mid] < J)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Coefficient-level slot map of local elements + contribution pairs for the
// H gather (key = slot, value = packed (e,a,b); invalid -> INT_MAX).
__global__ void k_slots(int64_t n_el, int nen, const int32_t* __restrict__ conn,
                        const int32_t* __restrict__ own_idx, const int32_t* __restrict__ rowptr_c,
                        const int32_t* __restrict__ cols_c, int32_t* __restrict__ slot,
                        int32_t* __restrict__ pkey, uint32_t* __restrict__ pval) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nen * nen;
  if (t >= n_el * per) return;
  const int64_t e = t / per;
  const int ab = (int)(t % per), a = ab / nen, b = ab % nen;
  const int32_t r = own_idx[conn[e * nen + a]];
  int32_t s = -1;
  if (r >= 0) s = find_in_row(rowptr_c, cols_c, r, conn[e * nen + b]);
  slot[t] = s;
  if (pkey) {
    pkey[t] = s >= 0 ? s : 0x7fffffff;
    pval[t] = pack_eab((uint32_t)e, (uint32_t)a, (uint32_t)b);
  }
}

__global__ void k_node_pairs(int64_t n_el, int nen, const int32_t* __restrict__ conn,
                             const int32_t* __restrict__ own_idx, int32_t* __restrict__ key,
                             uint32_t* __restrict__ val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_el * nen) return;
  const int64_t e = t / nen;
  const int a = (int)(t % nen);
  const int32_t r = own_idx[conn[t]];
  key[t] = r >= 0 ? r : 0x7fffffff;
  val[t] = ((uint32_t)e << 4) | (uint32_t)a;
}

__global__ void k_count(int64_t n, const int32_t* __restrict__ key, int32_t limit,
                        int32_t* __restrict__ cnt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t k = key[t];
  if (k < limit) atomicAdd(cnt + k, 1);
}

// Element mass m_ab = sum_q rho0 N_a N_b J w for the elements in
// `conn` (setup elements); output me [n][nen][nen].
__global__ void k_element_mass(int element, int64_t n_el, int nen, int nq, const int32_t* __restrict__ conn,
                               const double* __restrict__ X, const double* __restrict__ dims,
                               const double* __restrict__ qxi, const double* __restrict__ qw,
                               double rho, double* __restrict__ me) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  double* m = me + e * nen * nen;
  for (int r = 0; r < nen * nen; ++r) m[r] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double N[16], dN[16][3];
    const double xi[3] = {qxi[3 * q], qxi[3 * q + 1], qxi[3 * q + 2]};
    if (element == TLFEA_T10)
      t10_shape(xi, N, dN);
    else if (element == TLFEA_ANCF3443)
      ancf_shape(xi, dims + 3 * e, N, dN);
    else
      beam_shape(xi, dims + 3 * e, N, dN);
    double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int a = 0; a < nen; ++a) {
      const int64_t I = conn[e * nen + a];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) J[3 * i + k] += X[3 * I + i] * dN[a][k];
    }
    const double wq = rho * det3(J) * qw[q];
    for (int a = 0; a < nen; ++a)
      for (int b = 0; b < nen; ++b) m[a * nen + b] += wq * N[a] * N[b];
  }
}

// Setup-element contribution pairs for the mass gather.
__global__ void k_mass_pairs(int64_t n_el, int nen, const int32_t* __restrict__ conn,
                             const int32_t* __restrict__ own_idx, const int32_t* __restrict__ rowptr_c,
                             const int32_t* __restrict__ cols_c, int32_t* __restrict__ key,
                             int64_t* __restrict__ val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nen * nen;
  if (t >= n_el * per) return;
  const int64_t e = t / per;
  const int ab = (int)(t % per), a = ab / nen, b = ab % nen;
  const int32_t r = own_idx[conn[e * nen + a]];
  key[t] = r >= 0 ? find_in_row(rowptr_c, cols_c, r, conn[e * nen + b]) : 0x7fffffff;
  val[t] = t;
}

// M_IJ = sum of the element mass entries of block (I,J) in element order.
// cls != nullptr: congruent elements share their class's mass matrix
// (me then holds one nen x nen matrix per class).
__global__ void k_mass_gather(int64_t nnz_c, const int32_t* __restrict__ ptr,
                              const int64_t* __restrict__ ent, const double* __restrict__ me,
                              const uint8_t* __restrict__ cls, int nen2, double* __restrict__ M) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz_c) return;
  double s = 0.0;
  for (int32_t k = ptr[p]; k < ptr[p + 1]; ++k) {
    const int64_t t = ent[k];
    s += cls ? me[(int64_t)cls[t / nen2] * nen2 + t % nen2] : me[t];
  }
  M[p] = s;
}

__global__ void k_force_field(int64_t n_own, const int32_t* __restrict__ rowptr_c,
                              const double* __restrict__ M, double g0, double g1, double g2,
                              double* __restrict__ fff) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_own) return;
  double s = 0.0;
  for (int32_t p = rowptr_c[i]; p < rowptr_c[i + 1]; ++p) s += M[p];
  fff[3 * i] = g0 * s;
  fff[3 * i + 1] = g1 * s;
  fff[3 * i + 2] = g2 * s;
}

// Geometry classes: hash of an element's reference table (gradN, J0w)
// quantised at ~2^-36 of its largest entry. Congruent (translated) elements
// hash equal; every member is validated against its class representative.
__global__ void k_geom_hash(int64_t n_el, int len_g, int len_w, const double* __restrict__ gradN,
                            const double* __restrict__ J0w, unsigned long long* __restrict__ key,
                            int64_t* __restrict__ idx) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  const double* g = gradN + e * len_g;
  const double* w = J0w + e * len_w;
  double sg = 0.0, sw = 0.0;
  for (int i = 0; i < len_g; ++i) sg = fmax(sg, fabs(g[i]));
  for (int i = 0; i < len_w; ++i) sw = fmax(sw, fabs(w[i]));
  unsigned long long h = 1469598103934665603ull;
  auto mix = [&](double v, double s) {
    // coarse (2^-20 relative) so rounding-level differences between congruent
    // elements almost never straddle a bucket; exactness is checked afterwards
    const long long qv = s > 0.0 ? llrint(v / s * 1048576.0) : 0;
    h = (h ^ (unsigned long long)qv) * 1099511628211ull;
  };
  for (int i = 0; i < len_g; ++i) mix(g[i], sg);
  for (int i = 0; i < len_w; ++i) mix(w[i], sw);
  key[e] = h >> 1;  // keep clear of the all-ones sentinel
  idx[e] = e;
}

// cls_of_sorted: class id per sorted position (run index); rep = first e of the run.
__global__ void k_geom_assign(int64_t n, const unsigned long long* __restrict__ skey,
                              const int64_t* __restrict__ sidx, const int32_t* __restrict__ run_id,
                              uint8_t* __restrict__ cls) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  cls[sidx[t]] = (uint8_t)run_id[t];
}

__global__ void k_run_flags(int64_t n, const unsigned long long* __restrict__ skey, int32_t* __restrict__ flag) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  flag[t] = (t == 0 || skey[t] != skey[t - 1]) ? 1 : 0;
}

// An element joins its class when its own tables match the class tables to
// 1e-12 relative, or to the rounding floor of its own table, ~ 16 eps
// |X_o| / h_e (J is formed from coordinates of magnitude |X_o| over an element
// of size h_e = V_e^(1/3); e.g. a 2 km beam chain of 0.2 m elements).
__global__ void k_geom_validate(int64_t n_el, int len, const double* __restrict__ gradN,
                                const double* __restrict__ J0w, int nq, const uint8_t* __restrict__ cls,
                                const double* __restrict__ tab, const int32_t* __restrict__ conn, int nen,
                                const double* __restrict__ X, unsigned int* __restrict__ bad) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_el) return;
  double vol = 0.0;
  for (int q = 0; q < nq; ++q) vol += J0w[e * nq + q];
  const int64_t Io = conn[e * nen];
  const double xo = fmax(fabs(X[3 * Io]), fmax(fabs(X[3 * Io + 1]), fabs(X[3 * Io + 2])));
  const double tol = fmax(1e-12, 16.0 * 2.220446049250313e-16 * xo / cbrt(fabs(vol)));
  const int lg = len - nq;
  const double* t = tab + (int64_t)cls[e] * len;  // len = nq * (per + 1) per class
  // table layout per class: [q][lg/nq gradN entries ..., J0w]
  const int per = lg / nq;
  double sg = 0.0, dg = 0.0, sw = 0.0, dw = 0.0;
  for (int q = 0; q < nq; ++q) {
    for (int i = 0; i < per; ++i) {
      const double a = gradN[(e * nq + q) * per + i], b = t[q * (per + 1) + i];
      sg = fmax(sg, fabs(b));
      dg = fmax(dg, fabs(a - b));
    }
    const double a = J0w[e * nq + q], b = t[q * (per + 1) + per];
    sw = fmax(sw, fabs(b));
    dw = fmax(dw, fabs(a - b));
  }
  if (dg > tol * sg || dw > tol * sw) atomicOr(bad, 1u);
}

__global__ void k_geom_gather_rep(int n_cls, int nq, int per, const int64_t* __restrict__ rep,
                                  const double* __restrict__ gradN, const double* __restrict__ J0w,
                                  double* __restrict__ tab) {
  const int c = blockIdx.x;
  if (c >= n_cls) return;
  const int64_t e = rep[c];
  for (int t = threadIdx.x; t < nq * (per + 1); t += blockDim.x) {
    const int q = t / (per + 1), i = t % (per + 1);
    tab[(int64_t)c * nq * (per + 1) + t] = i < per ? gradN[(e * nq + q) * per + i] : J0w[e * nq + q];
  }
}

// Symmetric gather units: block p=(I,J) is a unit when I <= J (global ids) or
// when the transpose row J is not owned; pT = position of (J,I) in row J.
__global__ void k_units(int64_t nnz_c, const int32_t* __restrict__ blk_row, const int32_t* __restrict__ cols_c,
                        const int32_t* __restrict__ own_nodes, const int32_t* __restrict__ own_idx,
                        const int32_t* __restrict__ rowptr_c, int32_t* __restrict__ is_unit,
                        int32_t* __restrict__ pT) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz_c) return;
  const int32_t I = own_nodes[blk_row[p]], J = cols_c[p];
  const int32_t rJ = own_idx[J];
  int32_t t = -1;
  if (rJ >= 0 && J != I) {
    int32_t lo = rowptr_c[rJ], hi = rowptr_c[rJ + 1];
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (cols_c[mid] < I)
        lo = mid + 1;
      else
        hi = mid;
    }
    t = lo;
  }
  is_unit[p] = (J >= I || rJ < 0) ? 1 : 0;
  pT[p] = (J > I) ? t : -1;
}

__device__ __forceinline__ int ublk_s(int n, int a, int b) { return a * n - (a * (a - 1)) / 2 + (b - a); }

__global__ void k_unit_len(int64_t n_units, const int32_t* __restrict__ unit_p, const int32_t* __restrict__ blk_ptr,
                           int32_t* __restrict__ len) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int32_t p = unit_p[u];
  len[u] = blk_ptr[p + 1] - blk_ptr[p];
}

// dest[e][ub] = (position in the gather-sorted scratch << 1) | transpose
__global__ void k_unit_dest(int64_t n_units, int nen, int nub, const int32_t* __restrict__ unit_p,
                            const int32_t* __restrict__ unit_ptr, const int32_t* __restrict__ blk_ptr,
                            const uint32_t* __restrict__ blk_ent, int32_t* __restrict__ dest) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int32_t p = unit_p[u], t0 = blk_ptr[p], t1 = blk_ptr[p + 1], base = unit_ptr[u];
  for (int32_t t = t0; t < t1; ++t) {
    const uint32_t en = blk_ent[t];
    const int64_t e = en >> 8;
    const int a = (en >> 4) & 15, b = en & 15;
    const int ub = a <= b ? ublk_s(nen, a, b) : ublk_s(nen, b, a);
    dest[e * nub + ub] = ((base + (t - t0)) << 1) | (a > b ? 1 : 0);
  }
}

__global__ void k_unit_meta(int64_t n_units, const int32_t* __restrict__ unit_p, const int32_t* __restrict__ unit_pT,
                            const int32_t* __restrict__ blk_row, const int32_t* __restrict__ rowptr_c,
                            const double* __restrict__ M, int32_t* __restrict__ u_off, int32_t* __restrict__ u_offT,
                            int32_t* __restrict__ u_deg, double* __restrict__ u_m) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int32_t p = unit_p[u], pT = unit_pT[u];
  const int32_t i = blk_row[p], b0 = rowptr_c[i], deg = rowptr_c[i + 1] - b0;
  // FULL storage: block offsets 9 b0 + 3 k are multiples of 3; kept / 3 so
  // 32 bits address up to 3 x 2^31 H values (the gather multiplies back)
  u_off[u] = 3 * b0 + (p - b0);
  int32_t degT = 0, offT = -1;
  if (pT >= 0) {
    const int32_t j = blk_row[pT], c0 = rowptr_c[j];
    degT = rowptr_c[j + 1] - c0;
    offT = 3 * c0 + (pT - c0);
  }
  u_offT[u] = offT;
  u_deg[u] = deg | (degT << 16);
  u_m[u] = M[p];
}

// UPPER storage: unit (I, J), J >= I, of row i writes block rank k at
// ubase[i] + 3 k; u_deg = L_i | (k == 0) << 16; no transposed copy
__global__ void k_unit_meta_upper(int64_t n_units, const int32_t* __restrict__ unit_p,
                                  const int32_t* __restrict__ blk_row, const int32_t* __restrict__ rowptr_c,
                                  const int32_t* __restrict__ cols_c, const int32_t* __restrict__ own_nodes,
                                  const int32_t* __restrict__ ubase, const double* __restrict__ M,
                                  int32_t* __restrict__ u_off, int32_t* __restrict__ u_offT,
                                  int32_t* __restrict__ u_deg, double* __restrict__ u_m) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int32_t p = unit_p[u], i = blk_row[p], b = rowptr_c[i], deg = rowptr_c[i + 1] - b;
  const int32_t kd = diag_rank(rowptr_c, cols_c, i, own_nodes[i]);
  const int32_t k = p - b - kd, L = deg - kd - 1;
  u_off[u] = ubase[i] + 3 * k;
  u_offT[u] = -1;
  u_deg[u] = L | ((k == 0 ? 1 : 0) << 16);
  u_m[u] = M[p];
}

// Partitioned contexts: element blocks with neither row owned (and forces of
// nodes owned elsewhere) belong to no gather unit / owned node; they get the
// scratch positions after the unit ranges, in element-major order, and are
// read only by the pack kernels (partition.cu).
__global__ void k_neg_flag(int64_t n, const int32_t* __restrict__ arr, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = arr[i] < 0 ? 1 : 0;
}
__global__ void k_assign_rest(int64_t n, int32_t* __restrict__ arr, const int32_t* __restrict__ scan, int32_t base,
                              int shift) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && arr[i] < 0) arr[i] = (base + scan[i]) << shift;
}

__global__ void k_force_dest(int64_t n, int nen, const uint32_t* __restrict__ node_ent, int32_t* __restrict__ fdest) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t en = node_ent[t];
  fdest[(int64_t)(en >> 4) * nen + (en & 15)] = (int32_t)t;
}

// ------------------------------------------------------------- host helpers

// Sort (key,value) pairs stably by key, then build a CSR pointer over
// [0, n_seg) and return the number of valid entries (key < n_seg).
template <class V>
static tlfea_status sort_and_ptr(int64_t n, int32_t* key, V* val, int64_t n_seg, int32_t* ptr_out,
                                 V** sorted_val_out, int64_t* n_valid, TmpArr<V>& val_sorted) {
  TmpArr<int32_t> key_sorted;
  TL_TRY(key_sorted.get(n));
  TL_TRY(val_sorted.get(n));
  Tmp tmp;
  size_t bytes = 0;
  int end_bit = 31;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key_sorted.p, val, val_sorted.p, (int64_t)n, 0, end_bit);
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key, key_sorted.p, val, val_sorted.p, (int64_t)n, 0, end_bit));
  count_launch();
  // counts -> exclusive scan
  TmpArr<int32_t> cnt;
  TL_TRY(cnt.get(n_seg + 1));
  TL_CUDA(cudaMemset(cnt.p, 0, (n_seg + 1) * sizeof(int32_t)));
  k_count<<<grid_for(n, 256), 256>>>(n, key_sorted.p, (int32_t)n_seg, cnt.p);
  TL_CHECK_LAUNCH();
  bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, ptr_out, (int64_t)(n_seg + 1));
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, ptr_out, (int64_t)(n_seg + 1)));
  count_launch();
  int32_t nv = 0;
  TL_CUDA(cudaMemcpy(&nv, ptr_out + n_seg, sizeof(int32_t), cudaMemcpyDeviceToHost));
  *n_valid = nv;
  *sorted_val_out = val_sorted.p;
  return TLFEA_OK;
}

static tlfea_status build_geometry_classes(Context* c, const double* dX) {
  const int64_t n = c->n_el;
  const int nq = c->nq, per = c->nen * 3;
  const int max_cls = c->element == TLFEA_T10 ? 32 : 4;
  c->n_cls = 0;
  if (n == 0) return TLFEA_OK;
  if (c->force_tables == 1) return TLFEA_OK;  // options.reference_layout = 1: per-(e,q) tables
  TmpArr<unsigned long long> key, key2;
  TmpArr<int64_t> idx, idx2;
  TmpArr<int32_t> flag, run;
  TL_TRY(key.get(n));
  TL_TRY(key2.get(n));
  TL_TRY(idx.get(n));
  TL_TRY(idx2.get(n));
  TL_TRY(flag.get(n));
  TL_TRY(run.get(n));
  k_geom_hash<<<grid_for(n, 128), 128>>>(n, nq * per, nq, c->gradN, c->J0w, key.p, idx.p);
  TL_CHECK_LAUNCH();
  Tmp tmp;
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, idx.p, idx2.p, (int64_t)n);
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, idx.p, idx2.p, (int64_t)n));
  count_launch();
  k_run_flags<<<grid_for(n, 256), 256>>>(n, key2.p, flag.p);
  TL_CHECK_LAUNCH();
  bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, flag.p, run.p, (int64_t)n);
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, flag.p, run.p, (int64_t)n));
  count_launch();
  int32_t nruns = 0;
  TL_CUDA(cudaMemcpy(&nruns, run.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (nruns > max_cls) return TLFEA_OK;  // unstructured: keep per-element tables
  // representatives: the smallest element id of each run (stable sort)
  std::vector<int32_t> hflag(n);
  std::vector<int64_t> hidx(n);
  TL_CUDA(cudaMemcpy(hflag.data(), flag.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  TL_CUDA(cudaMemcpy(hidx.data(), idx2.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  std::vector<int64_t> rep;
  for (int64_t t = 0; t < n; ++t)
    if (hflag[t]) rep.push_back(hidx[t]);
  // run ids are 1-based from the inclusive scan: shift to 0-based via a decrement kernel-free trick
  std::vector<int32_t> hrun(n);
  TL_CUDA(cudaMemcpy(hrun.data(), run.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  for (auto& r : hrun) r -= 1;
  TL_CUDA(cudaMemcpy(run.p, hrun.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  TL_TRY(c->alloc(&c->cls, (size_t)n));
  k_geom_assign<<<grid_for(n, 256), 256>>>(n, key2.p, idx2.p, run.p, c->cls);
  TL_CHECK_LAUNCH();
  c->cls_rep = rep;
  TmpArr<int64_t> drep;
  TL_TRY(drep.get(rep.size()));
  TL_CUDA(cudaMemcpy(drep.p, rep.data(), sizeof(int64_t) * rep.size(), cudaMemcpyHostToDevice));
  TL_TRY(c->alloc(&c->cls_tab, (size_t)nruns * nq * (per + 1)));
  k_geom_gather_rep<<<nruns, 128>>>(nruns, nq, per, drep.p, c->gradN, c->J0w, c->cls_tab);
  TL_CHECK_LAUNCH();
  unsigned int* dbad = nullptr;
  TL_TRY(c->alloc(&dbad, 1));
  TL_CUDA(cudaMemset(dbad, 0, sizeof(unsigned int)));
  k_geom_validate<<<grid_for(n, 128), 128>>>(n, nq * (per + 1), c->gradN, c->J0w, nq, c->cls, c->cls_tab, c->conn,
                                              c->nen, dX, dbad);
  TL_CHECK_LAUNCH();
  unsigned int hb = 0;
  TL_CUDA(cudaMemcpy(&hb, dbad, sizeof(hb), cudaMemcpyDeviceToHost));
  if (hb == 0) c->n_cls = nruns;
  return TLFEA_OK;
}

static tlfea_status build_units(Context* c) {
  c->n_units = 0;
  if (c->nnz_c == 0) return TLFEA_OK;
  const int64_t n = c->nnz_c;
  TmpArr<int32_t> isu, pT;
  TL_TRY(isu.get(n));
  TL_TRY(pT.get(n));
  k_units<<<grid_for(n, 256), 256>>>(n, c->blk_row, c->cols_c, c->own_nodes, c->own_idx, c->rowptr_c, isu.p, pT.p);
  TL_CHECK_LAUNCH();
  TmpArr<int64_t> nsel;
  TL_TRY(nsel.get(1));
  TmpArr<int32_t> up, upT;
  TL_TRY(up.get(n));
  TL_TRY(upT.get(n));
  Tmp tmp;
  size_t bytes = 0;
  cub::CountingInputIterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, bytes, it, isu.p, up.p, nsel.p, (int64_t)n);
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, isu.p, up.p, nsel.p, (int64_t)n));
  count_launch();
  bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, bytes, pT.p, isu.p, upT.p, nsel.p, (int64_t)n);
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, pT.p, isu.p, upT.p, nsel.p, (int64_t)n));
  count_launch();
  int64_t nu = 0;
  TL_CUDA(cudaMemcpy(&nu, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
  c->n_units = nu;
  TL_TRY(c->alloc(&c->unit_p, (size_t)nu));
  TL_TRY(c->alloc(&c->unit_pT, (size_t)nu));
  TL_CUDA(cudaMemcpy(c->unit_p, up.p, sizeof(int32_t) * nu, cudaMemcpyDeviceToDevice));
  TL_CUDA(cudaMemcpy(c->unit_pT, upT.p, sizeof(int32_t) * nu, cudaMemcpyDeviceToDevice));
  return TLFEA_OK;
}

// Gather-sorted scratch layout (single-rank contexts; the partitioned path
// keeps element-major scratch for its pack lists).
static tlfea_status build_sorted_scratch(Context* c) {
  const int nen = c->nen, nub = n_ublk_of(nen);
  TL_TRY(c->alloc(&c->unit_ptr, (size_t)c->n_units + 1));
  TL_TRY(c->alloc(&c->dest, (size_t)std::max<int64_t>(c->n_el, 1) * nub));
  TL_TRY(c->alloc(&c->fdest, (size_t)std::max<int64_t>(c->n_el, 1) * nen));
  TL_CUDA(cudaMemset(c->dest, 0xff, sizeof(int32_t) * std::max<int64_t>(c->n_el, 1) * nub));
  TmpArr<int32_t> len;
  TL_TRY(len.get(c->n_units + 1));
  TL_CUDA(cudaMemset(len.p, 0, sizeof(int32_t) * (c->n_units + 1)));
  if (c->n_units > 0) {
    k_unit_len<<<grid_for(c->n_units, 256), 256>>>(c->n_units, c->unit_p, c->blk_ptr, len.p);
    TL_CHECK_LAUNCH();
  }
  Tmp tmp;
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.p, c->unit_ptr, (int64_t)(c->n_units + 1));
  TL_TRY(tmp.get(bytes));
  TL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, len.p, c->unit_ptr, (int64_t)(c->n_units + 1)));
  count_launch();
  int32_t npos = 0;
  TL_CUDA(cudaMemcpy(&npos, c->unit_ptr + c->n_units, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if ((int64_t)npos > c->n_el * nub || (c->nranks == 1 && (int64_t)npos != c->n_el * nub))
    return fail(TLFEA_E_CUDA, "internal: gather-sorted scratch covers " + std::to_string(npos) + " of " +
                                  std::to_string(c->n_el * nub) + " element blocks");
  if (c->n_units > 0) {
    k_unit_dest<<<grid_for(c->n_units, 256), 256>>>(c->n_units, nen, nub, c->unit_p, c->unit_ptr, c->blk_ptr,
                                                    c->blk_ent, c->dest);
    TL_CHECK_LAUNCH();
  }
  int32_t nf = 0;
  TL_CUDA(cudaMemcpy(&nf, c->node_ptr + c->n_own, sizeof(int32_t), cudaMemcpyDeviceToHost));
  TL_CUDA(cudaMemset(c->fdest, 0xff, sizeof(int32_t) * std::max<int64_t>(c->n_el, 1) * nen));
  if (nf > 0) {
    k_force_dest<<<grid_for(nf, 256), 256>>>(nf, nen, c->node_ent, c->fdest);
    TL_CHECK_LAUNCH();
  }
  // partitioned contexts: the blocks / forces no owned row receives
  auto rest = [&](int32_t* arr, int64_t n, int32_t base, int shift) -> tlfea_status {
    if (n == 0 || (int64_t)base >= n) return TLFEA_OK;
    TmpArr<int32_t> flag, scan;
    TL_TRY(flag.get(n));
    TL_TRY(scan.get(n));
    k_neg_flag<<<grid_for(n, 256), 256>>>(n, arr, flag.p);
    TL_CHECK_LAUNCH();
    Tmp t2;
    size_t b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b2, flag.p, scan.p, n);
    TL_TRY(t2.get(b2));
    TL_CUDA(cub::DeviceScan::ExclusiveSum(t2.p, b2, flag.p, scan.p, n));
    count_launch();
    k_assign_rest<<<grid_for(n, 256), 256>>>(n, arr, scan.p, base, shift);
    TL_CHECK_LAUNCH();
    return TLFEA_OK;
  };
  if (c->nranks > 1) {
    TL_TRY(rest(c->dest, c->n_el * nub, npos, 1));
    TL_TRY(rest(c->fdest, c->n_el * nen, nf, 0));
  }
  return TLFEA_OK;
}

static tlfea_status build_unit_meta(Context* c) {
  if (c->n_units == 0 || !c->unit_ptr) return TLFEA_OK;
  TL_TRY(c->alloc(&c->u_off, (size_t)c->n_units));
  TL_TRY(c->alloc(&c->u_offT, (size_t)c->n_units));
  TL_TRY(c->alloc(&c->u_deg, (size_t)c->n_units));
  TL_TRY(c->alloc(&c->u_m, (size_t)c->n_units));
  if (c->upper) {
    k_unit_meta_upper<<<grid_for(c->n_units, 256), 256>>>(c->n_units, c->unit_p, c->blk_row, c->rowptr_c, c->cols_c,
                                                          c->own_nodes, c->ubase, c->M, c->u_off, c->u_offT,
                                                          c->u_deg, c->u_m);
  } else {
    k_unit_meta<<<grid_for(c->n_units, 256), 256>>>(c->n_units, c->unit_p, c->unit_pT, c->blk_row, c->rowptr_c, c->M,
                                                    c->u_off, c->u_offT, c->u_deg, c->u_m);
  }
  TL_CHECK_LAUNCH();

  return TLFEA_OK;
}

static tlfea_status validate(const tlfea_mesh* mesh, const tlfea_material* mat,
                             const tlfea_options* opts) {
  if (!mesh || !mat || !opts) return fail(TLFEA_E_INVALID, "NULL mesh/material/options");
  if (mesh->element != TLFEA_T10 && mesh->element != TLFEA_ANCF3443 && mesh->element != TLFEA_ANCF3243)
    return fail(TLFEA_E_INVALID, "unknown element type");
  if (mesh->n_elements <= 0 || mesh->n_coef <= 0 || !mesh->conn || !mesh->X_ref)
    return fail(TLFEA_E_INVALID, "empty mesh or NULL conn/X_ref");
  if (mesh->element == TLFEA_T10 &&
      !(opts->quadrature == TLFEA_Q_T10_4PT || opts->quadrature == TLFEA_Q_T10_KEAST5))
    return fail(TLFEA_E_INVALID, "T10 needs quadrature TLFEA_Q_T10_4PT or TLFEA_Q_T10_KEAST5");
  if (mesh->element == TLFEA_ANCF3443 && opts->quadrature != TLFEA_Q_GL_4x4x3)
    return fail(TLFEA_E_INVALID, "ANCF3443 needs quadrature TLFEA_Q_GL_4x4x3");
  if (mesh->element == TLFEA_ANCF3243 && opts->quadrature != TLFEA_Q_GL_3x2x2)
    return fail(TLFEA_E_INVALID, "ANCF3243 needs quadrature TLFEA_Q_GL_3x2x2");
  if (mesh->element != TLFEA_T10 && (mesh->n_coef % 4) != 0)
    return fail(TLFEA_E_INVALID, "ANCF n_coef must be 4 * n_nodes");
  if (mat->model == TLFEA_SVK) {
    if (!(mat->E > 0.0) || !(mat->nu > -1.0 && mat->nu < 0.5))
      return fail(TLFEA_E_INVALID, "SVK needs E > 0 and -1 < nu < 0.5");
  } else if (mat->model == TLFEA_MOONEY_RIVLIN) {
    if (!(mat->C10 >= 0.0) || !(mat->C01 >= 0.0) || !(mat->kappa > 0.0))
      return fail(TLFEA_E_INVALID, "Mooney-Rivlin needs C10, C01 >= 0 and kappa > 0");
  } else {
    return fail(TLFEA_E_INVALID, "unknown material model");
  }
  if (!(mat->rho0 >= 0.0) || !(mat->eta_damp >= 0.0) || !(mat->lambda_damp >= 0.0))
    return fail(TLFEA_E_INVALID, "rho0 and damping must be >= 0");
  if (opts->mass_rule != 0 && opts->mass_rule != 1) return fail(TLFEA_E_INVALID, "mass_rule must be 0 or 1");
  if (opts->nranks < 1 || opts->rank < 0 || opts->rank >= opts->nranks)
    return fail(TLFEA_E_INVALID, "bad rank / nranks");
  if (opts->reference_layout < 0 || opts->reference_layout > 2)
    return fail(TLFEA_E_INVALID, "reference_layout must be 0, 1 or 2");
  if (opts->hessian_upper != 0 && opts->hessian_upper != 1)
    return fail(TLFEA_E_INVALID, "hessian_upper must be 0 or 1");
  if (opts->hessian_upper && (opts->nranks != 1 || (opts->constraints && opts->constraints->m > 0)))
    return fail(TLFEA_E_UNSUPPORTED, "UPPER H storage: single-rank contexts without constraints only");
  if (opts->kv_consistent_tangent != 0 && opts->kv_consistent_tangent != 1)
    return fail(TLFEA_E_INVALID, "kv_consistent_tangent must be 0 or 1");
  if (opts->kv_consistent_tangent && (opts->hessian_upper || opts->nranks != 1))
    return fail(TLFEA_E_UNSUPPORTED,
                "kv_consistent_tangent: the consistent tangent is non-symmetric (FULL storage, single rank)");
  if (mesh->n_elements >= (1ll << 31)) return fail(TLFEA_E_OVERFLOW, "n_elements >= 2^31");
  if (3 * mesh->n_coef >= (1ll << 31)) return fail(TLFEA_E_OVERFLOW, "3 n_coef >= 2^31");
  if (const tlfea_constraints* k = opts->constraints) {
    if (k->m < 0) return fail(TLFEA_E_INVALID, "constraints: m < 0");
    if (k->m > 0) {
      if (opts->nranks != 1) return fail(TLFEA_E_UNSUPPORTED, "constraints: single-rank contexts only");
      if (!k->rowptr || !k->b) return fail(TLFEA_E_INVALID, "constraints: NULL rowptr or b");
      if (k->rowptr[0] != 0) return fail(TLFEA_E_INVALID, "constraints: rowptr[0] != 0");
      for (int64_t r = 0; r < k->m; ++r)
        if (k->rowptr[r + 1] < k->rowptr[r]) return fail(TLFEA_E_INVALID, "constraints: rowptr decreases");
      const int64_t nz = k->rowptr[k->m];
      if (nz >= (1ll << 31)) return fail(TLFEA_E_OVERFLOW, "constraints: nnz >= 2^31");
      if (nz > 0 && (!k->cols || !k->vals)) return fail(TLFEA_E_INVALID, "constraints: NULL cols or vals");
      for (int64_t r = 0; r < k->m; ++r)
        for (int64_t p = k->rowptr[r]; p < k->rowptr[r + 1]; ++p) {
          if (k->cols[p] < 0 || k->cols[p] >= 3 * mesh->n_coef)
            return fail(TLFEA_E_INVALID, "constraints: DOF id out of range in row " + std::to_string(r));
          for (int64_t p2 = k->rowptr[r]; p2 < p; ++p2)
            if (k->cols[p2] == k->cols[p])
              return fail(TLFEA_E_INVALID, "constraints: repeated DOF in row " + std::to_string(r));
        }
    }
  }
  return TLFEA_OK;
}

// Coefficient couplings (I, J) of every constraint row, as pattern keys
// (single rank: owned row = I), ascending and unique.
static std::vector<unsigned long long> constraint_keys(const tlfea_constraints* k) {
  std::vector<unsigned long long> keys;
  if (!k) return keys;
  for (int64_t r = 0; r < k->m; ++r) {
    std::vector<int64_t> coefs;
    for (int64_t p = k->rowptr[r]; p < k->rowptr[r + 1]; ++p) coefs.push_back(k->cols[p] / 3);
    for (int64_t I : coefs)
      for (int64_t J : coefs) keys.push_back(((unsigned long long)I << 32) | (unsigned long long)J);
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  return keys;
}

// DOF slot of each C^T C pair (i << 32 | j) in the final pattern (binary
// search over the coefficient row), written in place.
__global__ void k_gram_slots(int64_t n, const int32_t* __restrict__ rowptr_c, const int32_t* __restrict__ cols_c,
                             int64_t* __restrict__ ij) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = ij[t] >> 32, j = ij[t] & 0xffffffff;
  const int32_t I = (int32_t)(i / 3), J = (int32_t)(j / 3);
  int32_t lo = rowptr_c[I], hi = rowptr_c[I + 1];
  const int32_t b0 = lo, deg = hi - lo;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cols_c[mid] < J) lo = mid + 1;
    else hi = mid;
  }
  ij[t] = 9 * (int64_t)b0 + 3 * (i % 3) * deg + 3 * (int64_t)(lo - b0) + (j % 3);
}

// C, C^T (entries of a DOF row in ascending constraint order) and the
// distinct C^T C pairs with their sums over ascending constraint index.
static tlfea_status setup_constraints(Context* c, const tlfea_constraints* k) {
  if (!k || k->m == 0) return TLFEA_OK;
  const int64_t m = k->m, nz = k->rowptr[m], n_dof = 3 * c->n_coef;
  c->n_con = m;
  std::vector<int32_t> ptr(m + 1), cols(nz), tptr(n_dof + 1, 0), trows(nz);
  std::vector<double> tvals(nz);
  for (int64_t r = 0; r <= m; ++r) ptr[r] = (int32_t)k->rowptr[r];
  for (int64_t p = 0; p < nz; ++p) {
    cols[p] = (int32_t)k->cols[p];
    tptr[cols[p] + 1]++;
  }
  for (int64_t i = 0; i < n_dof; ++i) tptr[i + 1] += tptr[i];
  {
    std::vector<int32_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t r = 0; r < m; ++r)
      for (int64_t p = k->rowptr[r]; p < k->rowptr[r + 1]; ++p) {
        const int32_t q = fill[cols[p]]++;
        trows[q] = (int32_t)r;
        tvals[q] = k->vals[p];
      }
  }
  std::vector<std::pair<int64_t, double>> gram;
  {
    std::vector<std::pair<int64_t, double>> terms;  // (i << 32 | j, C_ki C_kj) in ascending k
    for (int64_t r = 0; r < m; ++r)
      for (int64_t p1 = k->rowptr[r]; p1 < k->rowptr[r + 1]; ++p1)
        for (int64_t p2 = k->rowptr[r]; p2 < k->rowptr[r + 1]; ++p2)
          terms.push_back({(k->cols[p1] << 32) | k->cols[p2], k->vals[p1] * k->vals[p2]});
    std::stable_sort(terms.begin(), terms.end(),
                     [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
                       return a.first < b.first;
                     });
    for (auto& t : terms) {
      if (!gram.empty() && gram.back().first == t.first) gram.back().second += t.second;
      else gram.push_back(t);
    }
  }
  c->n_gram = (int64_t)gram.size();
  std::vector<int64_t> gij(c->n_gram);
  std::vector<double> gval(c->n_gram);
  for (int64_t t = 0; t < c->n_gram; ++t) {
    gij[t] = gram[t].first;
    gval[t] = gram[t].second;
  }
  TL_TRY(c->alloc(&c->con_ptr, (size_t)m + 1));
  TL_TRY(c->alloc(&c->con_cols, (size_t)std::max<int64_t>(nz, 1)));
  TL_TRY(c->alloc(&c->con_vals, (size_t)std::max<int64_t>(nz, 1)));
  TL_TRY(c->alloc(&c->con_b, (size_t)m));
  TL_TRY(c->alloc(&c->con_c, (size_t)m));
  TL_TRY(c->alloc(&c->conT_ptr, (size_t)n_dof + 1));
  TL_TRY(c->alloc(&c->conT_rows, (size_t)std::max<int64_t>(nz, 1)));
  TL_TRY(c->alloc(&c->conT_vals, (size_t)std::max<int64_t>(nz, 1)));
  TL_TRY(c->alloc(&c->gram_ij, (size_t)std::max<int64_t>(c->n_gram, 1)));
  TL_TRY(c->alloc(&c->gram_val, (size_t)std::max<int64_t>(c->n_gram, 1)));
  TL_CUDA(cudaMemcpy(c->con_ptr, ptr.data(), sizeof(int32_t) * (m + 1), cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->con_cols, cols.data(), sizeof(int32_t) * nz, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->con_vals, k->vals, sizeof(double) * nz, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->con_b, k->b, sizeof(double) * m, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->conT_ptr, tptr.data(), sizeof(int32_t) * (n_dof + 1), cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->conT_rows, trows.data(), sizeof(int32_t) * nz, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->conT_vals, tvals.data(), sizeof(double) * nz, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->gram_ij, gij.data(), sizeof(int64_t) * c->n_gram, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(c->gram_val, gval.data(), sizeof(double) * c->n_gram, cudaMemcpyHostToDevice));
  if (c->n_gram > 0) {
    k_gram_slots<<<grid_for(c->n_gram, 256), 256>>>(c->n_gram, c->rowptr_c, c->cols_c, c->gram_ij);
    TL_CHECK_LAUNCH();
  }
  return TLFEA_OK;
}

tlfea_status setup_context(Context* c, const tlfea_mesh* mesh, const tlfea_material* mat,
                           const tlfea_options* opts) {
  TL_TRY(validate(mesh, mat, opts));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(TLFEA_E_CUDA, "no CUDA device available (libtlfea has no CPU fallback)");
  }
  if (opts->device < 0 || opts->device >= ndev) return fail(TLFEA_E_INVALID, "bad device ordinal");
  TL_CUDA(cudaSetDevice(opts->device));
  c->device = opts->device;
  c->element = mesh->element;
  c->quadrature = opts->quadrature;
  c->nen = n_en_of(mesh->element);
  c->nq = n_qp_of(opts->quadrature);
  c->mass_rule = opts->mass_rule;
  c->force_tables = opts->reference_layout;
  c->kvc = opts->kv_consistent_tangent && (mat->eta_damp > 0.0 || mat->lambda_damp > 0.0);
  c->mat_in = *mat;
  c->mat = make_matdev(*mat);
  for (int k = 0; k < 3; ++k) c->gravity[k] = opts->gravity[k];
  c->rank = opts->rank;
  c->nranks = opts->nranks;
  c->n_el_global = mesh->n_elements;
  c->n_coef = mesh->n_coef;
  const int nen = c->nen, nq = c->nq;
  const int npe = n_nodes_of(mesh->element);
  const int64_t NE = mesh->n_elements;

  // ---- host: coefficient connectivity + validation (ids, distinct nodes)
  std::vector<int32_t> cc((size_t)NE * nen);
  for (int64_t e = 0; e < NE; ++e) {
    const int32_t* row = mesh->conn + e * npe;
    for (int a = 0; a < npe; ++a) {
      const int64_t id = row[a];
      const int64_t lim = mesh->element == TLFEA_T10 ? mesh->n_coef : mesh->n_coef / 4;
      if (id < 0 || id >= lim)
        return fail(TLFEA_E_INVALID, "element " + std::to_string(e) + " references node " +
                                         std::to_string(id) + " out of range");
      for (int b = 0; b < a; ++b)
        if (row[b] == row[a])
          return fail(TLFEA_E_INVALID, "element " + std::to_string(e) + " repeats node " + std::to_string(id));
    }
    if (mesh->element == TLFEA_T10) {
      for (int a = 0; a < 10; ++a) cc[e * 10 + a] = row[a];
    } else {
      for (int k = 0; k < npe; ++k)
        for (int m = 0; m < 4; ++m) cc[e * nen + 4 * k + m] = 4 * row[k] + m;
    }
  }
  std::vector<double> dims;
  if (mesh->element != TLFEA_T10) {
    dims.resize((size_t)NE * 3);
    for (int64_t e = 0; e < NE; ++e)
      for (int k = 0; k < 3; ++k) {
        const double d = mesh->ancf_dims ? mesh->ancf_dims[3 * e + k] : opts->ancf_dims[k];
        if (!(d > 0.0)) return fail(TLFEA_E_INVALID, "ANCF element dims must be > 0");
        dims[3 * e + k] = d;
      }
  }

  // ---- host: partition (reading Q20)
  std::vector<int32_t> part((size_t)NE, 0);
  if (c->nranks > 1) {
    for (int64_t e = 0; e < NE; ++e) {
      part[e] = opts->elem_part ? opts->elem_part[e] : (int32_t)((e * c->nranks) / NE);
      if (part[e] < 0 || part[e] >= c->nranks) return fail(TLFEA_E_INVALID, "elem_part out of range");
    }
  }
  std::vector<int32_t> owner((size_t)c->n_coef, c->nranks);
  for (int64_t e = 0; e < NE; ++e)
    for (int a = 0; a < nen; ++a) owner[cc[e * nen + a]] = std::min(owner[cc[e * nen + a]], part[e]);
  for (auto& o : owner)
    if (o == c->nranks) o = 0;  // unreferenced coefficient: owned by rank 0
  std::vector<int32_t> own_idx((size_t)c->n_coef, -1), own_nodes;
  for (int64_t I = 0; I < c->n_coef; ++I)
    if (owner[I] == c->rank) {
      own_idx[I] = (int32_t)own_nodes.size();
      own_nodes.push_back((int32_t)I);
    }
  c->n_own = (int64_t)own_nodes.size();
  std::vector<int64_t> local, setup_el;   // local elements; setup elements (touch an owned row)
  for (int64_t e = 0; e < NE; ++e) {
    if (part[e] == c->rank) local.push_back(e);
    bool touches = false;
    for (int a = 0; a < nen && !touches; ++a) touches = owner[cc[e * nen + a]] == c->rank;
    if (touches) setup_el.push_back(e);
  }
  // partitioned: boundary elements (a node owned elsewhere: they feed the
  // send buffer) first, so tlfea_eval_begin can pack them while the interior
  // elements run next to the exchange; the boundary
  // range is padded to whole element-kernel CTA tiles
  c->n_el_bnd = 0;
  if (c->nranks > 1) {
    std::vector<int64_t> bnd, inner;
    for (int64_t e : local) {
      bool b = false;
      for (int a = 0; a < nen && !b; ++a) b = owner[cc[e * nen + a]] != c->rank;
      (b ? bnd : inner).push_back(e);
    }
    const int64_t tile = el_per_tile(c->element);
    c->n_el_bnd = std::min<int64_t>((int64_t)local.size(), ((int64_t)bnd.size() + tile - 1) / tile * tile);
    local = bnd;
    local.insert(local.end(), inner.begin(), inner.end());
  }
  c->n_el = (int64_t)local.size();
  const int64_t NS = (int64_t)setup_el.size();
  // packed gather entries (e << 8 | a << 4 | b) hold LOCAL element ids
  if (c->n_el >= (1ll << 24))
    return fail(TLFEA_E_OVERFLOW, "more than 2^24 elements on one rank (packed gather entries): partition the mesh "
                                  "over more ranks");

  // ---- uploads
  double* dX = nullptr;
  double* ddims = nullptr;
  TL_TRY(c->alloc(&dX, (size_t)c->n_coef * 3));
  TL_CUDA(cudaMemcpy(dX, mesh->X_ref, sizeof(double) * 3 * c->n_coef, cudaMemcpyHostToDevice));
  std::vector<int32_t> lconn((size_t)std::max<int64_t>(c->n_el, 1) * nen), sconn((size_t)std::max<int64_t>(NS, 1) * nen);
  std::vector<double> ldims, sdims;
  for (int64_t i = 0; i < c->n_el; ++i)
    std::copy(cc.begin() + local[i] * nen, cc.begin() + (local[i] + 1) * nen, lconn.begin() + i * nen);
  for (int64_t i = 0; i < NS; ++i)
    std::copy(cc.begin() + setup_el[i] * nen, cc.begin() + (setup_el[i] + 1) * nen, sconn.begin() + i * nen);
  if (!dims.empty()) {
    ldims.resize((size_t)std::max<int64_t>(c->n_el, 1) * 3);
    sdims.resize((size_t)std::max<int64_t>(NS, 1) * 3);
    for (int64_t i = 0; i < c->n_el; ++i)
      for (int k = 0; k < 3; ++k) ldims[3 * i + k] = dims[3 * local[i] + k];
    for (int64_t i = 0; i < NS; ++i)
      for (int k = 0; k < 3; ++k) sdims[3 * i + k] = dims[3 * setup_el[i] + k];
  }
  TL_TRY(c->alloc(&c->conn, (size_t)c->n_el * nen));
  TL_CUDA(cudaMemcpy(c->conn, lconn.data(), sizeof(int32_t) * c->n_el * nen, cudaMemcpyHostToDevice));
  TL_TRY(c->alloc(&c->elem_gid, (size_t)c->n_el));
  TL_CUDA(cudaMemcpy(c->elem_gid, local.data(), sizeof(int64_t) * c->n_el, cudaMemcpyHostToDevice));
  if (!dims.empty()) {
    TL_TRY(c->alloc(&ddims, ldims.size()));
    TL_CUDA(cudaMemcpy(ddims, ldims.data(), sizeof(double) * ldims.size(), cudaMemcpyHostToDevice));
  }
  TL_TRY(c->alloc(&c->own_nodes, (size_t)c->n_own));
  TL_CUDA(cudaMemcpy(c->own_nodes, own_nodes.data(), sizeof(int32_t) * c->n_own, cudaMemcpyHostToDevice));
  TL_TRY(c->alloc(&c->own_idx, (size_t)c->n_coef));
  TL_CUDA(cudaMemcpy(c->own_idx, own_idx.data(), sizeof(int32_t) * c->n_coef, cudaMemcpyHostToDevice));
  TmpArr<int32_t> dsconn;
  TmpArr<double> dsdims;
  TL_TRY(dsconn.get((size_t)NS * nen));
  TL_CUDA(cudaMemcpy(dsconn.p, sconn.data(), sizeof(int32_t) * NS * nen, cudaMemcpyHostToDevice));
  if (!dims.empty()) {
    TL_TRY(dsdims.get(sdims.size()));
    TL_CUDA(cudaMemcpy(dsdims.p, sdims.data(), sizeof(double) * sdims.size(), cudaMemcpyHostToDevice));
  }

  // ---- a-1 precompute on local elements
  double hq[48 * 3], hw[48];
  const int nrule = make_rule(c->quadrature, hq, hw);
  (void)nrule;
  TmpArr<double> dq, dw;
  TL_TRY(dq.get(3 * 64));
  TL_TRY(dw.get(64));
  TL_CUDA(cudaMemcpy(dq.p, hq, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice));
  TL_CUDA(cudaMemcpy(dw.p, hw, sizeof(double) * nq, cudaMemcpyHostToDevice));
  TL_TRY(c->alloc(&c->gradN, (size_t)c->n_el * nq * nen * 3));
  TL_TRY(c->alloc(&c->J0w, (size_t)c->n_el * nq));
  TL_TRY(c->alloc(&c->err_flag, 2));
  const unsigned long long none = ~0ull;
  TL_CUDA(cudaMemcpy(c->err_flag, &none, sizeof(none), cudaMemcpyHostToDevice));
  if (c->n_el > 0) {
    k_precompute<<<grid_for(c->n_el * nq, 128), 128>>>(c->element, c->n_el, nq, nen, c->conn, dX, ddims,
                                                       dq.p, dw.p, c->gradN, c->J0w, c->err_flag);
    TL_CHECK_LAUNCH();
  }
  unsigned long long bad = 0;
  TL_CUDA(cudaMemcpy(&bad, c->err_flag, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != ~0ull)
    return fail(TLFEA_E_INVERTED_ELEMENT, "inverted element " + std::to_string(local[bad]) +
                                              " (J0 <= 0 at a quadrature point)");
  TL_CUDA(cudaMemcpy(c->err_flag, &none, sizeof(none), cudaMemcpyHostToDevice));
  if (c->element == TLFEA_T10 && c->n_el > 0) {
    unsigned int* dna = nullptr;
    TL_TRY(c->alloc(&dna, 1));
    TL_CUDA(cudaMemset(dna, 0, sizeof(unsigned int)));
    k_affine_check<<<grid_for(c->n_el, 256), 256>>>(c->n_el, c->conn, dX, dna);
    TL_CHECK_LAUNCH();
    unsigned int na = 0;
    TL_CUDA(cudaMemcpy(&na, dna, sizeof(na), cudaMemcpyDeviceToHost));
    c->affine = na ? 0 : 1;
  }
  if (c->force_tables != 2) TL_TRY(build_geometry_classes(c, dX));
  // straight-sided T10 with geometry classes: the affine layout of each class
  // representative (the force-only kernel evaluates the T10 basis from it)
  if (c->element == TLFEA_T10 && c->affine && c->n_cls > 0) {
    const int64_t nr = (int64_t)c->cls_rep.size();
    TmpArr<int64_t> drep;
    TL_TRY(drep.get(nr));
    TL_CUDA(cudaMemcpy(drep.p, c->cls_rep.data(), sizeof(int64_t) * nr, cudaMemcpyHostToDevice));
    TL_TRY(c->alloc(&c->cls_aff, (size_t)nr * 13));
    k_affine_layout<<<grid_for(nr, 128), 128>>>(nr, c->conn, dX, c->cls_aff, drep.p);
    TL_CHECK_LAUNCH();
  }
  // no classes: straight-sided T10 elements take the affine (min) layout
  if (c->element == TLFEA_T10 && c->affine && c->n_cls == 0 && c->force_tables != 1 && c->n_el > 0) {
    TL_TRY(c->alloc(&c->aff, (size_t)c->n_el * 13));
    k_affine_layout<<<grid_for(c->n_el, 256), 256>>>(c->n_el, c->conn, dX, c->aff);
    TL_CHECK_LAUNCH();
  }
  // curved T10 without classes: per (e,q) the inverse Jacobian and J0 w_q (10
  // fp64 instead of the 31 of the paper's grad N + J0 w tables);
  // the kernels rebuild grad N from the T10 basis at the rule's points
  if (c->element == TLFEA_T10 && !c->affine && c->n_cls == 0 && c->force_tables == 0 && c->n_el > 0) {
    TL_TRY(c->alloc(&c->jinv, (size_t)c->n_el * nq * 10));
    TmpArr<double> g2, w2;
    TL_TRY(g2.get((size_t)c->n_el * nq * nen * 3));
    TL_TRY(w2.get((size_t)c->n_el * nq));
    k_precompute<<<grid_for(c->n_el * nq, 128), 128>>>(c->element, c->n_el, nq, nen, c->conn, dX, ddims, dq.p, dw.p,
                                                       g2.p, w2.p, c->err_flag, c->jinv);
    TL_CHECK_LAUNCH();
  }

  // ---- a-2 pattern over setup elements (64-bit keys, sort, unique)
  // constraint couplings join the element keys (pattern union)
  const std::vector<unsigned long long> ckeys = constraint_keys(opts->constraints);
  const int64_t nekeys = NS * nen * nen;
  const int64_t nkeys = nekeys + (int64_t)ckeys.size();
  {
    TmpArr<unsigned long long> keys, keys2;
    TL_TRY(keys.get(nkeys));
    TL_TRY(keys2.get(nkeys));
    if (nekeys > 0) {
      k_keys<<<grid_for(nekeys, 256), 256>>>(NS, nen, dsconn.p, c->own_idx, keys.p);
      TL_CHECK_LAUNCH();
    }
    if (!ckeys.empty())
      TL_CUDA(cudaMemcpy(keys.p + nekeys, ckeys.data(), sizeof(unsigned long long) * ckeys.size(),
                         cudaMemcpyHostToDevice));
    Tmp tmp;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, keys2.p, (int64_t)nkeys);
    TL_TRY(tmp.get(bytes));
    TL_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, keys.p, keys2.p, (int64_t)nkeys));
    count_launch();
    TmpArr<int64_t> nsel;
    TL_TRY(nsel.get(1));
    bytes = 0;
    cub::DeviceSelect::Unique(nullptr, bytes, keys2.p, keys.p, nsel.p, (int64_t)nkeys);
    TL_TRY(tmp.get(bytes));
    TL_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, keys2.p, keys.p, nsel.p, (int64_t)nkeys));
    count_launch();
    int64_t nu = 0;
    TL_CUDA(cudaMemcpy(&nu, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    unsigned long long last = 0;
    if (nu > 0) TL_CUDA(cudaMemcpy(&last, keys.p + nu - 1, sizeof(last), cudaMemcpyDeviceToHost));
    c->nnz_c = nu - (nu > 0 && last == ~0ull ? 1 : 0);
    // 32-bit coefficient-level indices and block offsets / 3 (k_unit_meta):
    // H up to 3 x 2^31 values (51 GB), the DOF rowptr and slots are 64-bit
    if (3 * c->nnz_c >= (1ll << 31))
      return fail(TLFEA_E_OVERFLOW, "DOF-level nnz = " + std::to_string(9 * c->nnz_c) + " >= 3 x 2^31");
    TL_TRY(c->alloc(&c->cols_c, (size_t)c->nnz_c));
    TL_TRY(c->alloc(&c->blk_row, (size_t)c->nnz_c));
    TL_TRY(c->alloc(&c->rowptr_c, (size_t)c->n_own + 1));
    TmpArr<int32_t> cnt;
    TL_TRY(cnt.get(c->n_own + 1));
    TL_CUDA(cudaMemset(cnt.p, 0, sizeof(int32_t) * (c->n_own + 1)));
    if (c->nnz_c > 0) {
      k_split_keys<<<grid_for(c->nnz_c, 256), 256>>>(c->nnz_c, keys.p, c->cols_c, c->blk_row, cnt.p);
      TL_CHECK_LAUNCH();
    }
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, c->rowptr_c, (int64_t)(c->n_own + 1));
    TL_TRY(tmp.get(bytes));
    TL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, c->rowptr_c, (int64_t)(c->n_own + 1)));
    count_launch();
  }
  c->upper = opts->hessian_upper;
  c->nnz_H = 9 * c->nnz_c;
  if (c->upper) {
    // UPPER: per-row counts 6 + 9 L_I -> offsets; then the lifted pattern
    TmpArr<int32_t> ucnt;
    TL_TRY(ucnt.get(c->n_own + 1));
    TL_TRY(c->alloc(&c->ubase, (size_t)c->n_own + 1));
    if (c->n_own > 0) {
      k_upper_count<<<grid_for(c->n_own, 256), 256>>>(c->n_own, c->rowptr_c, c->cols_c, c->own_nodes, ucnt.p);
      TL_CHECK_LAUNCH();
    }
    TL_CUDA(cudaMemset(ucnt.p + c->n_own, 0, sizeof(int32_t)));
    Tmp tmp;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, ucnt.p, c->ubase, (int64_t)(c->n_own + 1));
    TL_TRY(tmp.get(bytes));
    TL_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, ucnt.p, c->ubase, (int64_t)(c->n_own + 1)));
    count_launch();
    int32_t nu = 0;
    TL_CUDA(cudaMemcpy(&nu, c->ubase + c->n_own, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (4.5 * (double)c->nnz_c + 3.0 * (double)c->n_own >= 2147483647.0)
      return fail(TLFEA_E_OVERFLOW, "UPPER storage: more than 2^31 values (32-bit offsets)");
    c->nnz_H = nu;
  }
  TL_TRY(c->alloc(&c->rowptr, (size_t)3 * c->n_own + 1));
  TL_TRY(c->alloc(&c->cols, (size_t)std::max<int64_t>(c->nnz_H, 1)));
  if (c->n_own > 0 && c->upper) {
    k_lift_upper<<<grid_for(std::max(c->nnz_c, c->n_own), 256), 256>>>(
        c->n_own, c->nnz_c, c->rowptr_c, c->cols_c, c->blk_row, c->own_nodes, c->ubase, c->rowptr, c->cols);
    TL_CHECK_LAUNCH();
  } else if (c->n_own > 0) {
    k_lift<<<grid_for(std::max(c->nnz_c, c->n_own), 256), 256>>>(c->n_own, c->nnz_c, c->rowptr_c, c->cols_c,
                                                                c->blk_row, c->rowptr, c->cols);
    TL_CHECK_LAUNCH();
  } else {
    TL_CUDA(cudaMemset(c->rowptr, 0, sizeof(int64_t)));
  }
  TL_TRY(setup_constraints(c, opts->constraints));

  // ---- slot map of local elements + H gather lists (the slot map replaces the
  // paper's binary search at P:520)
  const int64_t nloc = c->n_el * nen * nen;
  TL_TRY(c->alloc(&c->slot_c, (size_t)nloc));
  TL_TRY(c->alloc(&c->blk_ptr, (size_t)c->nnz_c + 1));
  {
    TmpArr<int32_t> pkey;
    TmpArr<uint32_t> pval, sorted;
    TL_TRY(pkey.get(nloc));
    TL_TRY(pval.get(nloc));
    if (c->n_el > 0) {
      k_slots<<<grid_for(nloc, 256), 256>>>(c->n_el, nen, c->conn, c->own_idx, c->rowptr_c, c->cols_c,
                                            c->slot_c, pkey.p, pval.p);
      TL_CHECK_LAUNCH();
    }
    uint32_t* sv = nullptr;
    int64_t nvalid = 0;
    TL_TRY(sort_and_ptr<uint32_t>(nloc, pkey.p, pval.p, c->nnz_c, c->blk_ptr, &sv, &nvalid, sorted));
    TL_TRY(c->alloc(&c->blk_ent, (size_t)nvalid));
    TL_CUDA(cudaMemcpy(c->blk_ent, sv, sizeof(uint32_t) * nvalid, cudaMemcpyDeviceToDevice));
  }
  TL_TRY(c->alloc(&c->node_ptr, (size_t)c->n_own + 1));
  {
    const int64_t n = c->n_el * nen;
    TmpArr<int32_t> key;
    TmpArr<uint32_t> val, sorted;
    TL_TRY(key.get(n));
    TL_TRY(val.get(n));
    if (n > 0) {
      k_node_pairs<<<grid_for(n, 256), 256>>>(c->n_el, nen, c->conn, c->own_idx, key.p, val.p);
      TL_CHECK_LAUNCH();
    }
    uint32_t* sv = nullptr;
    int64_t nvalid = 0;
    TL_TRY(sort_and_ptr<uint32_t>(n, key.p, val.p, c->n_own, c->node_ptr, &sv, &nvalid, sorted));
    TL_TRY(c->alloc(&c->node_ent, (size_t)nvalid));
    TL_CUDA(cudaMemcpy(c->node_ent, sv, sizeof(uint32_t) * nvalid, cudaMemcpyDeviceToDevice));
  }

  TL_TRY(build_units(c));
  TL_TRY(build_sorted_scratch(c));

  // ---- consistent mass over the setup elements (reading Q4) and f_ff
  TL_TRY(c->alloc(&c->M, (size_t)c->nnz_c));
  TL_TRY(c->alloc(&c->fff, (size_t)3 * c->n_own));
  {
    double mq[kMassRuleT10 * 3], mw[kMassRuleT10];
    int nmq;
    static_assert(kMassRuleBeam <= kMassRuleT10, "mass rule buffers");
    if (c->element == TLFEA_T10 && c->mass_rule == 0) {
      nmq = make_mass_rule_t10(mq, mw);
    } else if (c->element == TLFEA_ANCF3243 && c->mass_rule == 0) {
      nmq = make_mass_rule_beam(mq, mw);
    } else {
      nmq = make_rule(c->quadrature, mq, mw);
    }
    TmpArr<double> dmq, dmw, me;
    TL_TRY(dmq.get(3 * kMassRuleT10));
    TL_TRY(dmw.get(kMassRuleT10));
    TL_CUDA(cudaMemcpy(dmq.p, mq, sizeof(double) * 3 * nmq, cudaMemcpyHostToDevice));
    TL_CUDA(cudaMemcpy(dmw.p, mw, sizeof(double) * nmq, cudaMemcpyHostToDevice));
    const int64_t nm = NS * nen * nen;
    // single rank with geometry classes: one mass matrix per class (its
    // representative element), read through the class id in the gather
    const bool per_class = c->nranks == 1 && c->n_cls > 0 && NS == c->n_el;
    TmpArr<int32_t> rconn;
    TmpArr<double> rdims;
    if (per_class) {
      const int64_t nr = (int64_t)c->cls_rep.size();
      std::vector<int32_t> hc((size_t)nr * nen);
      std::vector<double> hd(dims.empty() ? 1 : (size_t)nr * 3, 0.0);
      for (int64_t r = 0; r < nr; ++r) {
        for (int a = 0; a < nen; ++a) hc[r * nen + a] = cc[c->cls_rep[r] * nen + a];
        if (!dims.empty())
          for (int k = 0; k < 3; ++k) hd[r * 3 + k] = dims[c->cls_rep[r] * 3 + k];
      }
      TL_TRY(rconn.get(hc.size()));
      TL_TRY(rdims.get(hd.size()));
      TL_TRY(me.get((size_t)nr * nen * nen));
      TL_CUDA(cudaMemcpy(rconn.p, hc.data(), sizeof(int32_t) * hc.size(), cudaMemcpyHostToDevice));
      TL_CUDA(cudaMemcpy(rdims.p, hd.data(), sizeof(double) * hd.size(), cudaMemcpyHostToDevice));
      k_element_mass<<<grid_for(nr, 64), 64>>>(c->element, nr, nen, nmq, rconn.p, dX, dims.empty() ? nullptr : rdims.p,
                                              dmq.p, dmw.p, c->mat.rho0, me.p);
      TL_CHECK_LAUNCH();
    } else {
      TL_TRY(me.get(nm));
      if (NS > 0) {
        k_element_mass<<<grid_for(NS, 64), 64>>>(c->element, NS, nen, nmq, dsconn.p, dX, dsdims.p, dmq.p,
                                                dmw.p, c->mat.rho0, me.p);
        TL_CHECK_LAUNCH();
      }
    }
    TmpArr<int32_t> key;
    TmpArr<int64_t> val, sorted;
    TL_TRY(key.get(nm));
    TL_TRY(val.get(nm));
    if (nm > 0) {
      k_mass_pairs<<<grid_for(nm, 256), 256>>>(NS, nen, dsconn.p, c->own_idx, c->rowptr_c, c->cols_c, key.p,
                                               val.p);
      TL_CHECK_LAUNCH();
    }
    TmpArr<int32_t> mptr;
    TL_TRY(mptr.get(c->nnz_c + 1));
    int64_t* sv = nullptr;
    int64_t nvalid = 0;
    TL_TRY(sort_and_ptr<int64_t>(nm, key.p, val.p, c->nnz_c, mptr.p, &sv, &nvalid, sorted));
    if (c->nnz_c > 0) {
      k_mass_gather<<<grid_for(c->nnz_c, 256), 256>>>(c->nnz_c, mptr.p, sv, me.p, per_class ? c->cls : nullptr,
                                                      nen * nen, c->M);
      TL_CHECK_LAUNCH();
    }
    if (per_class) {  // the class element masses, for the element-level inertia of the AdamW gradient
      TL_TRY(c->alloc(&c->cls_mass, (size_t)c->n_cls * nen * nen));
      TL_CUDA(cudaMemcpy(c->cls_mass, me.p, sizeof(double) * c->n_cls * nen * nen, cudaMemcpyDeviceToDevice));
    }
    if (c->n_own > 0) {
      k_force_field<<<grid_for(c->n_own, 256), 256>>>(c->n_own, c->rowptr_c, c->M, c->gravity[0],
                                                      c->gravity[1], c->gravity[2], c->fff);
      TL_CHECK_LAUNCH();
    }
  }

  TL_TRY(build_unit_meta(c));

  // ---- eval scratch
  // element blocks are addressed with 32-bit block positions
  if (c->n_el * (int64_t)n_ublk_of(nen) >= (int64_t(1) << 31))
    return fail(TLFEA_E_OVERFLOW, "element tangent scratch exceeds 2^31 blocks: partition the mesh over more ranks");
  // +4 doubles: the bulk-copy gather rounds its windows out to 16-byte bounds
  TL_TRY(c->alloc(&c->Kscr, (size_t)c->n_el * n_ublk_of(nen) * (c->kvc ? 18 : 9) + 4));
  TL_TRY(c->alloc(&c->fscr, (size_t)c->n_el * nen * 3));
  TL_TRY(c->alloc(&c->fpart, (size_t)3 * std::max<int64_t>(c->n_own, 1)));

  // ---- partition exchange lists
  if (c->nranks > 1) TL_TRY(setup_exchange(c, cc, part, owner, local));
  TL_CUDA(cudaDeviceSynchronize());
  return TLFEA_OK;
}

}  // namespace tlfea
