// common.cuh — internal types of libtlfea (B200 / sm_100a, fp64).
// Nothing here is shared with oracle/ (independent implementation).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/tlfea.h"

namespace tlfea {

// ------------------------------------------------------------ error plumbing
void set_error(const std::string& msg);
tlfea_status fail(tlfea_status st, const std::string& msg);
void count_launch(int n = 1);
// Dynamic shared memory (and static + dynamic above 48 KB) needs the
// per-device, per-kernel opt-in attribute: applied once per (kernel, current
// device, size), thread-safe.
tlfea_status ensure_dynamic_smem(const void* kernel, size_t bytes, int block_threads = 128);
// the maximum shared-memory carveout for a kernel (once per kernel and device)
tlfea_status ensure_carveout(const void* kernel);

#define TL_CUDA(call)                                                          \
  do {                                                                         \
    cudaError_t err__ = (call);                                                \
    if (err__ != cudaSuccess)                                                  \
      return ::tlfea::fail(err__ == cudaErrorMemoryAllocation ? TLFEA_E_OOM    \
                                                              : TLFEA_E_CUDA,  \
                           std::string(#call) + ": " + cudaGetErrorString(err__)); \
  } while (0)

#define TL_TRY_LAUNCH(expr)                    \
  do {                                         \
    const tlfea_status st_try__ = (expr);      \
    if (st_try__ != TLFEA_OK) return st_try__; \
  } while (0)

// propagate a non-OK status
#define TL_TRY(expr)                      \
  do {                                    \
    tlfea_status st__ = (expr);           \
    if (st__ != TLFEA_OK) return st__;    \
  } while (0)

#define TL_CHECK_LAUNCH()                                                      \
  do {                                                                         \
    ::tlfea::count_launch();                                                   \
    cudaError_t err__ = cudaGetLastError();                                    \
    if (err__ != cudaSuccess)                                                  \
      return ::tlfea::fail(TLFEA_E_CUDA, std::string("kernel launch: ") +      \
                                             cudaGetErrorString(err__));       \
  } while (0)

// ------------------------------------------------------------------- sizes
constexpr int kMaxQP = 48;
constexpr int kMaxEN = 16;

inline int n_en_of(int element) { return element == TLFEA_T10 ? 10 : element == TLFEA_ANCF3443 ? 16 : 8; }
// physical nodes per element in the caller's connectivity
inline int n_nodes_of(int element) { return element == TLFEA_T10 ? 10 : element == TLFEA_ANCF3443 ? 4 : 2; }
inline int n_qp_of(int quadrature) {
  return quadrature == TLFEA_Q_T10_4PT ? 4
         : quadrature == TLFEA_Q_T10_KEAST5 ? 5
         : quadrature == TLFEA_Q_GL_3x2x2 ? 12
                                          : 48;
}
// number of upper-triangular 3x3 blocks (a <= b) of the element matrix
inline int n_ublk_of(int nen) { return nen * (nen + 1) / 2; }
// element-kernel CTA tile: kElWarps warps of 3 T10 / 1 ANCF3443 / 4 ANCF3243 elements
#ifndef TLFEA_EL_WARPS
#define TLFEA_EL_WARPS 4
#endif
constexpr int kElWarps = TLFEA_EL_WARPS;
inline int el_per_tile(int element) {
  return kElWarps * (element == TLFEA_T10 ? 3 : element == TLFEA_ANCF3443 ? 1 : 4);
}
// gather CTA: 4 warps of 32 units (H) / 128 threads (f)
constexpr int kGatherThreads = 128;

// Packed contribution entry of the H gather: element (local id) << 8 | a << 4 | b
__host__ __device__ inline uint32_t pack_eab(uint32_t e, uint32_t a, uint32_t b) {
  return (e << 8) | (a << 4) | b;
}

// Material constants as used on the device.
struct MatDev {
  int model;       // 0 SVK, 1 MR
  int kv;          // Kelvin-Voigt active
  double lam, mu;  // SVK Lame constants
  double C10, C01, kappa;
  double eta, lamd;
  double rho0;
};

// Device buffer helper (raw cudaMalloc, owned by the context)
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Context {
  // problem
  int element = 0, quadrature = 0, nen = 10, nq = 5, mass_rule = 0;
  MatDev mat{};
  tlfea_material mat_in{};
  double gravity[3] = {0, 0, 0};
  int device = 0;
  int rank = 0, nranks = 1;
  int64_t n_el_global = 0, n_coef = 0;
  int64_t n_el = 0;            // local elements
  int64_t n_el_bnd = 0;        // partitioned: local elements [0, n_el_bnd) are the boundary range
  bool interior_pending = false;  // tlfea_eval_begin ran, tlfea_eval_interior not yet
  int64_t n_own = 0;           // owned coefficient rows
  int64_t nnz_c = 0;           // owned-row coefficient nnz
  int affine = 0;
  int force_tables = 0;         // options.reference_layout: 1 tables always, 2 affine (min) layout first
  // H storage: full DOF CSR (9 nnz_c values) or UPPER (col >= row). UPPER row
  // 3I+d starts at ubase[I] + d (3 + 3 L_I) - d (d - 1) / 2, L_I = blocks
  // J > I of coefficient row I; block (I, J) with rank k among J >= I (k = 0:
  // the diagonal) has entry (d, f) at ubase[I] + 3 k + f + d (2 + 3 L_I)
  // - d (d - 1) / 2 (f >= d when k = 0).
  int upper = 0;
  // consistent Kelvin-Voigt tangent (options.kv_consistent_tangent with damping,
  // NEXT-4): each gather-sorted scratch slot holds 18 values, the unit's (I,J)
  // and (J,I) contributions in their own orientation (non-symmetric blocks);
  // eval_inv_h = 1/h of the evaluation in flight (the consistent-KV element
  // kernels scale the df/dv part by 1/h so the gather's h * acc + M/h gives
  // h df/dx + df/dv; the AdamW element inertia m_e (v - v_n)_e is scaled by it).
  int kvc = 0;
  double eval_inv_h = 0.0;
  // element-level inertia request of the AdamW gradient (launch_element_kernel,
  // force only, T10 SVK affine kernel with classes; v then holds v - v_n)
  bool inr = false;
  double* dvscr = nullptr;        // [n_dof] v - v_n of the AdamW iteration (lazily allocated)
  int64_t nnz_H = 0;           // values of H as stored
  int32_t* ubase = nullptr;    // [n_own + 1] UPPER offsets of coefficient rows

  // device data
  int32_t* conn = nullptr;     // [n_el][nen] coefficient ids (local elements)
  int64_t* elem_gid = nullptr; // [n_el] global element id of each local element
  double* gradN = nullptr;     // [n_el][nq][nen][3]
  double* J0w = nullptr;       // [n_el][nq]
  int32_t* own_nodes = nullptr;   // [n_own] global coefficient ids, ascending
  int32_t* own_idx = nullptr;     // [n_coef] local row of a coefficient or -1
  int32_t* rowptr_c = nullptr;    // [n_own+1]
  int32_t* cols_c = nullptr;      // [nnz_c]
  int32_t* blk_row = nullptr;     // [nnz_c] owned row of each coefficient block
  int64_t* rowptr = nullptr;      // [3 n_own + 1]  DOF level (64-bit: H may exceed 2^31 values)
  int32_t* cols = nullptr;        // [9 nnz_c]
  double* M = nullptr;            // [nnz_c]
  double* fff = nullptr;          // [3 n_own]
  int32_t* slot_c = nullptr;      // [n_el][nen][nen] coefficient-level slot (-1 not owned)
  int32_t* blk_ptr = nullptr;     // [nnz_c+1]
  uint32_t* blk_ent = nullptr;    // [...] packed (e,a,b), e ascending per block
  int32_t* node_ptr = nullptr;    // [n_own+1]
  uint32_t* node_ent = nullptr;   // [...] (e << 4 | a)
  // geometry classes: congruent elements share one reference table
  // (gradN + J0w); the eval kernels then read it from shared memory.
  int n_cls = 0;                  // 0 = per-element tables (gradN / J0w above)
  uint8_t* cls = nullptr;         // [n_el] class id
  double* cls_tab = nullptr;      // [n_cls][nq][nen*3 + 1]  (gradN then J0w)
  // affine (min) layout of straight-sided T10 without classes: [n_el][13] =
  // grad_X z_0..3 (barycentric gradients), J0 (SURVEY §8(d) min layout)
  double* aff = nullptr;
  double* jinv = nullptr;         // [n_el][nq][10] J^-1 (row-major) and J0 w_q (curved T10 without classes)
  double* cls_aff = nullptr;
  double* cls_mass = nullptr;     // [n_cls][nen][nen] element mass per class (single rank, classes)      // [n_cls][13] the same per class (straight-sided T10 with classes)
  std::vector<int64_t> cls_rep;   // representative (first) element of each class
  // symmetric H gather units (upper blocks + blocks whose transpose is not owned)
  int64_t n_units = 0;
  int32_t* unit_p = nullptr;      // [n_units] coefficient block of (I,J)
  int32_t* unit_pT = nullptr;     // [n_units] block of (J,I) in row J, -1 if none
  // gather-sorted scratch (single-rank contexts): element upper block ub of
  // element e is written to position dest[e][ub] >> 1 (transposed if the low
  // bit is set), so the H gather streams unit_ptr[u] .. unit_ptr[u+1].
  int32_t* dest = nullptr;        // [n_el][n_ublk]
  int32_t* unit_ptr = nullptr;    // [n_units+1]
  int32_t* fdest = nullptr;       // [n_el][nen] position of f_a in the node-sorted force scratch
  // flattened per-unit output metadata (no dependent index chains in the gather)
  int32_t* u_off = nullptr;       // [n_units] H offset of block (I,J) / 3 = 3 rowptr_c[i] + k (UPPER: the offset)
  int32_t* u_offT = nullptr;      // [n_units] H offset of (J,I) / 3, or -1
  int32_t* u_deg = nullptr;       // [n_units] deg(I) | deg(J) << 16
  double* u_m = nullptr;          // [n_units] M_IJ
  double* Kscr = nullptr;         // [n_el][n_ublk][9]
  double* fscr = nullptr;         // [n_el][nen][3]
  unsigned long long* err_flag = nullptr;  // min over (e*64+q) with det F <= 0 (MR)

  // partition exchange (nranks > 1)
  std::vector<int64_t> send_counts, recv_counts;     // fp64 values per peer
  // the library's NCCL transport (tlfea_nccl_attach / tlfea_eval_exchange, nccl.cu)
  void* nccl_comm = nullptr;                 // ncclComm_t
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_exchanged = nullptr;
  bool exchange_pending = false;
  int64_t n_send_blk = 0, n_recv_blk = 0, n_send_node = 0, n_recv_node = 0;
  int32_t* sblk_ptr = nullptr;   // [n_send_blk+1] contribution lists of sent blocks
  uint32_t* sblk_ent = nullptr;
  int32_t* snode_ptr = nullptr;  // [n_send_node+1]
  uint32_t* snode_ent = nullptr;
  int64_t send_blk_vals = 0;     // 9 * n_send_blk (first part of send buffer)
  int32_t* rblk_slot = nullptr;  // [n_recv_blk] owned coefficient block receiving
  int32_t* rnode_row = nullptr;  // [n_recv_node] owned row receiving
  int64_t* send_blk_off = nullptr;   // [n_send_blk] offset in the send buffer
  int64_t* send_node_off = nullptr;  // [n_send_node]
  int64_t* recv_peer_blk_off = nullptr;  // host copies are enough
  std::vector<int64_t> recv_blk_count, recv_node_count, send_blk_count, send_node_count;
  double* fpart = nullptr;       // [3 n_own] local partial force (partitioned mode)
  double* norm_part = nullptr;   // [2 x kNormBlocks] partial sums of the AdamW norms

  // linear constraints c(q) = C q - b (NEXT-3, reading Q22; single rank)
  int64_t n_con = 0;
  int32_t* con_ptr = nullptr;    // [m+1] rows of C
  int32_t* con_cols = nullptr;   // DOF columns
  double* con_vals = nullptr;
  double* con_b = nullptr;       // [m]
  int32_t* conT_ptr = nullptr;   // [n_dof+1] rows of C^T (ascending constraint index)
  int32_t* conT_rows = nullptr;
  double* conT_vals = nullptr;
  int64_t n_gram = 0;            // distinct (i, j) DOF pairs of C^T C
  int64_t* gram_ij = nullptr;    // [n_gram] i << 32 | j (setup), then the H slot
  double* gram_val = nullptr;    // [n_gram] sum_k C_ki C_kj (ascending k)
  double* con_c = nullptr;       // [m] residual buffer

  // live timing (tlfea_set_timing)
  bool timing = false;
  struct TimedLaunch {
    int kind;
    cudaEvent_t start, stop;
  };
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> event_pool;
  // persistent staging of tlfea_eval_host
  double *h_x = nullptr, *h_v = nullptr, *h_vn = nullptr, *h_fe = nullptr, *h_g = nullptr, *h_H = nullptr,
         *h_f = nullptr;

  std::vector<DevBuf> owned;     // every cudaMalloc of this context
  int64_t device_bytes = 0;
  cudaStream_t last_stream = nullptr;

  ~Context();
  template <class T>
  tlfea_status alloc(T** p, size_t count);
};

template <class T>
tlfea_status Context::alloc(T** p, size_t count) {
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = sizeof(T);
  void* q = nullptr;
  cudaError_t err = cudaMalloc(&q, bytes);
  if (err != cudaSuccess) {
    cudaGetLastError();
    return fail(TLFEA_E_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " +
                                 cudaGetErrorString(err));
  }
  owned.push_back({q, bytes});
  device_bytes += (int64_t)bytes;
  *p = static_cast<T*>(q);
  return TLFEA_OK;
}

// Entry points implemented in setup.cu / eval.cu
tlfea_status setup_context(Context* c, const tlfea_mesh* mesh, const tlfea_material* mat,
                           const tlfea_options* opts);
tlfea_status launch_element_kernel(Context* c, const double* x, const double* v,
                                   bool tangent, cudaStream_t s, int64_t e_begin = 0, int64_t e_end = -1);
tlfea_status launch_gather_H(Context* c, double h, double* H, cudaStream_t s);
tlfea_status launch_gather_f(Context* c, const double* v, const double* vn, const double* fext,
                             double h, double* g, double* fint, bool partial_only,
                             cudaStream_t s);
tlfea_status launch_stress_only(Context* c, const double* x, const double* v, double* P,
                                cudaStream_t s);
tlfea_status launch_force_from_stress(Context* c, const double* P, cudaStream_t s);
tlfea_status launch_residual(Context* c, const double* fint, const double* v, const double* vn,
                             const double* fext, double h, double* g, cudaStream_t s);
tlfea_status launch_adamw_update(Context* c, int l, const tlfea_adamw_params& p, const double* g, double* m,
                                 double* s, double* v, const double* q_n, double h, double* q, cudaStream_t st,
                                 const double* vn = nullptr, double* dv = nullptr);
tlfea_status launch_norms2(Context* c, const double* a, const double* b, double* out, cudaStream_t st);
tlfea_status launch_constraint_residual(Context* c, const double* q, double* c_out, cudaStream_t st);
tlfea_status launch_constraint_terms(Context* c, const double* q, const double* lam, double rho, double h,
                                     double* g, double* H, cudaStream_t st);
tlfea_status launch_dual_update(Context* c, const double* q, double rho, double* lam, double* c_out,
                                cudaStream_t st);
tlfea_status launch_pack_send(Context* c, double* send, bool force_only, cudaStream_t s);
tlfea_status launch_gradient_inertia(Context* c, const double* fext, double* g, cudaStream_t s);
bool force_inertia_capable(const Context* c);
bool eval_small_ok(const Context* c);
tlfea_status launch_eval_small(Context* c, const double* x, const double* v, const double* vn, const double* fext,
                               double h, double* g, double* H, double* fint, cudaStream_t s);
tlfea_status nccl_get_unique_id(void* id_out);
tlfea_status nccl_attach(Context* c, const void* id);
void nccl_detach(Context* c);
tlfea_status nccl_exchange(Context* c, const double* send_buf, double* recv_buf, cudaStream_t s);
tlfea_status nccl_wait(Context* c, cudaStream_t s);
tlfea_status launch_unpack_recv(Context* c, const double* recv, double h, double* H,
                                bool force_only, cudaStream_t s);
tlfea_status launch_test_constitutive(const MatDev& m, int64_t n, const double* F,
                                      const double* Fd, double* P, double* A);
MatDev make_matdev(const tlfea_material& m);
tlfea_status setup_exchange(Context* c, const std::vector<int32_t>& cc, const std::vector<int32_t>& part,
                            const std::vector<int32_t>& owner, const std::vector<int64_t>& local);
const char* last_error();
int64_t launch_count();

}  // namespace tlfea
