/*
 * tlfea.h — C ABI of libtlfea.so, the B200 (sm_100a) fp64 hot path of
 * arXiv 2604.10357 ("A Total Lagrangian Finite Element Framework for
 * Multibody Dynamics: Part II — GPU Implementation").
 *
 * Citation convention: "P:n" = line n of the paper text, with the
 * section / equation it falls in; SURVEY §8 rows name the hot-path steps.
 *
 * What the library computes:
 *   a-1  reference precompute per (element e, quadrature point q):
 *        grad_X N_a = (dN_a/dxi) J^{-1},  J0*w_q            (§4.1)
 *   a-2  fixed-sparsity CSR pattern from 64-bit (row,col) keys, sorted and
 *        de-duplicated on the device, lifted to 3x3 DOF blocks; the
 *        element-entry -> CSR-slot map; consistent mass M and f_ff
 *                                                     (§4.2)
 *   a-3  Stage 1 per (e,q): F = sum_a x_a (x) grad_X N_a, P = P_el(F) + P_vis
 *                                         (§4.3 Eq. F_assembly)
 *   a-4  Stage 2 force f_a = sum_q P grad_X N_a J0 w_q and its assembly
 *                        (Eqs. fint_local / fint_global)
 *   a-5  element tangent [K_ab]_de = A_dJeL gradN_aJ gradN_bL J0 w_q
 *                        (Eq. tangent_block)
 *   a-6  H = M/h + h K_t scattered into the fixed CSR through the slot map,
 *        deterministically (no floating-point atomics)
 *                        (Eq. hessian)
 *   a-7  residual g = (1/h) M (v - v_n) + f_int - f_ext - f_ff
 *                        (Eq. residual, Eq. grad_L)
 *
 * Conventions shared by every entry point
 *   - All floating point is IEEE fp64.
 *   - DOF map: dof(I,d) = 3*I + d (node/coefficient-major, component-minor;
 *     P:457-458). For ANCF3443 coefficient I = 4*node + m, m in {r, r_x, r_y, r_z}.
 *   - "device" pointers are CUDA device pointers on the context's device
 *     (e.g. torch.Tensor.data_ptr() of a CUDA tensor); "host" pointers are
 *     ordinary CPU memory. Each argument says which.
 *   - Every call returns tlfea_status; no C++ exception or abort crosses the
 *     ABI. On error tlfea_last_error() returns a thread-local message.
 *   - Evaluation calls are asynchronous on the caller's cudaStream_t (passed
 *     as void*; NULL = legacy default stream) and perform no host sync.
 *     One context is used by one stream at a time.
 *   - Nothing here falls back to the CPU: without a usable CUDA device,
 *     tlfea_setup returns TLFEA_E_CUDA.
 */
#ifndef TLFEA_H_
#define TLFEA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLFEA_ABI_VERSION 8

typedef struct tlfea_ctx_s* tlfea_ctx;

typedef enum {
  TLFEA_OK = 0,
  TLFEA_E_INVALID = 1,          /* bad argument, mesh, material or option     */
  TLFEA_E_INVERTED_ELEMENT = 2, /* J0 <= 0 at some (e,q) during setup         */
  TLFEA_E_INVERTED_STATE = 3,   /* Mooney-Rivlin det F <= 0 during an eval    */
  TLFEA_E_OVERFLOW = 4,         /* an index exceeds the int32 build limits    */
  TLFEA_E_OOM = 5,              /* device allocation failed                   */
  TLFEA_E_CUDA = 6,             /* CUDA runtime error / no device             */
  TLFEA_E_UNSUPPORTED = 7,      /* valid request this build does not provide  */
  TLFEA_E_NCCL = 8              /* NCCL unavailable or an NCCL call failed    */
} tlfea_status;

typedef enum { TLFEA_T10 = 0, TLFEA_ANCF3443 = 1, TLFEA_ANCF3243 = 2 } tlfea_element;

/* Quadrature rules. T10: 4-point degree-2 rule (BASELINE config 1)
 * or the 5-point Keast rule (negative centroid weight); ANCF3443: 4x4x3
 * Gauss-Legendre; ANCF3243 beam: 3x2x2
 * Gauss-Legendre; product rules ordered xi-major, eta, zeta-minor. */
typedef enum {
  TLFEA_Q_T10_4PT = 0,
  TLFEA_Q_T10_KEAST5 = 1,
  TLFEA_Q_GL_4x4x3 = 2,
  TLFEA_Q_GL_3x2x2 = 3
} tlfea_quadrature;

typedef enum { TLFEA_SVK = 0, TLFEA_MOONEY_RIVLIN = 1 } tlfea_model;

/* Constitutive parameters (Appendix tables).
 *  SVK: S = lambda tr(E) I + 2 mu E, E = (F^T F - I)/2, P = F S, with
 *       lambda = E nu/((1+nu)(1-2nu)), mu = E/(2(1+nu)).
 *  MR : W = C10(I1b-3) + C01(I2b-3) + kappa/2 (J-1)^2 (reading Q6).
 *  Kelvin-Voigt (active when eta_damp>0 or lambda_damp>0):
 *       Edot = (Fdot^T F + F^T Fdot)/2, S_v = 2 eta Edot + lambda_d tr(Edot) I,
 *       P_v = F S_v (reading Q7). Its tangent is NOT in H (Eq. hessian, Q8)
 *       unless options.kv_consistent_tangent asks for dg/dv (NEXT-4). */
typedef struct {
  int32_t model; /* tlfea_model */
  double E, nu;            /* SVK */
  double C10, C01, kappa;  /* Mooney-Rivlin */
  double rho0;             /* reference density (mass, f_ff) */
  double eta_damp, lambda_damp;
} tlfea_material;

/* Mesh, all HOST memory, copied by tlfea_setup (caller may free afterwards).
 *  T10     : conn [n_elements][10] node ids; local order = 4 corners, then
 *            edges (0,1),(1,2),(2,0),(0,3),(1,3),(2,3) (reading Q2).
 *            X_ref [n_coef][3] node reference positions.
 *  ANCF3443: conn [n_elements][4] physical node ids, counter-clockwise from
 *            (xi,eta)=(-1,-1); X_ref [n_coef][3] with n_coef = 4*n_nodes and
 *            coefficient 4*node+m = (r, r_x, r_y, r_z)[m] (reading Q11).
 *            ancf_dims [n_elements][3] = (L, W, H) per element, or NULL to
 *            use options.ancf_dims for every element.
 *  ANCF3243: conn [n_elements][2] physical node ids (A at xi = -1, B at
 *            xi = +1); X_ref and ancf_dims as for ANCF3443 (reading Q23:
 *            cubic Hermite (r, r_x) along the axis, linear (r_y, r_z)). */
typedef struct {
  int32_t element; /* tlfea_element */
  int64_t n_elements;
  int64_t n_coef;
  const int32_t* conn;
  const double* X_ref;
  const double* ancf_dims;
} tlfea_mesh;

/* Options.
 *  mass_rule: 0 = exact consistent mass (T10: degree-5 collapsed Gauss rule;
 *             ANCF: the force rule, already exact), 1 = same rule as the force
 *             (literal P:309-310; T10 mass then singular/indefinite, reading Q4).
 *  gravity  : body-force field g for f_ff[3I+d] = g_d sum_J M_IJ (Eq. residual).
 *  Multi-GPU element partition; nranks = 1 for a single GPU:
 *   rank, nranks, elem_part (host [n_elements] owning rank, or NULL for
 *   contiguous equal element blocks). A node is owned by the lowest rank
 *   among its incident elements (reading Q20).
 *  device   : CUDA device ordinal the context lives on.
 *  constraints: linear bilateral constraints (below), or NULL. */

/* Linear bilateral constraints c(q) = C q - b with a constant Jacobian C
 * (m x n_dof), all HOST memory copied by tlfea_setup (SURVEY §8(f) NEXT-3,
 * reading Q22; Eq. residual).
 * Clamped Dirichlet DOFs are identity rows (C row = e_i, b = clamped value).
 *  rowptr [m+1], cols [rowptr[m]] DOF ids (3 I + d) distinct within a row,
 *  vals [rowptr[m]], b [m]. The H pattern becomes the union of the element
 *  couplings and those of C^T C. Single-rank contexts only. */
typedef struct {
  int64_t m;
  const int64_t* rowptr;
  const int64_t* cols;
  const double* vals;
  const double* b;
} tlfea_constraints;

typedef struct {
  int32_t quadrature; /* tlfea_quadrature */
  int32_t mass_rule;
  double gravity[3];
  double ancf_dims[3];
  int32_t rank, nranks;
  const int32_t* elem_part;
  int32_t device;
  const tlfea_constraints* constraints;
  int32_t hessian_upper;  /* 0: full DOF CSR of H (default); 1: UPPER storage
                             (entries with col >= row only, rows in order, the
                             cuDSS-facing matrix view).
                             UPPER: single rank, no constraints. */
  int32_t reference_layout; /* 0 (default): geometry classes when every element
                             is congruent to one of <= 32 (T10) / 4 (ANCF)
                             reference shapes; else, for straight-sided T10,
                             the affine "min" layout (13 fp64 per element:
                             grad_X z_0..3 and J0); else the
                             per-(e,q) J^-1 and J0 w_q of curved T10 (10 fp64
                             per point, grad N rebuilt from the T10 basis);
                             else the per-(e,q) tables of §4.1.
                             1: the per-(e,q) tables always (the paper's
                             layout, on any mesh). 2: the affine layout
                             whenever the T10 mesh is straight-sided (no
                             classes), else the tables. Results agree to
                             rounding whichever is used. */
  int32_t kv_consistent_tangent; /* 0 (default): H = M/h + h K_t with the
                             elastic tangent only (Eq. hessian, K_t
                             "from F" P:526; reading Q8). 1 (SURVEY §8(f)
                             NEXT-4): with Kelvin-Voigt damping, H is the
                             consistent tangent of the velocity residual,
                             H = dg/dv = M/h + h df_int/dx + df_int/dv with
                             x = q_n + h v (Eq. residual, reading Q9):
                             per element block K_ab = h K_ab^el + eta w (g_b ga^T
                             + d_ab F F^T) + lambda_d w g_a g_b^T (from Fdot's
                             dependence on v) + h w (s^v_ab I + eta d_ab F Fdot^T
                             + eta g_b gdot_a^T + lambda_d g_a gdot_b^T) (from
                             F's, with S_v fixed), g = F grad N, gdot = Fdot grad N,
                             s^v_ab = grad N_a . S_v grad N_b, d_ab = grad N_a .
                             grad N_b, summed over q with w = J0 w_q. NOT
                             symmetric: FULL storage, single rank only
                             (TLFEA_E_INVALID with hessian_upper or nranks > 1);
                             tlfea_assemble_hessian (no velocities) then
                             returns TLFEA_E_INVALID. No effect without damping. */
} tlfea_options;

/* Sizes of a context (tlfea_info). Rows/DOFs are GLOBAL indices; in a
 * partitioned context the outputs of tlfea_eval cover the owned DOF rows
 * [row_begin, row_begin + n_rows) which are the DOFs of the owned nodes; the
 * owned nodes are contiguous in a node numbering produced by the caller's
 * partition; otherwise see owned_node list (tlfea_owned_nodes). */
typedef struct {
  int32_t element, quadrature, n_qp, n_en;
  int64_t n_elements;      /* elements processed by this context (local)   */
  int64_t n_elements_global;
  int64_t n_coef, n_dof;   /* global                                       */
  int64_t nnz_coef;        /* coefficient-level CSR nnz of the owned rows  */
  int64_t nnz;             /* DOF-level CSR nnz of the owned rows (= 9*nnz_coef) */
  int64_t n_owned_nodes;   /* owned coefficient rows                       */
  int32_t affine;          /* 1 if every T10 is straight-sided (compressed layout) */
  int32_t rank, nranks;
  int64_t device_bytes;    /* device memory held by the context            */
  int32_t n_geometry_classes; /* > 0: congruent elements share reference
                                 tables (staged in shared memory); 0: the
                                 per-(e,q) tables of §4.1 are read from HBM */
  int32_t fused_eval;      /* 1: tlfea_eval runs as ONE cooperative launch
                              (small class-mode T10 SVK meshes, <= 3,000
                              elements: element groups, grid barrier, H and
                              f / g gathers; bitwise the three-launch path);
                              0: element kernel + H gather + f/g gather. */
  int64_t n_constraints;   /* rows m of the context's constraint set (0: none) */
  int32_t reference_layout;/* in use: 0 geometry classes, 1 per-(e,q) tables,
                              2 affine (min) layout, 3 per-(e,q) J^-1 + J0 w
                              (curved T10, 10 fp64 per point) */
  int32_t kv_consistent_tangent; /* 1 if H is the consistent Kelvin-Voigt
                              tangent (options.kv_consistent_tangent with
                              damping), else 0 */
} tlfea_info_t;

/* ---------------------------------------------------------------- setup -- */

/* tlfea_setup — a-1 + a-2. Validates the mesh
 * (ids in range, distinct nodes per element), the material (E>0,
 * -1<nu<0.5 for SVK; C10,C01>=0, kappa>0 for MR; rho0>=0; damping>=0) and the
 * options; builds on the device: grad_X N and J0 w per (e,q), the coefficient
 * CSR (64-bit keys, radix sort, unique, counts, scan), its DOF lift, the
 * slot map, the mass M, f_ff, and the assembly schedule.
 * Errors: TLFEA_E_INVALID, TLFEA_E_INVERTED_ELEMENT (message names e),
 * TLFEA_E_OVERFLOW (owned-row nnz >= 2^31, or more than 2^24 elements on one
 * rank), TLFEA_E_OOM, TLFEA_E_CUDA.
 * Synchronizes the device. On success *out owns all device buffers. */
tlfea_status tlfea_setup(const tlfea_mesh* mesh, const tlfea_material* mat,
                         const tlfea_options* opts, tlfea_ctx* out);

/* Releases every device buffer of ctx. NULL is a no-op. */
void tlfea_destroy(tlfea_ctx ctx);

tlfea_status tlfea_info(tlfea_ctx ctx, tlfea_info_t* out);

/* ------------------------------------------------ pattern / slot map -- */

/* DOF-level CSR of H over the owned rows (reading Q14/Q15):
 * rowptr [n_rows+1] int64 (relative: rowptr[0]=0; 64-bit so H may hold 2^31
 * or more values, reading Q17), cols [nnz] int32 GLOBAL DOF columns,
 * strictly increasing per row; row r of the block is DOF row
 * 3*owned_node[r/3] + r%3. Pointers are DEVICE, borrowed until destroy.
 * Limits: nnz < 3 x 2^31 (FULL), < 2^31 (UPPER); 3 n_coef < 2^31. */
tlfea_status tlfea_pattern(tlfea_ctx ctx, const int64_t** rowptr,
                           const int32_t** cols);

/* Coefficient-level CSR (the mass / adjacency pattern of §4.2):
 * rowptr [n_owned_nodes+1], cols [nnz_coef] (global coefficient ids). DEVICE,
 * borrowed. */
tlfea_status tlfea_coef_pattern(tlfea_ctx ctx, const int32_t** rowptr,
                                const int32_t** cols);

/* Owned coefficient ids, ascending: DEVICE int32 [n_owned_nodes], borrowed.
 * For nranks = 1 it is 0..n_coef-1. */
tlfea_status tlfea_owned_nodes(tlfea_ctx ctx, const int32_t** nodes);

/* Copies of the patterns into caller DEVICE buffers (any may be NULL):
 * rowptr_out int64 [3 n_owned+1], cols_out int32 [nnz], rowptr_c_out int32
 * [n_owned+1], cols_c_out int32 [nnz_coef], owned_out int32 [n_owned].
 * Asynchronous on stream. */
tlfea_status tlfea_export_pattern(tlfea_ctx ctx, int64_t* rowptr_out, int32_t* cols_out,
                                  int32_t* rowptr_c_out, int32_t* cols_c_out,
                                  int32_t* owned_out, void* stream);

/* Canonical slot map (reading Q16): out_host int64 [e_count][3n_en][3n_en],
 * entry [e][3a+d][3b+f] = index into the DOF CSR values of the entry
 * (row 3*conn[e][a]+d, column 3*conn[e][b]+f), or -1 when that row is not
 * owned by this context. e indexes the context's LOCAL element list.
 * HOST output; synchronizes. */
tlfea_status tlfea_slot_map(tlfea_ctx ctx, int64_t e_begin, int64_t e_count,
                            int64_t* out_host);

/* ------------------------------------------------ setup exports (a-1,a-2) -- */

/* a-1: grad_out DEVICE [n_el][n_qp][n_en][3] = grad_X N_a at
 * (e,q); J0w_out DEVICE [n_el][n_qp] = det(dX/dxi) * w_q. Local elements. */
tlfea_status tlfea_export_precompute(tlfea_ctx ctx, double* grad_out,
                                     double* J0w_out, void* stream);

/* a-2: M_out DEVICE [nnz_coef] values of the
 * coefficient-level consistent mass on the coefficient pattern (global M,
 * owned rows); fff_out DEVICE [3*n_owned_nodes] = f_ff (Eq. residual). */
tlfea_status tlfea_export_mass(tlfea_ctx ctx, double* M_out, double* fff_out,
                               void* stream);

/* ------------------------------------------------------------ evaluation -- */

/* tlfea_eval — the fused hot path a-3..a-7 (Alg. 3 lines P:826-834 minus the
 * constraint terms). Inputs (DEVICE, GLOBAL length n_dof):
 *   x   current coordinates q_n + h v (the caller applies the step map, Eq. stepmap)
 *   v   current velocity (drives Fdot for Kelvin-Voigt, reading Q9)
 *   v_n previous-step velocity, or NULL (= 0)
 *   f_ext external nodal forces, or NULL (= 0)
 *   h   time step (> 0, else TLFEA_E_INVALID)
 * Outputs (DEVICE, owned rows): g_out [3*n_owned_nodes] residual;
 *   H_out [nnz] values of M/h + h K_t on tlfea_pattern (elastic tangent, or the
 *         consistent Kelvin-Voigt tangent per options.kv_consistent_tangent;
 *         full or UPPER storage per options.hessian_upper, info.nnz entries);
 *   f_int_out [3*n_owned_nodes] or NULL.
 * In a partitioned context (nranks > 1) use the begin/finish pair below.
 * Deterministic: bitwise identical results for identical inputs. */
tlfea_status tlfea_eval(tlfea_ctx ctx, const double* x, const double* v,
                        const double* v_n, const double* f_ext, double h,
                        double* g_out, double* H_out, double* f_int_out,
                        void* stream);

/* tlfea_eval_constrained — tlfea_eval plus the constraint terms of the
 * context's constraint set (NEXT-3; Eq. residual P:101-113, P:484-489 and
 * Eq. hessian), with c = C x - b (x = q_n + h v):
 *   g += h C^T (lambda + rho c),   H += h^2 rho C^T C.
 * lambda DEVICE [m] (NULL = 0), rho >= 0. Each H value receives its C^T C
 * sum once and each g entry its C^T row in ascending constraint order
 * (deterministic). Without constraints it equals tlfea_eval. */
tlfea_status tlfea_eval_constrained(tlfea_ctx ctx, const double* x, const double* v,
                                    const double* v_n, const double* f_ext, double h,
                                    const double* lambda, double rho, double* g_out,
                                    double* H_out, double* f_int_out, void* stream);

/* tlfea_constraint_residual — c_out DEVICE [m] = C q - b for DEVICE q [n_dof]. */
tlfea_status tlfea_constraint_residual(tlfea_ctx ctx, const double* q, double* c_out,
                                       void* stream);

/* tlfea_update_multipliers — the dual ascent step of the ALM outer loop,
 * lambda <- lambda + rho c(q) (Eq. lambda_update, Alg. 2):
 * lambda DEVICE [m] read and overwritten; c_out DEVICE [m] or NULL receives
 * c(q) (the outer stopping test ||c|| <= eps_out). */
tlfea_status tlfea_update_multipliers(tlfea_ctx ctx, const double* q, double rho,
                                      double* lambda, double* c_out, void* stream);

/* tlfea_force_only — f_int only (the AdamW inner evaluation, Alg. 2
 * P:617-621): DEVICE x, v (v may be NULL when damping is off), f_int_out
 * [3*n_owned_nodes]. */
tlfea_status tlfea_force_only(tlfea_ctx ctx, const double* x, const double* v,
                              double* f_int_out, void* stream);

/* AdamW hyper-parameters of Alg. 2: step alpha, moment decays
 * beta1 / beta2, eps, decoupled weight decay lambda_wd. */
typedef struct {
  double alpha, beta1, beta2, eps, weight_decay;
} tlfea_adamw_params;

/* tlfea_adamw_iteration — one inner AdamW iteration l >= 1 of Alg. 2
 * (SURVEY §8(f) NEXT-2), single-rank contexts:
 *   m <- b1 m + (1-b1) g;  s <- b2 s + (1-b2) g.g;
 *   m^ = m/(1-b1^l);  s^ = s/(1-b2^l);
 *   v <- (1 - alpha wd) v - alpha m^/(sqrt(s^) + eps);  q <- q_n + h v;
 *   f_int(q, v) (Stage 1 + 2; Kelvin-Voigt driven by the new v, reading Q9);
 *   g <- M (v - v_n)/h + f_int - f_ext - f_ff  (Eq. residual, reading Q10)
 *        + h C^T (lambda + rho c(q))  (with the context's constraints, NEXT-3);
 *   norms_out[0] = ||g||_2, norms_out[1] = ||v||_2 (the inner stopping test
 *   ||g|| <= eps_in (1 + ||v||)), reduced on the device in a fixed
 *   order (bitwise reproducible).
 * All vectors are DEVICE [3 n_coef], DOF-major: q_n, v_n read; f_ext read
 * (nullable = 0); v, m, s, g read AND overwritten (g on entry = the previous
 * iteration's gradient, zeros for l = 1 after a reset); q_out written;
 * f_int_out and norms_out (DEVICE [2]) nullable; lambda DEVICE [m] (NULL = 0)
 * and rho >= 0 enter only with constraints. Returns TLFEA_E_INVALID for
 * l < 1, rho < 0, NULL required pointers or a partitioned context. */
tlfea_status tlfea_adamw_iteration(tlfea_ctx ctx, const double* q_n, const double* v_n,
                                   const double* f_ext, double h, int32_t l,
                                   const tlfea_adamw_params* params, const double* lambda,
                                   double rho, double* v, double* m,
                                   double* s, double* g, double* q_out, double* f_int_out,
                                   double* norms_out, void* stream);

/* tlfea_eval_host — tlfea_eval with HOST buffers (end-to-end path): copies
 * x, v, v_n, f_ext host->device, evaluates, copies g, H (and f_int if
 * non-NULL) device->host, and synchronizes the stream before returning.
 * Host buffers may be pageable; pinned buffers are faster. */
tlfea_status tlfea_eval_host(tlfea_ctx ctx, const double* x, const double* v,
                             const double* v_n, const double* f_ext, double h,
                             double* g_out, double* H_out, double* f_int_out,
                             void* stream);

/* ----------------------------------------------- step-level entry points -- */

/* Stage 1 alone (compute_p): P_out DEVICE [n_el][n_qp][9]
 * (row-major 3x3, P_iJ at 3i+J) = P_el + P_vis at every local (e,q). */
tlfea_status tlfea_compute_stress(tlfea_ctx ctx, const double* x,
                                  const double* v, double* P_out, void* stream);

/* Stage 2 force alone (compute_internal_force, Eqs. fint_local/fint_global,
 * P:408-423): from a Stage-1 buffer P DEVICE [n_el][n_qp][9] to f_int_out
 * DEVICE [3*n_owned_nodes]. Single-rank contexts only. */
tlfea_status tlfea_internal_force_from_stress(tlfea_ctx ctx, const double* P,
                                              double* f_int_out, void* stream);

/* Residual alone (compute_grad_l, Eq. grad_L, P:459-489 without C_q):
 * g = (1/h) M (v - v_n) + f_int - f_ext - f_ff on the owned rows. f_int DEVICE
 * [3*n_owned_nodes]; v, v_n (nullable), f_ext (nullable) DEVICE global. */
tlfea_status tlfea_compute_gradient(tlfea_ctx ctx, const double* f_int,
                                    const double* v, const double* v_n,
                                    const double* f_ext, double h,
                                    double* g_out, void* stream);

/* Hessian alone (Eq. hessian + tangent_block): H_out DEVICE [nnz]
 * = M/h + h K_t(x). Single-rank contexts only. */
tlfea_status tlfea_assemble_hessian(tlfea_ctx ctx, const double* x, double h,
                                    double* H_out, void* stream);

/* ------------------------------------------------- multi-GPU partition -- */

/* Sizes of the boundary exchange of a partitioned context:
 * send_counts/recv_counts HOST int64 [nranks]: number of fp64 values this
 * rank sends to / receives from each peer per eval (partial H 3x3 blocks and
 * partial nodal forces of shared nodes). Peer buffers are laid out
 * contiguously in rank order; offsets are exclusive prefix sums. */
tlfea_status tlfea_exchange_sizes(tlfea_ctx ctx, int64_t* send_counts,
                                  int64_t* recv_counts);

/* The partitioned evaluation, three calls on one stream (the
 * exchange overlaps the interior elements, step 3):
 *  begin    : Stage 1 + 2 of the BOUNDARY elements (local elements with a
 *             node owned elsewhere; the context orders them first) and the
 *             pack of the non-owned partials (H 3x3 blocks, nodal forces) into
 *             send_buf (DEVICE [sum send_counts]). When the stream reaches the
 *             end of begin, send_buf is complete: the caller then starts the
 *             transfer send_buf -> peers' recv_buf (e.g. NCCL send/recv over
 *             NVLink on its own stream).
 *  interior : Stage 1 + 2 of the remaining local elements (concurrently with
 *             the transfer), then the owned rows of H (H_out) and of the
 *             nodal force from all local elements.
 *  finish   : once recv_buf has arrived (the caller orders its stream after
 *             the transfer): adds the received partials in ascending peer
 *             order (deterministic for a fixed partition) and completes g (and
 *             f_int_out if non-NULL).
 * force_only = 1 skips H (H_out may be NULL). Calling the three out of order
 * returns TLFEA_E_INVALID. A single-rank context accepts the same sequence
 * (no exchange). */
tlfea_status tlfea_eval_begin(tlfea_ctx ctx, const double* x, const double* v,
                              int32_t force_only, double h, double* H_out,
                              double* send_buf, void* stream);
tlfea_status tlfea_eval_interior(tlfea_ctx ctx, const double* x, const double* v,
                                 int32_t force_only, double h, double* H_out,
                                 void* stream);
tlfea_status tlfea_eval_finish(tlfea_ctx ctx, const double* recv_buf,
                               const double* v, const double* v_n,
                               const double* f_ext, double h,
                               int32_t force_only, double* g_out,
                               double* H_out, double* f_int_out, void* stream);

/* The library's own NCCL transport of the exchange (SURVEY §8(b) / §8(e)
 * steps 2-4), an alternative to moving send_buf / recv_buf yourself.
 * libnccl.so.2 is loaded at run time (TLFEA_E_NCCL if it cannot be).
 *  tlfea_nccl_get_unique_id: id_out HOST [TLFEA_NCCL_ID_BYTES], an ncclUniqueId
 *    made on one rank (rank 0) and handed to every rank out of band (e.g. a
 *    torch.distributed broadcast of the bytes).
 *  tlfea_nccl_attach: every rank of the partition, with the same id, creates
 *    the context's communicator (ncclCommInitRank over options.nranks,
 *    options.rank; collective: all ranks must call it), a communication stream
 *    and two events. Destroyed with the context.
 *  tlfea_eval_exchange: between tlfea_eval_begin and tlfea_eval_interior on
 *    the same stream: sends send_buf's per-peer segments and receives
 *    recv_buf's (DEVICE, tlfea_exchange_sizes layout) as one NCCL group of
 *    ncclSend / ncclRecv on the communication stream, which an event orders
 *    after begin's pack; tlfea_eval_interior then overlaps the transfer, and
 *    tlfea_eval_finish makes the stream wait for it (events only, no host
 *    synchronization). A single-rank context without a communicator: no-op. */
#define TLFEA_NCCL_ID_BYTES 128
tlfea_status tlfea_nccl_get_unique_id(void* id_out);
tlfea_status tlfea_nccl_attach(tlfea_ctx ctx, const void* id);
tlfea_status tlfea_eval_exchange(tlfea_ctx ctx, const double* send_buf,
                                 double* recv_buf, void* stream);

/* Global ids of the context's local elements, in its local order (the order
 * of tlfea_slot_map / tlfea_export_precompute rows; partitioned contexts put
 * the boundary elements first). out_host HOST int64 [n_elements]. */
tlfea_status tlfea_local_elements(tlfea_ctx ctx, int64_t* out_host);

/* Host-only partition planner (no GPU needed; used by setup and by the CPU
 * tests of the exchange protocol). Given the GLOBAL mesh connectivity
 * (n_en node/coefficient ids per element, ANCF: already expanded to the 16
 * coefficient ids) and elem_part, returns for `rank`:
 *   owner_out   HOST int32 [n_coef] owning rank of every coefficient
 *   The send lists, in canonical order (peer ascending, then (I,J)
 *   ascending): pairs (I,J) of coefficient blocks whose row I is owned by the
 *   peer and receives a contribution from this rank's elements; and nodes I
 *   (owned by the peer, touched by this rank).
 * Two-call protocol: call with NULL arrays to get the counts, then again. */
tlfea_status tlfea_plan_partition(int64_t n_elements, int32_t n_en,
                                  const int32_t* conn_coef, int64_t n_coef,
                                  const int32_t* elem_part, int32_t nranks,
                                  int32_t rank, int32_t* owner_out,
                                  int64_t* n_send_blocks, int64_t* send_blocks,
                                  int64_t* send_block_peer,
                                  int64_t* n_send_nodes, int64_t* send_nodes,
                                  int64_t* send_node_peer);

/* ------------------------------------------------------------ diagnostics -- */

/* Synchronizes the last eval stream and returns TLFEA_E_INVERTED_STATE with
 * the first (element, quadrature point) that had det F <= 0 under
 * Mooney-Rivlin, or TLFEA_OK. Resets the flag. */
tlfea_status tlfea_sync_status(tlfea_ctx ctx, int64_t* bad_elem,
                               int32_t* bad_qp);

/* Test hook: the device constitutive functions on a batch of n deformation
 * gradients. F, Fdot (nullable) DEVICE [n][9]; P_out DEVICE [n][9] total
 * stress P_el + P_vis; A_out DEVICE [n][81] (nullable) elastic tangent
 * A[(3i+J)*9 + 3k+L] = dP_iJ/dF_kL (Eq. tangent_block). Synchronizes. */
tlfea_status tlfea_test_constitutive(const tlfea_material* mat, int64_t n,
                                     const double* F, const double* Fdot,
                                     double* P_out, double* A_out);

/* Live per-kernel timing (bench.py roofline): with enable = 1 every eval
 * kernel of this context is bracketed by CUDA events recorded on its launch
 * stream. tlfea_timing_report synchronizes and returns, per kernel class
 * (0 element kernel, 1 H gather, 2 force gather / residual, 3 partition
 * pack/unpack, 4 fused persistent eval), the number of launches and their
 * summed duration in ms, and resets the record. counts/ms are HOST arrays of
 * length TLFEA_N_TIMING. */
#define TLFEA_N_TIMING 5
tlfea_status tlfea_set_timing(tlfea_ctx ctx, int32_t enable);
tlfea_status tlfea_timing_report(tlfea_ctx ctx, int64_t* counts, double* ms);

/* Number of kernels this library launched since load (for gpu_launches). */
int64_t tlfea_launch_count(void);

const char* tlfea_last_error(void);
int32_t tlfea_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TLFEA_H_ */
