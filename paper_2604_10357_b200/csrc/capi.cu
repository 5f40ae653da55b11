// capi.cu — the extern "C" boundary of libtlfea (include/tlfea.h). Argument
// checking and orchestration only; every step of the path runs in the kernels
// of setup.cu / eval.cu / partition.cu.
#include <algorithm>
#include <new>

#include "common.cuh"

using namespace tlfea;

struct tlfea_ctx_s {
  Context c;
};

#define CTX_OR_FAIL(ctx)                                                      \
  do {                                                                        \
    if (!(ctx)) return fail(TLFEA_E_INVALID, "NULL context");                 \
  } while (0)
#define TRY(expr)                      \
  do {                                 \
    tlfea_status st__ = (expr);        \
    if (st__ != TLFEA_OK) return st__; \
  } while (0)

static cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

static tlfea_status use_device(Context& c) {
  TL_CUDA(cudaSetDevice(c.device));
  return TLFEA_OK;
}

// CUDA events around one launch on its stream (tlfea_set_timing).
static cudaEvent_t take_event(Context& c) {
  if (!c.event_pool.empty()) {
    cudaEvent_t e = c.event_pool.back();
    c.event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
struct Timed {
  Context& c;
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  Timed(Context& c_, int k, cudaStream_t s_) : c(c_), kind(k), s(s_) {
    if (c.timing) {
      a = take_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~Timed() {
    if (a) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, s);
      c.timed.push_back({kind, a, b});
    }
  }
};
#define TIMED(kind, expr)          \
  do {                             \
    Timed t__(c, (kind), s);       \
    TRY(expr);                     \
  } while (0)

extern "C" {

int32_t tlfea_abi_version(void) { return TLFEA_ABI_VERSION; }
const char* tlfea_last_error(void) { return last_error(); }
int64_t tlfea_launch_count(void) { return launch_count(); }

tlfea_status tlfea_setup(const tlfea_mesh* mesh, const tlfea_material* mat, const tlfea_options* opts,
                         tlfea_ctx* out) {
  if (!out) return fail(TLFEA_E_INVALID, "NULL output context");
  *out = nullptr;
  tlfea_ctx_s* h = new (std::nothrow) tlfea_ctx_s();
  if (!h) return fail(TLFEA_E_OOM, "host allocation failed");
  tlfea_status st = setup_context(&h->c, mesh, mat, opts);
  if (st != TLFEA_OK) {
    std::string keep = last_error();
    delete h;
    cudaGetLastError();
    return fail(st, keep);
  }
  *out = h;
  return TLFEA_OK;
}

void tlfea_destroy(tlfea_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  cudaDeviceSynchronize();
  delete ctx;
}

tlfea_status tlfea_info(tlfea_ctx ctx, tlfea_info_t* o) {
  CTX_OR_FAIL(ctx);
  if (!o) return fail(TLFEA_E_INVALID, "NULL info");
  const Context& c = ctx->c;
  o->element = c.element;
  o->quadrature = c.quadrature;
  o->n_qp = c.nq;
  o->n_en = c.nen;
  o->n_elements = c.n_el;
  o->n_elements_global = c.n_el_global;
  o->n_coef = c.n_coef;
  o->n_dof = 3 * c.n_coef;
  o->nnz_coef = c.nnz_c;
  o->nnz = c.nnz_H;
  o->n_owned_nodes = c.n_own;
  o->affine = c.affine;
  o->rank = c.rank;
  o->nranks = c.nranks;
  o->device_bytes = c.device_bytes;
  o->n_geometry_classes = c.n_cls;
  o->fused_eval = eval_small_ok(&c) ? 1 : 0;
  o->n_constraints = c.n_con;
  o->reference_layout = c.n_cls > 0 ? 0 : (c.aff ? 2 : (c.jinv ? 3 : 1));
  o->kv_consistent_tangent = c.kvc;
  return TLFEA_OK;
}

tlfea_status tlfea_pattern(tlfea_ctx ctx, const int64_t** rowptr, const int32_t** cols) {
  CTX_OR_FAIL(ctx);
  if (rowptr) *rowptr = ctx->c.rowptr;
  if (cols) *cols = ctx->c.cols;
  return TLFEA_OK;
}

tlfea_status tlfea_coef_pattern(tlfea_ctx ctx, const int32_t** rowptr, const int32_t** cols) {
  CTX_OR_FAIL(ctx);
  if (rowptr) *rowptr = ctx->c.rowptr_c;
  if (cols) *cols = ctx->c.cols_c;
  return TLFEA_OK;
}

tlfea_status tlfea_owned_nodes(tlfea_ctx ctx, const int32_t** nodes) {
  CTX_OR_FAIL(ctx);
  if (nodes) *nodes = ctx->c.own_nodes;
  return TLFEA_OK;
}

tlfea_status tlfea_export_pattern(tlfea_ctx ctx, int64_t* rowptr_out, int32_t* cols_out, int32_t* rowptr_c_out,
                                  int32_t* cols_c_out, int32_t* owned_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
  if (rowptr_out) TL_CUDA(cudaMemcpyAsync(rowptr_out, c.rowptr, sizeof(int64_t) * (3 * c.n_own + 1), k, s));
  if (cols_out) TL_CUDA(cudaMemcpyAsync(cols_out, c.cols, sizeof(int32_t) * c.nnz_H, k, s));
  if (rowptr_c_out) TL_CUDA(cudaMemcpyAsync(rowptr_c_out, c.rowptr_c, sizeof(int32_t) * (c.n_own + 1), k, s));
  if (cols_c_out) TL_CUDA(cudaMemcpyAsync(cols_c_out, c.cols_c, sizeof(int32_t) * c.nnz_c, k, s));
  if (owned_out) TL_CUDA(cudaMemcpyAsync(owned_out, c.own_nodes, sizeof(int32_t) * c.n_own, k, s));
  return TLFEA_OK;
}

tlfea_status tlfea_slot_map(tlfea_ctx ctx, int64_t e_begin, int64_t e_count, int64_t* out_host) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!out_host || e_begin < 0 || e_count < 0 || e_begin + e_count > c.n_el)
    return fail(TLFEA_E_INVALID, "tlfea_slot_map: bad range or NULL output");
  TRY(use_device(c));
  const int nen = c.nen, nd = 3 * nen;
  std::vector<int32_t> sc((size_t)e_count * nen * nen);
  std::vector<int32_t> rowptr_c(c.n_own + 1), blk_row_dummy;
  if (e_count > 0)
    TL_CUDA(cudaMemcpy(sc.data(), c.slot_c + e_begin * nen * nen, sizeof(int32_t) * sc.size(), cudaMemcpyDeviceToHost));
  TL_CUDA(cudaMemcpy(rowptr_c.data(), c.rowptr_c, sizeof(int32_t) * (c.n_own + 1), cudaMemcpyDeviceToHost));
  // row of each referenced slot: the row block of a's coefficient
  std::vector<int32_t> conn((size_t)e_count * nen), own_idx(c.n_coef);
  if (e_count > 0)
    TL_CUDA(cudaMemcpy(conn.data(), c.conn + e_begin * nen, sizeof(int32_t) * conn.size(), cudaMemcpyDeviceToHost));
  TL_CUDA(cudaMemcpy(own_idx.data(), c.own_idx, sizeof(int32_t) * c.n_coef, cudaMemcpyDeviceToHost));
  // UPPER storage: slot of (a,d; b,f) only when col >= row (common.cuh layout)
  std::vector<int32_t> cols_c, ubase;
  if (c.upper) {
    cols_c.resize(c.nnz_c);
    ubase.resize(c.n_own + 1);
    TL_CUDA(cudaMemcpy(cols_c.data(), c.cols_c, sizeof(int32_t) * c.nnz_c, cudaMemcpyDeviceToHost));
    TL_CUDA(cudaMemcpy(ubase.data(), c.ubase, sizeof(int32_t) * (c.n_own + 1), cudaMemcpyDeviceToHost));
  }
  if (c.upper) {
    for (int64_t e = 0; e < e_count; ++e)
      for (int a = 0; a < nen; ++a) {
        const int32_t i = own_idx[conn[e * nen + a]];
        const int32_t b0 = rowptr_c[i], deg = rowptr_c[i + 1] - b0;
        const int32_t kd = (int32_t)(std::lower_bound(cols_c.begin() + b0, cols_c.begin() + b0 + deg,
                                                      conn[e * nen + a]) - (cols_c.begin() + b0));
        for (int b = 0; b < nen; ++b) {
          const int32_t k = sc[(e * nen + a) * nen + b] - b0 - kd, L = deg - kd - 1;
          for (int d = 0; d < 3; ++d)
            for (int f = 0; f < 3; ++f)
              out_host[(e * nd + 3 * a + d) * nd + 3 * b + f] =
                  (k < 0 || (k == 0 && f < d)) ? -1 : ubase[i] + 3 * k + f + d * (2 + 3 * L) - d * (d - 1) / 2;
        }
      }
    return TLFEA_OK;
  }
  // DOF slot = 9 rowptr_c[i] + 3 d deg_i + 3 (s_c - rowptr_c[i]) + f  (DOF lift)
  for (int64_t e = 0; e < e_count; ++e)
    for (int a = 0; a < nen; ++a) {
      const int32_t i = own_idx[conn[e * nen + a]];
      for (int b = 0; b < nen; ++b) {
        const int32_t s = sc[(e * nen + a) * nen + b];
        for (int d = 0; d < 3; ++d)
          for (int f = 0; f < 3; ++f) {
            int64_t v = -1;
            if (s >= 0 && i >= 0) {
              const int64_t b0 = rowptr_c[i], deg = rowptr_c[i + 1] - b0;
              v = 9 * b0 + 3 * d * deg + 3 * (s - b0) + f;
            }
            out_host[(e * nd + 3 * a + d) * nd + 3 * b + f] = v;
          }
      }
    }
  return TLFEA_OK;
}

tlfea_status tlfea_export_precompute(tlfea_ctx ctx, double* grad_out, double* J0w_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  if (grad_out)
    TL_CUDA(cudaMemcpyAsync(grad_out, c.gradN, sizeof(double) * c.n_el * c.nq * c.nen * 3, cudaMemcpyDeviceToDevice, s));
  if (J0w_out) TL_CUDA(cudaMemcpyAsync(J0w_out, c.J0w, sizeof(double) * c.n_el * c.nq, cudaMemcpyDeviceToDevice, s));
  return TLFEA_OK;
}

tlfea_status tlfea_export_mass(tlfea_ctx ctx, double* M_out, double* fff_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  if (M_out) TL_CUDA(cudaMemcpyAsync(M_out, c.M, sizeof(double) * c.nnz_c, cudaMemcpyDeviceToDevice, s));
  if (fff_out) TL_CUDA(cudaMemcpyAsync(fff_out, c.fff, sizeof(double) * 3 * c.n_own, cudaMemcpyDeviceToDevice, s));
  return TLFEA_OK;
}

static tlfea_status check_h(double h) {
  if (!(h > 0.0)) return fail(TLFEA_E_INVALID, "time step h must be > 0");
  return TLFEA_OK;
}

tlfea_status tlfea_eval(tlfea_ctx ctx, const double* x, const double* v, const double* v_n, const double* f_ext,
                        double h, double* g_out, double* H_out, double* f_int_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "partitioned context: use tlfea_eval_begin/finish");
  if (!x || !v || !g_out || !H_out) return fail(TLFEA_E_INVALID, "tlfea_eval: NULL x, v, g_out or H_out");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;
  c.eval_inv_h = 1.0 / h;
  if (eval_small_ok(&c)) {  // small class-mode T10 SVK meshes: one cooperative launch
    TIMED(4, launch_eval_small(&c, x, v, v_n, f_ext, h, g_out, H_out, f_int_out, s));
    return TLFEA_OK;
  }
  TIMED(0, launch_element_kernel(&c, x, v, true, s));
  TIMED(1, launch_gather_H(&c, h, H_out, s));
  TIMED(2, launch_gather_f(&c, v, v_n, f_ext, h, g_out, f_int_out, false, s));
  return TLFEA_OK;
}

tlfea_status tlfea_eval_constrained(tlfea_ctx ctx, const double* x, const double* v, const double* v_n,
                                    const double* f_ext, double h, const double* lambda, double rho, double* g_out,
                                    double* H_out, double* f_int_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!(rho >= 0.0)) return fail(TLFEA_E_INVALID, "tlfea_eval_constrained: rho must be >= 0");
  TRY(tlfea_eval(ctx, x, v, v_n, f_ext, h, g_out, H_out, f_int_out, stream));
  const cudaStream_t s = as_stream(stream);
  TIMED(2, launch_constraint_terms(&c, x, lambda, rho, h, g_out, H_out, s));
  return TLFEA_OK;
}

tlfea_status tlfea_constraint_residual(tlfea_ctx ctx, const double* q, double* c_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (c.n_con > 0 && (!q || !c_out)) return fail(TLFEA_E_INVALID, "tlfea_constraint_residual: NULL q or c_out");
  TRY(use_device(c));
  return launch_constraint_residual(&c, q, c_out, as_stream(stream));
}

tlfea_status tlfea_update_multipliers(tlfea_ctx ctx, const double* q, double rho, double* lambda, double* c_out,
                                      void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!(rho >= 0.0)) return fail(TLFEA_E_INVALID, "tlfea_update_multipliers: rho must be >= 0");
  if (c.n_con > 0 && (!q || !lambda)) return fail(TLFEA_E_INVALID, "tlfea_update_multipliers: NULL q or lambda");
  TRY(use_device(c));
  return launch_dual_update(&c, q, rho, lambda, c_out, as_stream(stream));
}

tlfea_status tlfea_force_only(tlfea_ctx ctx, const double* x, const double* v, double* f_int_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "partitioned context: use tlfea_eval_begin/finish");
  if (!x || !f_int_out) return fail(TLFEA_E_INVALID, "tlfea_force_only: NULL x or f_int_out");
  if (c.mat.kv && !v) return fail(TLFEA_E_INVALID, "tlfea_force_only: Kelvin-Voigt damping needs v");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;
  TIMED(0, launch_element_kernel(&c, x, v, false, s));
  TIMED(2, launch_gather_f(&c, nullptr, nullptr, nullptr, 1.0, nullptr, f_int_out, true, s));
  return TLFEA_OK;
}

tlfea_status tlfea_adamw_iteration(tlfea_ctx ctx, const double* q_n, const double* v_n, const double* f_ext,
                                   double h, int32_t l, const tlfea_adamw_params* params, const double* lambda,
                                   double rho, double* v, double* m, double* s_mom, double* g, double* q_out,
                                   double* f_int_out, double* norms_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (!(rho >= 0.0)) return fail(TLFEA_E_INVALID, "tlfea_adamw_iteration: rho must be >= 0");
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "tlfea_adamw_iteration: single-rank contexts only");
  if (l < 1) return fail(TLFEA_E_INVALID, "tlfea_adamw_iteration: iteration index l must be >= 1");
  if (!q_n || !v_n || !params || !v || !m || !s_mom || !g || !q_out)
    return fail(TLFEA_E_INVALID, "tlfea_adamw_iteration: NULL q_n, v_n, params, v, m, s, g or q_out");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;
  // (i) velocity update and step map
  const bool inr = !f_int_out && force_inertia_capable(&c);
  if (inr && !c.dvscr) TRY(c.alloc(&c.dvscr, (size_t)3 * c.n_coef));
  TIMED(2, launch_adamw_update(&c, l, *params, g, m, s_mom, v, q_n, h, q_out, s, inr ? v_n : nullptr,
                               inr ? c.dvscr : nullptr));
  // (iii)-(iv) Stage 1 + Stage 2 at q, (vi) gradient
  if (inr) {
    // straight-sided T10 SVK with classes: the element kernel adds each element's
    // inertia m_e (v - v_n)_e / h to its nodal forces (v - v_n written by the
    // update), so the gradient is the force-scratch sum minus f_ext, f_ff (no
    // mass-row SpMV; f_int is not formed)
    c.inr = true;
    c.eval_inv_h = 1.0 / h;
    tlfea_status st;
    {
      Timed t__(c, 0, s);
      st = launch_element_kernel(&c, q_out, c.dvscr, false, s);
    }
    c.inr = false;
    TRY(st);
    TIMED(2, launch_gradient_inertia(&c, f_ext, g, s));
  } else {
    TIMED(0, launch_element_kernel(&c, q_out, v, false, s));
    TIMED(2, launch_gather_f(&c, v, v_n, f_ext, h, g, f_int_out, false, s));
  }
  // (v) constraint residual and its gradient term
  TIMED(2, launch_constraint_terms(&c, q_out, lambda, rho, h, g, nullptr, s));
  // device ||g||, ||v|| for the inner stopping test
  if (norms_out) TIMED(2, launch_norms2(&c, g, v, norms_out, s));
  return TLFEA_OK;
}

tlfea_status tlfea_eval_host(tlfea_ctx ctx, const double* x, const double* v, const double* v_n,
                             const double* f_ext, double h, double* g_out, double* H_out, double* f_int_out,
                             void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "tlfea_eval_host: single-rank contexts only");
  if (!x || !v || !g_out || !H_out) return fail(TLFEA_E_INVALID, "tlfea_eval_host: NULL x, v, g_out or H_out");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  const int64_t nd = 3 * c.n_coef, nown = 3 * c.n_own, nnz = c.nnz_H;
  if (!c.h_x) {  // persistent device staging, allocated on first use
    TRY(c.alloc(&c.h_x, nd));
    TRY(c.alloc(&c.h_v, nd));
    TRY(c.alloc(&c.h_vn, nd));
    TRY(c.alloc(&c.h_fe, nd));
    TRY(c.alloc(&c.h_g, std::max<int64_t>(nown, 1)));
    TRY(c.alloc(&c.h_H, std::max<int64_t>(nnz, 1)));
    TRY(c.alloc(&c.h_f, std::max<int64_t>(nown, 1)));
  }
  double* dx = c.h_x;
  double* dv = c.h_v;
  double* dvn = v_n ? c.h_vn : nullptr;
  double* dfe = f_ext ? c.h_fe : nullptr;
  double* dg = c.h_g;
  double* dH = c.h_H;
  double* df = f_int_out ? c.h_f : nullptr;
  auto cleanup = [&]() {};
  cudaError_t err = cudaSuccess;
  if (err == cudaSuccess) err = cudaMemcpyAsync(dx, x, sizeof(double) * nd, cudaMemcpyHostToDevice, s);
  if (err == cudaSuccess) err = cudaMemcpyAsync(dv, v, sizeof(double) * nd, cudaMemcpyHostToDevice, s);
  if (err == cudaSuccess && v_n) err = cudaMemcpyAsync(dvn, v_n, sizeof(double) * nd, cudaMemcpyHostToDevice, s);
  if (err == cudaSuccess && f_ext) err = cudaMemcpyAsync(dfe, f_ext, sizeof(double) * nd, cudaMemcpyHostToDevice, s);
  if (err != cudaSuccess) {
    cleanup();
    cudaGetLastError();
    return fail(err == cudaErrorMemoryAllocation ? TLFEA_E_OOM : TLFEA_E_CUDA,
                std::string("tlfea_eval_host staging: ") + cudaGetErrorString(err));
  }
  tlfea_status st = tlfea_eval(ctx, dx, dv, dvn, dfe, h, dg, dH, df, stream);
  if (st == TLFEA_OK) {
    err = cudaMemcpyAsync(g_out, dg, sizeof(double) * nown, cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = cudaMemcpyAsync(H_out, dH, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess && f_int_out)
      err = cudaMemcpyAsync(f_int_out, df, sizeof(double) * nown, cudaMemcpyDeviceToHost, s);
  }
  cleanup();
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (st != TLFEA_OK) return st;
  if (err != cudaSuccess || e2 != cudaSuccess)
    return fail(TLFEA_E_CUDA, std::string("tlfea_eval_host copy-back: ") +
                                  cudaGetErrorString(err != cudaSuccess ? err : e2));
  return TLFEA_OK;
}

tlfea_status tlfea_compute_stress(tlfea_ctx ctx, const double* x, const double* v, double* P_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!x || !P_out) return fail(TLFEA_E_INVALID, "tlfea_compute_stress: NULL x or P_out");
  TRY(use_device(c));
  c.last_stream = as_stream(stream);
  return launch_stress_only(&c, x, v, P_out, as_stream(stream));
}

tlfea_status tlfea_internal_force_from_stress(tlfea_ctx ctx, const double* P, double* f_int_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "single-rank contexts only");
  if (!P || !f_int_out) return fail(TLFEA_E_INVALID, "NULL P or f_int_out");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  TRY(launch_force_from_stress(&c, P, s));
  return launch_gather_f(&c, nullptr, nullptr, nullptr, 1.0, nullptr, f_int_out, true, s);
}

tlfea_status tlfea_compute_gradient(tlfea_ctx ctx, const double* f_int, const double* v, const double* v_n,
                                    const double* f_ext, double h, double* g_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (!f_int || !v || !g_out) return fail(TLFEA_E_INVALID, "NULL f_int, v or g_out");
  TRY(use_device(c));
  return launch_residual(&c, f_int, v, v_n, f_ext, h, g_out, as_stream(stream));
}

tlfea_status tlfea_assemble_hessian(tlfea_ctx ctx, const double* x, double h, double* H_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (c.nranks > 1) return fail(TLFEA_E_INVALID, "single-rank contexts only");
  if (!x || !H_out) return fail(TLFEA_E_INVALID, "NULL x or H_out");
  if (c.kvc) return fail(TLFEA_E_INVALID, "kv_consistent_tangent context: the tangent needs v (use tlfea_eval)");
  // the tangent is elastic only (reading Q8): evaluated without velocities
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;  // tlfea_sync_status waits on it (MR det F <= 0 flag)
  TIMED(0, launch_element_kernel(&c, x, nullptr, true, s));
  TIMED(1, launch_gather_H(&c, h, H_out, s));
  return TLFEA_OK;
}

tlfea_status tlfea_exchange_sizes(tlfea_ctx ctx, int64_t* send_counts, int64_t* recv_counts) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  for (int p = 0; p < c.nranks; ++p) {
    if (send_counts) send_counts[p] = c.nranks > 1 ? c.send_counts[p] : 0;
    if (recv_counts) recv_counts[p] = c.nranks > 1 ? c.recv_counts[p] : 0;
  }
  return TLFEA_OK;
}

tlfea_status tlfea_eval_begin(tlfea_ctx ctx, const double* x, const double* v, int32_t force_only, double h,
                              double* H_out, double* send_buf, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (!x || (!force_only && !H_out)) return fail(TLFEA_E_INVALID, "tlfea_eval_begin: NULL x or H_out");
  if (c.mat.kv && !v) return fail(TLFEA_E_INVALID, "tlfea_eval_begin: Kelvin-Voigt damping needs v");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;
  c.eval_inv_h = 1.0 / h;
  // the boundary elements (local [0, n_el_bnd)) and the send buffer
  TIMED(0, launch_element_kernel(&c, x, v, !force_only, s, 0, c.nranks > 1 ? c.n_el_bnd : c.n_el));
  if (c.nranks > 1) {
    if (!send_buf) return fail(TLFEA_E_INVALID, "tlfea_eval_begin: NULL send_buf");
    TIMED(3, launch_pack_send(&c, send_buf, force_only != 0, s));
  }
  c.interior_pending = true;
  return TLFEA_OK;
}

tlfea_status tlfea_eval_interior(tlfea_ctx ctx, const double* x, const double* v, int32_t force_only, double h,
                                 double* H_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (!c.interior_pending) return fail(TLFEA_E_INVALID, "tlfea_eval_interior: call tlfea_eval_begin first");
  if (!x || (!force_only && !H_out)) return fail(TLFEA_E_INVALID, "tlfea_eval_interior: NULL x or H_out");
  if (c.mat.kv && !v) return fail(TLFEA_E_INVALID, "tlfea_eval_interior: Kelvin-Voigt damping needs v");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  c.last_stream = s;
  if (c.nranks > 1) TIMED(0, launch_element_kernel(&c, x, v, !force_only, s, c.n_el_bnd, c.n_el));
  // owned rows from the local elements: H blocks and the partial nodal forces
  if (!force_only) TIMED(1, launch_gather_H(&c, h, H_out, s));
  TIMED(2, launch_gather_f(&c, nullptr, nullptr, nullptr, h, nullptr, c.fpart, true, s));
  c.interior_pending = false;
  return TLFEA_OK;
}

tlfea_status tlfea_eval_finish(tlfea_ctx ctx, const double* recv_buf, const double* v, const double* v_n,
                               const double* f_ext, double h, int32_t force_only, double* g_out, double* H_out,
                               double* f_int_out, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(check_h(h));
  if (c.interior_pending) return fail(TLFEA_E_INVALID, "tlfea_eval_finish: call tlfea_eval_interior first");
  TRY(use_device(c));
  const cudaStream_t s = as_stream(stream);
  TRY(nccl_wait(&c, s));  // a library exchange (tlfea_eval_exchange) in flight
  if (c.nranks > 1) {
    if (!recv_buf) return fail(TLFEA_E_INVALID, "tlfea_eval_finish: NULL recv_buf");
    TIMED(3, launch_unpack_recv(&c, recv_buf, h, H_out, force_only != 0, s));
  }
  if (g_out) {
    if (!v) return fail(TLFEA_E_INVALID, "tlfea_eval_finish: residual needs v");
    TIMED(2, launch_residual(&c, c.fpart, v, v_n, f_ext, h, g_out, s));
  }
  if (f_int_out)
    TL_CUDA(cudaMemcpyAsync(f_int_out, c.fpart, sizeof(double) * 3 * c.n_own, cudaMemcpyDeviceToDevice, s));
  return TLFEA_OK;
}

tlfea_status tlfea_nccl_get_unique_id(void* id_out) {
  if (!id_out) return fail(TLFEA_E_INVALID, "NULL id_out");
  return nccl_get_unique_id(id_out);
}

tlfea_status tlfea_nccl_attach(tlfea_ctx ctx, const void* id) {
  CTX_OR_FAIL(ctx);
  if (!id) return fail(TLFEA_E_INVALID, "NULL NCCL unique id");
  Context& c = ctx->c;
  TRY(use_device(c));
  return nccl_attach(&c, id);
}

tlfea_status tlfea_eval_exchange(tlfea_ctx ctx, const double* send_buf, double* recv_buf, void* stream) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!c.interior_pending) return fail(TLFEA_E_INVALID, "tlfea_eval_exchange: call tlfea_eval_begin first");
  int64_t ns = 0, nr = 0;
  for (int p = 0; p < c.nranks && c.nranks > 1; ++p) {
    ns += c.send_counts[p];
    nr += c.recv_counts[p];
  }
  if ((ns > 0 && !send_buf) || (nr > 0 && !recv_buf)) return fail(TLFEA_E_INVALID, "tlfea_eval_exchange: NULL buffer");
  TRY(use_device(c));
  if (c.nranks == 1 && !c.nccl_comm) return TLFEA_OK;  // nothing to move
  return nccl_exchange(&c, send_buf, recv_buf, as_stream(stream));
}

tlfea_status tlfea_local_elements(tlfea_ctx ctx, int64_t* out_host) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  if (!out_host) return fail(TLFEA_E_INVALID, "tlfea_local_elements: NULL output");
  TRY(use_device(c));
  if (c.n_el > 0) TL_CUDA(cudaMemcpy(out_host, c.elem_gid, sizeof(int64_t) * c.n_el, cudaMemcpyDeviceToHost));
  return TLFEA_OK;
}

tlfea_status tlfea_sync_status(tlfea_ctx ctx, int64_t* bad_elem, int32_t* bad_qp) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(use_device(c));
  TL_CUDA(cudaStreamSynchronize(c.last_stream));
  unsigned long long flag = 0;
  TL_CUDA(cudaMemcpy(&flag, c.err_flag, sizeof(flag), cudaMemcpyDeviceToHost));
  if (flag == ~0ull) {
    if (bad_elem) *bad_elem = -1;
    if (bad_qp) *bad_qp = -1;
    return TLFEA_OK;
  }
  const unsigned long long none = ~0ull;
  TL_CUDA(cudaMemcpy(c.err_flag, &none, sizeof(none), cudaMemcpyHostToDevice));
  int64_t gid = 0;
  TL_CUDA(cudaMemcpy(&gid, c.elem_gid + (flag / 64), sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (bad_elem) *bad_elem = gid;
  if (bad_qp) *bad_qp = (int32_t)(flag % 64);
  return fail(TLFEA_E_INVERTED_STATE, "Mooney-Rivlin det F <= 0 at element " + std::to_string(gid) + ", qp " +
                                          std::to_string(flag % 64));
}

tlfea_status tlfea_set_timing(tlfea_ctx ctx, int32_t enable) {
  CTX_OR_FAIL(ctx);
  ctx->c.timing = enable != 0;
  return TLFEA_OK;
}

tlfea_status tlfea_timing_report(tlfea_ctx ctx, int64_t* counts, double* ms) {
  CTX_OR_FAIL(ctx);
  Context& c = ctx->c;
  TRY(use_device(c));
  for (int k = 0; k < TLFEA_N_TIMING; ++k) {
    if (counts) counts[k] = 0;
    if (ms) ms[k] = 0.0;
  }
  for (auto& t : c.timed) {
    TL_CUDA(cudaEventSynchronize(t.stop));
    float el = 0.f;
    TL_CUDA(cudaEventElapsedTime(&el, t.start, t.stop));
    if (t.kind >= 0 && t.kind < TLFEA_N_TIMING) {
      if (counts) counts[t.kind] += 1;
      if (ms) ms[t.kind] += el;
    }
    c.event_pool.push_back(t.start);
    c.event_pool.push_back(t.stop);
  }
  c.timed.clear();
  return TLFEA_OK;
}

tlfea_status tlfea_test_constitutive(const tlfea_material* mat, int64_t n, const double* F, const double* Fdot,
                                     double* P_out, double* A_out) {
  if (!mat || !F || !P_out || n < 0) return fail(TLFEA_E_INVALID, "tlfea_test_constitutive: bad arguments");
  return launch_test_constitutive(make_matdev(*mat), n, F, Fdot, P_out, A_out);
}

}  // extern "C"
