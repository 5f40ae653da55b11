"""CPU oracle for arXiv 2604.10357's hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  The product path
(``paper_2604_10357_b200`` / ``libtlfea.so``) never imports it and shares no
code with it.  The arithmetic lives in ``tlfea_oracle.cpp`` (plain fp64 C++,
``-O2 -ffp-contract=off``, single thread, per-element loops); this module only
builds it, marshals numpy arrays and orchestrates setup -> eval in the order
of the paper (precompute §4.1, pattern §4.2, mass, Stage 1/2 §4.3, gradient
§4.4.1, Hessian §4.4.2).

Parity status per function: see the header of tlfea_oracle.cpp and DESIGN.md
("Oracle pins").  The ANCF3443 basis is "parity unpinned" against the paper's
own (unavailable, Part I) element definition; it is pinned by invariants only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tlfea_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_lock = threading.Lock()
_lib = None
_lib_omp = None

MAT_FIELDS = ("E", "nu", "C10", "C01", "kappa", "rho0", "eta_damp", "lambda_damp")


def build(force: bool = False, openmp: bool = False) -> str:
    """Compile the oracle (g++, fp64, no FMA contraction). openmp: the same
    source with -fopenmp (liboracle_omp.so, the all-core CPU baseline: only
    orc_eval_chunked runs on several threads)."""
    out = _LIB_OMP if openmp else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-std=c++17", "-shared",
                               "-fPIC", *(["-fopenmp"] if openmp else []), "-o", tmp, _SRC])
        os.replace(tmp, out)
    return out


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = C.CDLL(build())
            _declare(_lib)
    return _lib


def lib_omp():
    """The OpenMP build (all-core element loop of orc_eval_chunked)."""
    global _lib_omp
    with _lock:
        if _lib_omp is None:
            _lib_omp = C.CDLL(build(openmp=True))
            _declare(_lib_omp)
    return _lib_omp


def max_threads() -> int:
    return int(lib_omp().orc_max_threads())


_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)


def _declare(L):
    i, i64, d = C.c_int, C.c_int64, C.c_double
    L.orc_quadrature.argtypes = [i, _d, _d]
    L.orc_quadrature.restype = i
    L.orc_t10_shape.argtypes = [_d, _d, _d]
    L.orc_t10_shape_csd.argtypes = [_d, i, _d]
    L.orc_ancf_shape.argtypes = [_d, _d, _d, _d]
    L.orc_ancf_shape_csd.argtypes = [_d, _d, i, _d]
    L.orc_beam_shape.argtypes = [_d, _d, _d, _d]
    L.orc_beam_shape_csd.argtypes = [_d, _d, i, _d]
    L.orc_precompute.argtypes = [i, i, i64, _i32, _d, _d, _d, _d]
    L.orc_precompute.restype = i64
    L.orc_coef_pattern.argtypes = [i, i64, _i32, i64, _i64, _i64]
    L.orc_coef_pattern.restype = i64
    L.orc_lift.argtypes = [i64, _i64, _i64, _i64, _i64]
    L.orc_slot_map.argtypes = [i, i64, _i32, _i64, _i64, _i64]
    L.orc_mass.argtypes = [i, i, i, d, i64, _i32, _d, _d, i64, _i64, _i64, _d]
    L.orc_element_mass.argtypes = [i, i, i, d, _i32, _d, _d, _d]
    L.orc_force_field.argtypes = [i64, _i64, _d, _d, _d]
    L.orc_pk1.argtypes = [i, _d, _d, _d, _d]
    L.orc_pk1_elastic.argtypes = [i, _d, _d, _d]
    L.orc_pk1_viscous.argtypes = [_d, _d, _d, _d]
    L.orc_energy.argtypes = [i, _d, _d]
    L.orc_energy.restype = d
    L.orc_energy_grad_csd.argtypes = [i, _d, _d, _d]
    L.orc_tangent.argtypes = [i, _d, _d, _d]
    L.orc_element.argtypes = [i, i, i, _d, _i32, _d, _d, _d, _d, _d, _d]
    L.orc_element_energy.argtypes = [i, i, i, _d, _i32, _d, _d, _d]
    L.orc_element_energy.restype = d
    L.orc_element_energy_grad_csd.argtypes = [i, i, i, _d, _i32, _d, _d, _d, _d]
    L.orc_stress.argtypes = [i, i, i, _d, i64, _i32, _d, _d, _d, _d, _d]
    L.orc_force_from_stress.argtypes = [i, i, i64, _i32, _d, _d, _d, i64, _d]
    L.orc_eval.argtypes = [i, i, i, _d, i64, _i32, i64, _d, _d, _i64, _i64, _d, _d, _i64, _i64,
                           _d, _d, _d, _d, d, _d, _d, _d]
    L.orc_eval_chunked.argtypes = L.orc_eval.argtypes
    L.orc_eval_kvc.argtypes = L.orc_eval.argtypes
    L.orc_element_force_local.argtypes = [i, i, i, _d, _i32, _d, _d, _d, _d, _d]
    L.orc_element_kvc.argtypes = [i, i, i, _d, _i32, _d, _d, _d, _d, d, _d]
    L.orc_max_threads.restype = i
    L.orc_eval_rows.argtypes = [i, i, i, i, _d, _i32, _d, _d, _d, _d, d, i64, _i64, _i64, _i64,
                                i64, _i64, _d, _d, _d]
    L.orc_eval_rows.restype = i64
    L.orc_adamw_update.argtypes = [i64, i, _d, _d, _d, _d, _d, _d, d, _d]


def _p(a, kind=_d):
    if a is None:
        return None
    return a.ctypes.data_as(kind)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32a(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def mat_array(mat: dict) -> np.ndarray:
    return np.array([float(mat.get(k, 0.0)) for k in MAT_FIELDS], dtype=np.float64)


def n_en(elem: int) -> int:
    return {0: 10, 1: 16, 2: 8}[int(elem)]


# ------------------------------------------------------------ primitives --

def quadrature(rule: int):
    pts = np.zeros((48, 3))
    w = np.zeros(48)
    n = lib().orc_quadrature(rule, _p(pts), _p(w))
    return pts[:n].copy(), w[:n].copy()


def t10_shape(xi):
    xi = _f64(xi)
    N = np.zeros(10)
    dN = np.zeros((10, 3))
    lib().orc_t10_shape(_p(xi), _p(N), _p(dN))
    return N, dN


def t10_shape_csd(xi, direction: int):
    xi = _f64(xi)
    out = np.zeros(10)
    lib().orc_t10_shape_csd(_p(xi), direction, _p(out))
    return out


def ancf_shape(xi, LWH):
    xi, LWH = _f64(xi), _f64(LWH)
    S = np.zeros(16)
    dS = np.zeros((16, 3))
    lib().orc_ancf_shape(_p(xi), _p(LWH), _p(S), _p(dS))
    return S, dS


def ancf_shape_csd(xi, LWH, direction: int):
    xi, LWH = _f64(xi), _f64(LWH)
    out = np.zeros(16)
    lib().orc_ancf_shape_csd(_p(xi), _p(LWH), direction, _p(out))
    return out


def beam_shape(xi, LWH):
    """ANCF3243 basis (reading Q23): S [8], dS/dxi [8][3]."""
    xi, LWH = _f64(xi), _f64(LWH)
    S = np.zeros(8)
    dS = np.zeros((8, 3))
    lib().orc_beam_shape(_p(xi), _p(LWH), _p(S), _p(dS))
    return S, dS


def beam_shape_csd(xi, LWH, direction: int):
    xi, LWH = _f64(xi), _f64(LWH)
    out = np.zeros(8)
    lib().orc_beam_shape_csd(_p(xi), _p(LWH), direction, _p(out))
    return out


def pk1(model, mat, F, Fdot=None):
    P = np.zeros(9)
    lib().orc_pk1(model, _p(mat_array(mat)), _p(_f64(np.ravel(F))),
                  _p(_f64(None if Fdot is None else np.ravel(Fdot))), _p(P))
    return P.reshape(3, 3)


def pk1_elastic(model, mat, F):
    P = np.zeros(9)
    lib().orc_pk1_elastic(model, _p(mat_array(mat)), _p(_f64(np.ravel(F))), _p(P))
    return P.reshape(3, 3)


def pk1_viscous(mat, F, Fdot):
    P = np.zeros(9)
    lib().orc_pk1_viscous(_p(mat_array(mat)), _p(_f64(np.ravel(F))), _p(_f64(np.ravel(Fdot))),
                          _p(P))
    return P.reshape(3, 3)


def energy(model, mat, F) -> float:
    return float(lib().orc_energy(model, _p(mat_array(mat)), _p(_f64(np.ravel(F)))))


def energy_grad_csd(model, mat, F):
    out = np.zeros(9)
    lib().orc_energy_grad_csd(model, _p(mat_array(mat)), _p(_f64(np.ravel(F))), _p(out))
    return out.reshape(3, 3)


def tangent(model, mat, F):
    """A[i,J,k,L] = dP_iJ/dF_kL (complex step)."""
    A = np.zeros(81)
    lib().orc_tangent(model, _p(mat_array(mat)), _p(_f64(np.ravel(F))), _p(A))
    return A.reshape(3, 3, 3, 3)


def element_mass(elem, rule, mass_rule, rho, conn_e, X, LWH=None):
    nen = n_en(elem)
    me = np.zeros(nen * nen)
    lib().orc_element_mass(elem, rule, mass_rule, rho, _p(_i32a(conn_e), _i32), _p(_f64(X)),
                           _p(_f64(LWH)), _p(me))
    return me.reshape(nen, nen)


def element(elem, rule, model, mat, conn_e, X, x, v=None, LWH=None, tangent=True):
    """(f_e [3 n_en], K_e [3n_en, 3n_en] or None) for one element; x, v global."""
    nd = 3 * n_en(elem)
    fe = np.zeros(nd)
    Ke = np.zeros(nd * nd) if tangent else None
    lib().orc_element(elem, rule, model, _p(mat_array(mat)), _p(_i32a(conn_e), _i32), _p(_f64(X)),
                      _p(_f64(LWH)), _p(_f64(x)), _p(_f64(v)), _p(fe), _p(Ke))
    return fe, (Ke.reshape(nd, nd) if tangent else None)


def element_force_local(elem, rule, model, mat, conn_e, X, xe, ve, LWH=None):
    """f_e [3 n_en] from LOCAL coordinates xe and velocities ve [3 n_en]."""
    fe = np.zeros(3 * n_en(elem))
    lib().orc_element_force_local(elem, rule, model, _p(mat_array(mat)), _p(_i32a(conn_e), _i32), _p(_f64(X)),
                                  _p(_f64(LWH)), _p(_f64(xe)), _p(_f64(ve)), _p(fe))
    return fe


def element_kvc(elem, rule, model, mat, conn_e, X, x, v, h, LWH=None):
    """Consistent Kelvin-Voigt element tangent Kc = h df/dx + df/dv [3n_en, 3n_en]
    (NEXT-4; complex step of the element force with x = q_n + h v)."""
    nd = 3 * n_en(elem)
    Kc = np.zeros(nd * nd)
    lib().orc_element_kvc(elem, rule, model, _p(mat_array(mat)), _p(_i32a(conn_e), _i32), _p(_f64(X)),
                          _p(_f64(LWH)), _p(_f64(x)), _p(_f64(v)), float(h), _p(Kc))
    return Kc.reshape(nd, nd)


def element_energy(elem, rule, model, mat, conn_e, X, xe, LWH=None) -> float:
    return float(lib().orc_element_energy(elem, rule, model, _p(mat_array(mat)),
                                          _p(_i32a(conn_e), _i32), _p(_f64(X)), _p(_f64(LWH)),
                                          _p(_f64(xe))))


def element_energy_grad_csd(elem, rule, model, mat, conn_e, X, xe, LWH=None):
    out = np.zeros(3 * n_en(elem))
    lib().orc_element_energy_grad_csd(elem, rule, model, _p(mat_array(mat)),
                                      _p(_i32a(conn_e), _i32), _p(_f64(X)), _p(_f64(LWH)),
                                      _p(_f64(xe)), _p(out))
    return out


# ------------------------------------------------------------- problem --

class Problem:
    """Setup (a-1, a-2) of one mesh: precompute, coefficient + DOF pattern,
    slot map (on demand), consistent mass and f_ff."""

    def __init__(self, mesh, mat: dict, rule: int, mass_rule: int = 0, gravity=(0.0, 0.0, 0.0),
                 with_precompute: bool = True, with_pattern: bool = True, constraints: dict | None = None):
        """constraints (NEXT-3, reading Q22): linear bilateral constraints
        c(q) = C q - b with a constant CSR Jacobian C (m x n_dof): dict
        rowptr [m+1], cols (DOF ids), vals, b [m]. Clamp rows are the special
        case C row = e_i, b = the clamped value. The H pattern is
        the union of the element couplings and C^T C's."""
        self.C = None
        if constraints is not None:
            self.C = {k: np.asarray(constraints[k]) for k in ("rowptr", "cols", "vals", "b")}
            self.C["rowptr"] = self.C["rowptr"].astype(np.int64)
            self.C["cols"] = self.C["cols"].astype(np.int64)
            self.C["vals"] = self.C["vals"].astype(np.float64)
            self.C["b"] = self.C["b"].astype(np.float64)
        self.mesh = mesh
        self.elem = int(mesh.element)
        self.rule = int(rule)
        self.mass_rule = int(mass_rule)
        self.mat = dict(mat)
        self.model = int(mat.get("model", 0))
        self.matv = mat_array(mat)
        self.conn = _i32a(mesh.conn)
        self.X = _f64(mesh.X)
        self.dims = _f64(mesh.dims) if mesh.dims is not None else None
        self.n_el = mesh.n_el
        self.n_coef = mesh.n_coef
        self.nen = n_en(self.elem)
        self.gravity = _f64(gravity)
        self.pts, self.w = quadrature(self.rule)
        self.nq = len(self.w)
        L = lib()
        if with_precompute:
            self.gradN = np.zeros((self.n_el, self.nq, self.nen, 3))
            self.J0w = np.zeros((self.n_el, self.nq))
            bad = L.orc_precompute(self.elem, self.rule, self.n_el, _p(self.conn, _i32), _p(self.X),
                                   _p(self.dims), _p(self.gradN), _p(self.J0w))
            if bad >= 0:
                raise ValueError(f"inverted element {bad}")
        if with_pattern:
            nnz = L.orc_coef_pattern(self.elem, self.n_el, _p(self.conn, _i32), self.n_coef, None, None)
            self.rowptr_c = np.zeros(self.n_coef + 1, np.int64)
            self.cols_c = np.zeros(nnz, np.int64)
            L.orc_coef_pattern(self.elem, self.n_el, _p(self.conn, _i32), self.n_coef,
                               _p(self.rowptr_c, _i64), _p(self.cols_c, _i64))
            if self.C is not None:
                # union with the coefficient couplings of every constraint row
                rows = [set(self.cols_c[self.rowptr_c[I]:self.rowptr_c[I + 1]].tolist())
                        for I in range(self.n_coef)]
                for k in range(self.C["b"].size):
                    coefs = {int(j) // 3 for j in self.C["cols"][self.C["rowptr"][k]:self.C["rowptr"][k + 1]]}
                    for I in coefs:
                        rows[I] |= coefs
                self.rowptr_c = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
                self.cols_c = np.array([j for r in rows for j in sorted(r)], np.int64)
                nnz = self.cols_c.size
            self.rowptr = np.zeros(3 * self.n_coef + 1, np.int64)
            self.cols = np.zeros(9 * nnz, np.int64)
            L.orc_lift(self.n_coef, _p(self.rowptr_c, _i64), _p(self.cols_c, _i64),
                       _p(self.rowptr, _i64), _p(self.cols, _i64))
            self.M = np.zeros(nnz)
            L.orc_mass(self.elem, self.rule, self.mass_rule, float(self.matv[5]), self.n_el,
                       _p(self.conn, _i32), _p(self.X), _p(self.dims), self.n_coef,
                       _p(self.rowptr_c, _i64), _p(self.cols_c, _i64), _p(self.M))
            self.fff = np.zeros(3 * self.n_coef)
            L.orc_force_field(self.n_coef, _p(self.rowptr_c, _i64), _p(self.M), _p(self.gravity),
                              _p(self.fff))

    @property
    def nnz_c(self):
        return int(self.cols_c.size)

    @property
    def nnz(self):
        return int(self.cols.size)

    def slot_map(self, e_begin: int = 0, e_count: int | None = None):
        if e_count is None:
            e_count = self.n_el - e_begin
        nd = 3 * self.nen
        out = np.zeros((e_count, nd, nd), np.int64)
        conn = np.ascontiguousarray(self.conn[e_begin:e_begin + e_count])
        lib().orc_slot_map(self.elem, e_count, _p(conn, _i32), _p(self.rowptr, _i64),
                           _p(self.cols, _i64), _p(out, _i64))
        return out

    def stress(self, x, v=None):
        P = np.zeros((self.n_el, self.nq, 9))
        lib().orc_stress(self.elem, self.rule, self.model, _p(self.matv), self.n_el,
                         _p(self.conn, _i32), _p(self.X), _p(self.dims), _p(_f64(x)), _p(_f64(v)),
                         _p(P))
        return P

    def force_from_stress(self, P):
        f = np.zeros(3 * self.n_coef)
        lib().orc_force_from_stress(self.elem, self.rule, self.n_el, _p(self.conn, _i32), _p(self.X),
                                    _p(self.dims), _p(_f64(P)), self.n_coef, _p(f))
        return f

    def eval(self, x, v, vn=None, fext=None, h=1e-3, hessian=True, use_fff=True, lam=None, rho=0.0,
             all_cores=False, kv_consistent=False):
        """Returns (g, H or None, f_int) on the full DOF pattern. With
        constraints: g += h C^T (lam + rho c(x)) (Eq. residual P:101-113,
        P:484-489) and H += h^2 rho C^T C (Eq. hessian).
        all_cores: the element loop on every host core (orc_eval_chunked of
        the OpenMP build; bitwise equal to the serial evaluation).
        kv_consistent (NEXT-4): H = M/h + sum_e (h df_e/dx + df_e/dv), the
        consistent Kelvin-Voigt tangent dg/dv (orc_eval_kvc), non-symmetric."""
        nd = 3 * self.n_coef
        g = np.zeros(nd)
        fint = np.zeros(nd)
        H = np.zeros(self.nnz) if hessian else None
        fn = lib_omp().orc_eval_chunked if all_cores else lib().orc_eval
        if kv_consistent and hessian:
            fn = lib().orc_eval_kvc
        fn(self.elem, self.rule, self.model, _p(self.matv), self.n_el,
                       _p(self.conn, _i32), self.n_coef, _p(self.X), _p(self.dims),
                       _p(self.rowptr_c, _i64), _p(self.cols_c, _i64), _p(self.M),
                       _p(self.fff if use_fff else None), _p(self.rowptr, _i64),
                       _p(self.cols, _i64), _p(_f64(x)), _p(_f64(v)), _p(_f64(vn)), _p(_f64(fext)),
                       float(h), _p(g), _p(H), _p(fint))
        if self.C is not None:
            C = self.C
            c = self.constraint_residual(x)
            y = (np.zeros_like(c) if lam is None else _f64(lam)) + rho * c
            for k in range(c.size):
                for p in range(C["rowptr"][k], C["rowptr"][k + 1]):
                    g[C["cols"][p]] += h * C["vals"][p] * y[k]
            if hessian:
                for k in range(c.size):
                    r = range(C["rowptr"][k], C["rowptr"][k + 1])
                    for p1 in r:
                        for p2 in r:
                            H[self.dof_slot(C["cols"][p1], C["cols"][p2])] += h * h * rho * C["vals"][p1] * C["vals"][p2]
        return g, H, fint

    def upper_view(self):
        """UPPER storage of H (NEXT-4, reading Q14): the entries with
        col >= row of the full DOF pattern, rows in order. Returns
        (rowptr_u, cols_u, index into the full value array)."""
        keep = self.cols >= np.repeat(np.arange(self.rowptr.size - 1), np.diff(self.rowptr))
        counts = np.add.reduceat(keep.astype(np.int64), self.rowptr[:-1]) if keep.size else np.zeros(0, np.int64)
        counts[np.diff(self.rowptr) == 0] = 0
        rowptr_u = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return rowptr_u, self.cols[keep], np.nonzero(keep)[0]

    def dof_slot(self, i: int, j: int) -> int:
        """CSR index of DOF entry (i, j) (binary search over the row's columns)."""
        a, b = self.rowptr[i], self.rowptr[i + 1]
        k = a + int(np.searchsorted(self.cols[a:b], j))
        if k >= b or self.cols[k] != j:
            raise KeyError((i, j))
        return k

    def constraint_residual(self, x):
        """c(q) = C q - b (reading Q22)."""
        C = self.C
        xq = _f64(x)
        c = -C["b"].copy()
        for k in range(c.size):
            for p in range(C["rowptr"][k], C["rowptr"][k + 1]):
                c[k] += C["vals"][p] * xq[C["cols"][p]]
        return c


ADAMW_FIELDS = ("alpha", "beta1", "beta2", "eps", "weight_decay")


def adamw_update(l: int, prm: dict, g, m, s, v, q_n, h):
    """Alg. 2 lines 6-10 for inner iteration l >= 1: returns the
    updated (m, s, v, q) (inputs are not modified)."""
    m, s, v = _f64(m).copy(), _f64(s).copy(), _f64(v).copy()
    q = np.zeros_like(v)
    p = np.array([prm[k] for k in ADAMW_FIELDS], np.float64)
    lib().orc_adamw_update(v.size, int(l), _p(p), _p(_f64(g)), _p(m), _p(s), _p(v), _p(_f64(q_n)), float(h), _p(q))
    return m, s, v, q


def adamw_iteration(problem: "Problem", l: int, prm: dict, q_n, v_n, fext, h, v, m, s, g, lam=None, rho=0.0):
    """One AdamW inner iteration of Alg. 2: the update above,
    then Stage 1 + Stage 2 at q = q_n + h v (Kelvin-Voigt driven by the new
    v, reading Q9) and the gradient g = M (v - v_n)/h + f_int - f_ext - f_ff
    (Eq. residual, reading Q10) + h C^T (lam + rho c(q)) when the problem has
    constraints. Returns (v, m, s, g, q, f_int, ||g||, ||v||)."""
    m, s, v, q = adamw_update(l, prm, g, m, s, v, q_n, h)
    g, _, f = problem.eval(q, v, v_n, fext, h, hessian=False, lam=lam, rho=rho)
    return v, m, s, g, q, f, float(np.linalg.norm(g)), float(np.linalg.norm(v))


def incidence(conn_coef: np.ndarray, nodes: np.ndarray):
    """For each node in `nodes`: ascending ids of the elements containing it."""
    nodes = np.asarray(nodes, np.int64)
    n_el, nen = conn_coef.shape
    flat = conn_coef.ravel().astype(np.int64)
    elem = np.repeat(np.arange(n_el, dtype=np.int64), nen)
    pos = {int(n): i for i, n in enumerate(nodes)}
    sel = np.isin(flat, nodes)
    lists = [[] for _ in nodes]
    for f, e in zip(flat[sel], elem[sel]):
        lists[pos[int(f)]].append(int(e))
    ptr = np.zeros(len(nodes) + 1, np.int64)
    ptr[1:] = np.cumsum([len(set(l)) for l in lists])
    inc = np.concatenate([np.array(sorted(set(l)), np.int64) for l in lists]) if len(nodes) else np.zeros(0, np.int64)
    return ptr, inc


def eval_rows(mesh, mat: dict, rule: int, mass_rule: int, x, v, h, nodes, max_cols: int = 96, inc=None):
    """Sampled-row oracle: for each coefficient node I in `nodes`, returns
    (cols [n][max_cols] coefficient columns (-1 padded), H [n][3][max_cols][3],
    f_int [n][3], M [n][max_cols]). Elements visited in ascending order.
    inc: optional (ptr, elements) incidence of `nodes` (as `incidence` returns)."""
    nodes = np.ascontiguousarray(nodes, np.int64)
    if inc is None:
        ptr, inc = incidence(mesh.coef_conn(), nodes)
    else:
        ptr, inc = (np.ascontiguousarray(a, np.int64) for a in inc)
    n = len(nodes)
    while True:
        cols = np.zeros((n, max_cols), np.int64)
        H = np.zeros((n, 3, max_cols, 3))
        f = np.zeros((n, 3))
        M = np.zeros((n, max_cols))
        need = lib().orc_eval_rows(int(mesh.element), rule, mass_rule, int(mat.get("model", 0)),
                                   _p(mat_array(mat)), _p(_i32a(mesh.conn), _i32), _p(_f64(mesh.X)),
                                   _p(_f64(mesh.dims)), _p(_f64(x)), _p(_f64(v)), float(h), n,
                                   _p(nodes, _i64), _p(ptr, _i64), _p(inc, _i64), max_cols,
                                   _p(cols, _i64), _p(H), _p(f), _p(M))
        if need <= max_cols:
            return cols, H, f, M
        max_cols = int(need)
