"""paper_2604_10357_b200 — B200-native (sm_100a, fp64) hot path of arXiv 2604.10357.

Thin Python binding of ``libtlfea.so`` (C ABI in ``include/tlfea.h``): argument
marshalling only. Every step of the path (precompute, pattern, slot map, mass,
Stage 1/2, tangent, deterministic CSR scatter, residual) runs in the CUDA
kernels of ``csrc/``. PyTorch supplies device memory, streams and
``torch.distributed``. There is no CPU fallback: if the library is missing or
no CUDA device is present, calls raise.

Function names follow the C ABI (``tlfea_setup``, ``tlfea_eval``,
``tlfea_force_only`` ...); :class:`Context` is a convenience owner of one
``tlfea_ctx``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ABI_VERSION = 8  # include/tlfea.h TLFEA_ABI_VERSION (struct layouts of this binding)
LIB_PATH = os.environ.get("TLFEA_LIB") or os.path.join(_HERE, "libtlfea.so")
_lib = None
_lock = threading.Lock()

T10, ANCF3443 = 0, 1
Q_T10_4PT, Q_T10_KEAST5, Q_GL_4x4x3 = 0, 1, 2
SVK, MOONEY_RIVLIN = 0, 1
STATUS = {0: "OK", 1: "INVALID", 2: "INVERTED_ELEMENT", 3: "INVERTED_STATE", 4: "OVERFLOW", 5: "OOM",
          6: "CUDA", 7: "UNSUPPORTED", 8: "NCCL"}


class TlfeaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"tlfea {STATUS.get(status, status)}: {msg}")
        self.status = status


class Material(C.Structure):
    _fields_ = [("model", C.c_int32), ("E", C.c_double), ("nu", C.c_double), ("C10", C.c_double),
                ("C01", C.c_double), ("kappa", C.c_double), ("rho0", C.c_double), ("eta_damp", C.c_double),
                ("lambda_damp", C.c_double)]


class Mesh(C.Structure):
    _fields_ = [("element", C.c_int32), ("n_elements", C.c_int64), ("n_coef", C.c_int64),
                ("conn", C.POINTER(C.c_int32)), ("X_ref", C.POINTER(C.c_double)),
                ("ancf_dims", C.POINTER(C.c_double))]


class Constraints(C.Structure):
    _fields_ = [("m", C.c_int64), ("rowptr", C.POINTER(C.c_int64)), ("cols", C.POINTER(C.c_int64)),
                ("vals", C.POINTER(C.c_double)), ("b", C.POINTER(C.c_double))]


class Options(C.Structure):
    _fields_ = [("quadrature", C.c_int32), ("mass_rule", C.c_int32), ("gravity", C.c_double * 3),
                ("ancf_dims", C.c_double * 3), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("elem_part", C.POINTER(C.c_int32)), ("device", C.c_int32),
                ("constraints", C.POINTER(Constraints)), ("hessian_upper", C.c_int32),
                ("reference_layout", C.c_int32), ("kv_consistent_tangent", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("element", C.c_int32), ("quadrature", C.c_int32), ("n_qp", C.c_int32), ("n_en", C.c_int32),
                ("n_elements", C.c_int64), ("n_elements_global", C.c_int64), ("n_coef", C.c_int64),
                ("n_dof", C.c_int64), ("nnz_coef", C.c_int64), ("nnz", C.c_int64), ("n_owned_nodes", C.c_int64),
                ("affine", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32), ("device_bytes", C.c_int64),
                ("n_geometry_classes", C.c_int32), ("fused_eval", C.c_int32), ("n_constraints", C.c_int64),
                ("reference_layout", C.c_int32), ("kv_consistent_tangent", C.c_int32)]

class AdamWParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double)]


N_TIMING = 5
TIMING_KINDS = ("element", "gather_H", "gather_f", "exchange", "fused")


_vp, _i64, _i32, _d = C.c_void_p, C.c_int64, C.c_int32, C.c_double
_SIGS = {
    "tlfea_setup": [C.POINTER(Mesh), C.POINTER(Material), C.POINTER(Options), C.POINTER(_vp)],
    "tlfea_destroy": [_vp],
    "tlfea_info": [_vp, C.POINTER(Info)],
    "tlfea_pattern": [_vp, C.POINTER(_vp), C.POINTER(_vp)],
    "tlfea_coef_pattern": [_vp, C.POINTER(_vp), C.POINTER(_vp)],
    "tlfea_owned_nodes": [_vp, C.POINTER(_vp)],
    "tlfea_slot_map": [_vp, _i64, _i64, _vp],
    "tlfea_export_pattern": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "tlfea_export_precompute": [_vp, _vp, _vp, _vp],
    "tlfea_export_mass": [_vp, _vp, _vp, _vp],
    "tlfea_eval": [_vp, _vp, _vp, _vp, _vp, _d, _vp, _vp, _vp, _vp],
    "tlfea_eval_constrained": [_vp, _vp, _vp, _vp, _vp, _d, _vp, _d, _vp, _vp, _vp, _vp],
    "tlfea_constraint_residual": [_vp, _vp, _vp, _vp],
    "tlfea_update_multipliers": [_vp, _vp, _d, _vp, _vp, _vp],
    "tlfea_force_only": [_vp, _vp, _vp, _vp, _vp],
    "tlfea_adamw_iteration": [_vp, _vp, _vp, _vp, _d, _i32, _vp, _vp, _d, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "tlfea_eval_host": [_vp, _vp, _vp, _vp, _vp, _d, _vp, _vp, _vp, _vp],
    "tlfea_compute_stress": [_vp, _vp, _vp, _vp, _vp],
    "tlfea_internal_force_from_stress": [_vp, _vp, _vp, _vp],
    "tlfea_compute_gradient": [_vp, _vp, _vp, _vp, _vp, _d, _vp, _vp],
    "tlfea_assemble_hessian": [_vp, _vp, _d, _vp, _vp],
    "tlfea_exchange_sizes": [_vp, _vp, _vp],
    "tlfea_eval_begin": [_vp, _vp, _vp, _i32, _d, _vp, _vp, _vp],
    "tlfea_eval_interior": [_vp, _vp, _vp, _i32, _d, _vp, _vp],
    "tlfea_eval_finish": [_vp, _vp, _vp, _vp, _vp, _d, _i32, _vp, _vp, _vp, _vp],
    "tlfea_nccl_get_unique_id": [_vp],
    "tlfea_nccl_attach": [_vp, _vp],
    "tlfea_eval_exchange": [_vp, _vp, _vp, _vp],
    "tlfea_local_elements": [_vp, _vp],
    "tlfea_plan_partition": [_i64, _i32, _vp, _i64, _vp, _i32, _i32, _vp, C.POINTER(_i64), _vp, _vp,
                             C.POINTER(_i64), _vp, _vp],
    "tlfea_sync_status": [_vp, C.POINTER(_i64), C.POINTER(_i32)],
    "tlfea_test_constitutive": [C.POINTER(Material), _i64, _vp, _vp, _vp, _vp],
    "tlfea_set_timing": [_vp, _i32],
    "tlfea_timing_report": [_vp, _vp, _vp],
    "tlfea_launch_count": [],
    "tlfea_last_error": [],
    "tlfea_abi_version": [],
}
EXPORTED = tuple(_SIGS)


def lib():
    """Load libtlfea.so (built in-tree by ``paper_2604_10357_b200.build``)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2604_10357_b200.build` "
                                   "(the CUDA library is required; there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = C.c_int
            L.tlfea_destroy.restype = None
            L.tlfea_launch_count.restype = C.c_int64
            L.tlfea_last_error.restype = C.c_char_p
            L.tlfea_abi_version.restype = C.c_int32
            if L.tlfea_abi_version() != ABI_VERSION:
                raise RuntimeError(f"{LIB_PATH}: ABI {L.tlfea_abi_version()}, binding expects {ABI_VERSION} (rebuild)")
            _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise TlfeaError(st, lib().tlfea_last_error().decode())


def _ptr(t):
    """Device/host address of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def make_material(mat: dict) -> Material:
    return Material(int(mat.get("model", 0)), *(float(mat.get(k, 0.0)) for k in
                                                 ("E", "nu", "C10", "C01", "kappa", "rho0", "eta_damp",
                                                  "lambda_damp")))


def launch_count() -> int:
    return int(lib().tlfea_launch_count())


def tlfea_test_constitutive(mat: dict, F, Fdot=None, with_tangent=True):
    """Device constitutive functions on a batch (torch CUDA tensors [n,9])."""
    import torch
    n = F.shape[0]
    P = torch.empty((n, 9), dtype=torch.float64, device=F.device)
    A = torch.empty((n, 81), dtype=torch.float64, device=F.device) if with_tangent else None
    m = make_material(mat)
    _check(lib().tlfea_test_constitutive(C.byref(m), n, _ptr(F), _ptr(Fdot), _ptr(P), _ptr(A)))
    return P, A


def tlfea_plan_partition(conn_coef: np.ndarray, n_coef: int, elem_part, nranks: int, rank: int):
    """Host-only partition planner (no GPU needed). Returns (owner [n_coef],
    send_blocks [n,2] (I,J), send_block_peer [n], send_nodes [m], send_node_peer [m])."""
    L = lib()
    conn_coef = np.ascontiguousarray(conn_coef, np.int32)
    n_el, nen = conn_coef.shape
    part = None if elem_part is None else np.ascontiguousarray(elem_part, np.int32)
    nb, nn = C.c_int64(0), C.c_int64(0)
    _check(L.tlfea_plan_partition(n_el, nen, _ptr(conn_coef), n_coef, _ptr(part), nranks, rank, None,
                                  C.byref(nb), None, None, C.byref(nn), None, None))
    owner = np.zeros(n_coef, np.int32)
    sb = np.zeros((nb.value, 2), np.int64)
    sbp = np.zeros(nb.value, np.int64)
    sn = np.zeros(nn.value, np.int64)
    snp = np.zeros(nn.value, np.int64)
    _check(L.tlfea_plan_partition(n_el, nen, _ptr(conn_coef), n_coef, _ptr(part), nranks, rank, _ptr(owner),
                                  C.byref(nb), _ptr(sb), _ptr(sbp), C.byref(nn), _ptr(sn), _ptr(snp)))
    return owner, sb, sbp, sn, snp


def nccl_unique_id() -> bytes:
    """tlfea_nccl_get_unique_id: the 128-byte NCCL unique id (made on one rank,
    handed to every rank of the partition out of band)."""
    buf = C.create_string_buffer(128)
    _check(lib().tlfea_nccl_get_unique_id(buf))
    return buf.raw


class Context:
    """Owns one tlfea_ctx (tlfea_setup ... tlfea_destroy)."""

    def __init__(self, element: int, conn: np.ndarray, X: np.ndarray, mat: dict, quadrature: int,
                 dims: np.ndarray | None = None, mass_rule: int = 0, gravity=(0.0, 0.0, 0.0),
                 rank: int = 0, nranks: int = 1, elem_part=None, device: int = 0, constraints: dict | None = None,
                 hessian: str = "full", reference_layout: str = "auto", kv_consistent: bool = False):
        """constraints: dict rowptr, cols (DOF ids), vals, b of c(q) = C q - b
        (tlfea_constraints; NEXT-3). hessian: "full" or "upper" storage of H
        (options.hessian_upper; NEXT-4). reference_layout: "auto" (geometry
        classes when the mesh allows) or "tables" (the paper's per-(e,q)
        tables always) or "affine" (the min layout of straight-sided T10
        before classes; options.reference_layout). kv_consistent: H is the
        consistent Kelvin-Voigt tangent dg/dv (options.kv_consistent_tangent;
        NEXT-4; non-symmetric, FULL storage, single rank)."""
        if hessian not in ("full", "upper"):
            raise ValueError("hessian must be 'full' or 'upper'")
        if reference_layout not in ("auto", "tables", "affine"):
            raise ValueError("reference_layout must be 'auto', 'tables' or 'affine'")
        L = lib()
        con = None
        if constraints is not None:
            self._con = [np.ascontiguousarray(constraints[k], t) for k, t in
                         (("rowptr", np.int64), ("cols", np.int64), ("vals", np.float64), ("b", np.float64))]
            p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))
            pd = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
            con = Constraints(self._con[3].size, p64(self._con[0]), p64(self._con[1]), pd(self._con[2]),
                              pd(self._con[3]))
        self._conn = np.ascontiguousarray(conn, np.int32)
        self._X = np.ascontiguousarray(X, np.float64)
        self._dims = None if dims is None else np.ascontiguousarray(dims, np.float64)
        self._part = None if elem_part is None else np.ascontiguousarray(elem_part, np.int32)
        mesh = Mesh(element, self._conn.shape[0], self._X.shape[0],
                    self._conn.ctypes.data_as(C.POINTER(C.c_int32)), self._X.ctypes.data_as(C.POINTER(C.c_double)),
                    None if self._dims is None else self._dims.ctypes.data_as(C.POINTER(C.c_double)))
        opts = Options(quadrature, mass_rule, (C.c_double * 3)(*gravity), (C.c_double * 3)(0, 0, 0), rank, nranks,
                       None if self._part is None else self._part.ctypes.data_as(C.POINTER(C.c_int32)), device,
                       None if con is None else C.pointer(con), 1 if hessian == "upper" else 0,
                       {"auto": 0, "tables": 1, "affine": 2}[reference_layout], 1 if kv_consistent else 0)
        self.material = dict(mat)
        m = make_material(mat)
        h = C.c_void_p()
        _check(L.tlfea_setup(C.byref(mesh), C.byref(m), C.byref(opts), C.byref(h)))
        self.handle = h
        self.device = device
        info = Info()
        _check(L.tlfea_info(h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in Info._fields_}

    @classmethod
    def from_mesh(cls, mesh, mat: dict, quadrature: int, **kw):
        """From a ``synth.Mesh``-like object (element, conn, X, dims)."""
        return cls(int(mesh.element), mesh.conn, mesh.X, mat, quadrature, dims=mesh.dims, **kw)

    def close(self):
        if getattr(self, "handle", None):
            lib().tlfea_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sizes
    @property
    def n_own(self):
        return self.info["n_owned_nodes"]

    @property
    def nnz(self):
        return self.info["nnz"]

    def _torch(self):
        import torch
        return torch

    @property
    def n_dof(self):
        return 3 * self.info["n_coef"]

    def _d(self, t, n, name):
        """Device pointer of a contiguous float64 CUDA tensor with >= n values
        on this context's device (argument checks only; None passes through)."""
        if t is None:
            return None
        torch = self._torch()
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.device.index != self.device:
            raise ValueError(f"{name}: expected a CUDA tensor on cuda:{self.device}")
        if t.dtype != torch.float64:
            raise ValueError(f"{name}: expected float64, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
        if t.numel() < n:
            raise ValueError(f"{name}: {t.numel()} values, {n} required")
        return C.c_void_p(t.data_ptr())

    def empty_outputs(self):
        torch = self._torch()
        dev = torch.device("cuda", self.device)
        g = torch.empty(3 * self.n_own, dtype=torch.float64, device=dev)
        H = torch.empty(self.nnz, dtype=torch.float64, device=dev)
        f = torch.empty(3 * self.n_own, dtype=torch.float64, device=dev)
        return g, H, f

    # -- exports
    def export_pattern(self, stream=None):
        """Copies (rowptr [3 n_own+1] int64, cols [nnz], rowptr_c [n_own+1], cols_c [nnz_coef],
        owned [n_own] int32) as CUDA tensors (tlfea_export_pattern)."""
        torch = self._torch()
        dev = torch.device("cuda", self.device)
        i = self.info
        out = [torch.empty(n, dtype=torch.int64 if k == 0 else torch.int32, device=dev) for k, n in
               enumerate((3 * self.n_own + 1, self.nnz, self.n_own + 1, i["nnz_coef"], self.n_own))]
        _check(lib().tlfea_export_pattern(self.handle, *[_ptr(t) for t in out], _stream(stream)))
        return tuple(out)

    def slot_map(self, e_begin=0, e_count=None):
        n = self.info["n_elements"]
        if e_count is None:
            e_count = n - e_begin
        nd = 3 * self.info["n_en"]
        out = np.zeros((e_count, nd, nd), np.int64)
        _check(lib().tlfea_slot_map(self.handle, e_begin, e_count, _ptr(out)))
        return out

    def export_precompute(self, stream=None):
        torch = self._torch()
        i = self.info
        dev = torch.device("cuda", self.device)
        gN = torch.empty((i["n_elements"], i["n_qp"], i["n_en"], 3), dtype=torch.float64, device=dev)
        Jw = torch.empty((i["n_elements"], i["n_qp"]), dtype=torch.float64, device=dev)
        _check(lib().tlfea_export_precompute(self.handle, _ptr(gN), _ptr(Jw), _stream(stream)))
        return gN, Jw

    def export_mass(self, stream=None):
        torch = self._torch()
        dev = torch.device("cuda", self.device)
        M = torch.empty(self.info["nnz_coef"], dtype=torch.float64, device=dev)
        fff = torch.empty(3 * self.n_own, dtype=torch.float64, device=dev)
        _check(lib().tlfea_export_mass(self.handle, _ptr(M), _ptr(fff), _stream(stream)))
        return M, fff

    # -- evaluation
    def _eval_ptrs(self, x, v, v_n, f_ext):
        n = self.n_dof
        return self._d(x, n, "x"), self._d(v, n, "v"), self._d(v_n, n, "v_n"), self._d(f_ext, n, "f_ext")

    def eval(self, x, v, v_n=None, f_ext=None, h=1e-3, g=None, H=None, f_int=None, stream=None, lam=None,
             rho=None):
        """tlfea_eval, or tlfea_eval_constrained when lam / rho are given."""
        if g is None or H is None:
            g0, H0, _ = self.empty_outputs()
            g = g0 if g is None else g
            H = H0 if H is None else H
        if lam is None and rho is None:
            _check(lib().tlfea_eval(self.handle, *self._eval_ptrs(x, v, v_n, f_ext), float(h),
                                    self._d(g, 3 * self.n_own, "g"), self._d(H, self.nnz, "H"),
                                    self._d(f_int, 3 * self.n_own, "f_int"), _stream(stream)))
        else:
            _check(lib().tlfea_eval_constrained(self.handle, *self._eval_ptrs(x, v, v_n, f_ext), float(h),
                                                self._d(lam, self.info["n_constraints"], "lam"), float(rho or 0.0),
                                                self._d(g, 3 * self.n_own, "g"), self._d(H, self.nnz, "H"),
                                                self._d(f_int, 3 * self.n_own, "f_int"), _stream(stream)))
        return g, H, f_int

    def constraint_residual(self, q, c=None, stream=None):
        """c(q) = C q - b on the device (tlfea_constraint_residual)."""
        torch = self._torch()
        if c is None:
            c = torch.empty(max(self.info["n_constraints"], 1), dtype=torch.float64, device=q.device)
        _check(lib().tlfea_constraint_residual(self.handle, _ptr(q), _ptr(c), _stream(stream)))
        return c

    def update_multipliers(self, q, rho, lam, c=None, stream=None):
        """lam += rho c(q) in place (tlfea_update_multipliers); returns c if given."""
        _check(lib().tlfea_update_multipliers(self.handle, _ptr(q), float(rho), _ptr(lam), _ptr(c), _stream(stream)))
        return c

    def force_only(self, x, v=None, f_int=None, stream=None):
        if f_int is None:
            f_int = self.empty_outputs()[2]
        _check(lib().tlfea_force_only(self.handle, self._d(x, self.n_dof, "x"), self._d(v, self.n_dof, "v"),
                                      self._d(f_int, 3 * self.n_own, "f_int"), _stream(stream)))
        return f_int

    def adamw_iteration(self, q_n, v_n, f_ext, h, l, params, v, m, s, g, q=None, f_int=None, norms=None,
                        stream=None, lam=None, rho=0.0):
        """tlfea_adamw_iteration: one AdamW inner iteration l >= 1 (Alg. 2).
        params: dict alpha, beta1, beta2, eps, weight_decay. v, m, s, g are
        CUDA tensors updated in place; returns (q, norms) with norms =
        [||g||, ||v||] on the device. lam / rho: constraint multipliers and
        penalty (contexts with constraints)."""
        import torch
        if q is None:
            q = torch.empty_like(v)
        if norms is None:
            norms = torch.empty(2, dtype=torch.float64, device=v.device)
        p = AdamWParams(*(float(params[k]) for k in ("alpha", "beta1", "beta2", "eps", "weight_decay")))
        n = self.n_dof
        d = self._d
        _check(lib().tlfea_adamw_iteration(self.handle, d(q_n, n, "q_n"), d(v_n, n, "v_n"), d(f_ext, n, "f_ext"),
                                           float(h), int(l), C.byref(p), d(lam, self.info["n_constraints"], "lam"),
                                           float(rho), d(v, n, "v"), d(m, n, "m"), d(s, n, "s"), d(g, n, "g"),
                                           d(q, n, "q"), d(f_int, n, "f_int"), d(norms, 2, "norms"),
                                           _stream(stream)))
        return q, norms

    def eval_host(self, x, v, v_n=None, f_ext=None, h=1e-3, g=None, H=None, f_int=None, stream=None):
        """Host (numpy or pinned CPU tensors) in and out; synchronizes."""
        _check(lib().tlfea_eval_host(self.handle, _ptr(x), _ptr(v), _ptr(v_n), _ptr(f_ext), float(h), _ptr(g),
                                     _ptr(H), _ptr(f_int), _stream(stream)))
        return g, H, f_int

    def compute_stress(self, x, v=None, P=None, stream=None):
        torch = self._torch()
        i = self.info
        if P is None:
            P = torch.empty((i["n_elements"], i["n_qp"], 9), dtype=torch.float64, device=x.device)
        _check(lib().tlfea_compute_stress(self.handle, self._d(x, self.n_dof, "x"), self._d(v, self.n_dof, "v"),
                                          self._d(P, i["n_elements"] * i["n_qp"] * 9, "P"), _stream(stream)))
        return P

    def internal_force_from_stress(self, P, f_int=None, stream=None):
        if f_int is None:
            f_int = self.empty_outputs()[2]
        i = self.info
        _check(lib().tlfea_internal_force_from_stress(self.handle, self._d(P, i["n_elements"] * i["n_qp"] * 9, "P"),
                                                      self._d(f_int, 3 * self.n_own, "f_int"), _stream(stream)))
        return f_int

    def compute_gradient(self, f_int, v, v_n=None, f_ext=None, h=1e-3, g=None, stream=None):
        if g is None:
            g = self.empty_outputs()[0]
        n = self.n_dof
        _check(lib().tlfea_compute_gradient(self.handle, self._d(f_int, 3 * self.n_own, "f_int"),
                                            self._d(v, n, "v"), self._d(v_n, n, "v_n"), self._d(f_ext, n, "f_ext"),
                                            float(h), self._d(g, 3 * self.n_own, "g"), _stream(stream)))
        return g

    def assemble_hessian(self, x, h=1e-3, H=None, stream=None):
        if H is None:
            H = self.empty_outputs()[1]
        _check(lib().tlfea_assemble_hessian(self.handle, self._d(x, self.n_dof, "x"), float(h),
                                            self._d(H, self.nnz, "H"), _stream(stream)))
        return H

    def exchange_sizes(self):
        P = self.info["nranks"]
        s = np.zeros(P, np.int64)
        r = np.zeros(P, np.int64)
        _check(lib().tlfea_exchange_sizes(self.handle, _ptr(s), _ptr(r)))
        return s, r

    def eval_begin(self, x, v, h, H, send_buf, force_only=False, stream=None):
        n = self.n_dof
        _check(lib().tlfea_eval_begin(self.handle, self._d(x, n, "x"), self._d(v, n, "v"), int(force_only), float(h),
                                      self._d(H, 0 if force_only else self.nnz, "H"),
                                      self._d(send_buf, int(self.exchange_sizes()[0].sum()), "send_buf"),
                                      _stream(stream)))

    def eval_interior(self, x, v, h, H, force_only=False, stream=None):
        """tlfea_eval_interior: the elements the exchange overlaps, then the
        owned rows (call between eval_begin and eval_finish)."""
        n = self.n_dof
        _check(lib().tlfea_eval_interior(self.handle, self._d(x, n, "x"), self._d(v, n, "v"), int(force_only),
                                         float(h), self._d(H, 0 if force_only else self.nnz, "H"), _stream(stream)))

    def nccl_attach(self, uid: bytes):
        """tlfea_nccl_attach (collective over the partition's ranks): the
        context's own NCCL communicator for eval_exchange."""
        if len(uid) != 128:
            raise ValueError("NCCL unique id: 128 bytes")
        _check(lib().tlfea_nccl_attach(self.handle, C.create_string_buffer(uid, 128)))

    def eval_exchange(self, send_buf, recv_buf, stream=None):
        """tlfea_eval_exchange: the library's NCCL transfer of the packed
        partials (between eval_begin and eval_interior on the same stream;
        eval_finish waits for it)."""
        s, r = self.exchange_sizes()
        _check(lib().tlfea_eval_exchange(self.handle, self._d(send_buf, int(s.sum()), "send_buf"),
                                         self._d(recv_buf, int(r.sum()), "recv_buf"), _stream(stream)))

    def local_elements(self):
        """Global ids of the local elements in the context's local order."""
        out = np.zeros(self.info["n_elements"], np.int64)
        _check(lib().tlfea_local_elements(self.handle, _ptr(out)))
        return out

    def eval_finish(self, recv_buf, v, v_n, f_ext, h, g, H, f_int=None, force_only=False, stream=None):
        n, no = self.n_dof, 3 * self.n_own
        _check(lib().tlfea_eval_finish(self.handle, self._d(recv_buf, int(self.exchange_sizes()[1].sum()), "recv_buf"),
                                       self._d(v, n, "v"), self._d(v_n, n, "v_n"), self._d(f_ext, n, "f_ext"),
                                       float(h), int(force_only), self._d(g, no, "g"),
                                       self._d(H, 0 if force_only else self.nnz, "H"), self._d(f_int, no, "f_int"),
                                       _stream(stream)))

    def set_timing(self, enable: bool):
        _check(lib().tlfea_set_timing(self.handle, int(enable)))

    def timing_report(self):
        """{kind: (launches, total_ms)} for kinds element / gather_H / gather_f / exchange / fused."""
        cnt = np.zeros(N_TIMING, np.int64)
        ms = np.zeros(N_TIMING, np.float64)
        _check(lib().tlfea_timing_report(self.handle, _ptr(cnt), _ptr(ms)))
        return {k: (int(cnt[i]), float(ms[i])) for i, k in enumerate(TIMING_KINDS)}

    def sync_status(self):
        e, q = C.c_int64(0), C.c_int32(0)
        st = lib().tlfea_sync_status(self.handle, C.byref(e), C.byref(q))
        if st == 3:
            return int(e.value), int(q.value)
        _check(st)
        return None
