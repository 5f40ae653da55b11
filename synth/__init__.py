"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no shape functions, quadrature,
stress, force or assembly): only mesh topology/geometry generators, seeded
deformation/velocity fields and the named BASELINE configurations.  Both the
CPU oracle (``oracle/``) and the CUDA path consume its output; neither is
imported here.

Input recipe:
  * T10 meshes: Kuhn 6-tetrahedron split of an nx*ny*nz cell box along the
    000->111 diagonal; nodes on the refined (2n+1)^3 grid, x slowest; elements
    lexicographic by cell then by the 6 permutations.  Odd permutations are
    negatively oriented and get corners 1<->2 swapped.  3x2x1 cells reproduce
    the paper's T10 RES0 row exactly: 105 nodes / 36 elements / 315 DOFs / 45
    clamped DOFs (PAPER.md Table "T10 beam mesh statistics").
  * ANCF3443 plates: n*n elements on a 4 x 2 plate, thickness 0.1;
    reproduces every row of PAPER.md Table P:1133-1138.
  * Deformation: cantilever bending u_z = -delta s^2 (3-s)/2, s = X/Lx,
    delta = 0.02 Lx, plus N(0,(0.01 l)^2) per coordinate (l = node spacing);
    v, v_n ~ N(0, 0.05^2).  Seeds: base 20261017 (+0 x, +1 v, +2 v_n, +3 f_ext,
    + body id for the many-body scene).
"""
from __future__ import annotations

import dataclasses
import numpy as np

SEED_BASE = 20261017

# T10 local node order (reading Q2): 4 corners, then edges
# (0,1),(1,2),(2,0),(0,3),(1,3),(2,3).
T10_EDGES = ((0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3))

_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_ODD = {(0, 2, 1), (1, 0, 2), (2, 1, 0)}


@dataclasses.dataclass
class Mesh:
    element: int            # 0 = T10, 1 = ANCF3443 (tlfea_element)
    X: np.ndarray           # [n_coef, 3] float64 reference coefficients
    conn: np.ndarray        # [n_el, n_nodes_per_el] int32 (T10: 10 nodes; ANCF: 4 nodes)
    dims: np.ndarray | None = None   # ANCF [n_el, 3] (L, W, H)
    body_of_elem: np.ndarray | None = None
    name: str = ""

    @property
    def n_el(self) -> int:
        return int(self.conn.shape[0])

    @property
    def n_coef(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_dof(self) -> int:
        return 3 * self.n_coef

    def coef_conn(self) -> np.ndarray:
        """Connectivity in coefficient ids ([n_el, n_en]); ANCF expands node k
        to coefficients 4k..4k+3 (reading Q11)."""
        if self.element == 0:
            return self.conn
        c = self.conn.astype(np.int64)
        out = (4 * c[:, :, None] + np.arange(4)[None, None, :]).reshape(c.shape[0], 4 * c.shape[1])
        return out.astype(np.int32)


def kuhn_t10_box(nx: int, ny: int, nz: int, Lx: float, Ly: float, Lz: float,
                 order: str = "lex") -> Mesh:
    """Kuhn-split T10 box mesh (straight-sided, so every element is affine)."""
    Nx, Ny, Nz = 2 * nx + 1, 2 * ny + 1, 2 * nz + 1
    ii, jj, kk = np.meshgrid(np.arange(Nx), np.arange(Ny), np.arange(Nz), indexing="ij")
    X = np.stack([ii.ravel() * (Lx / (2 * nx)), jj.ravel() * (Ly / (2 * ny)),
                  kk.ravel() * (Lz / (2 * nz))], axis=1).astype(np.float64)

    def nid(p):
        return (p[..., 0] * Ny + p[..., 1]) * Nz + p[..., 2]

    cells = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                                 indexing="ij"), axis=-1).reshape(-1, 3)
    if order == "morton":
        cells = cells[np.argsort(_morton3(cells), kind="stable")]
    elif order != "lex":
        raise ValueError(order)
    conns = []
    eye = np.eye(3, dtype=np.int64)
    for perm in _PERMS:
        v = [np.zeros(3, np.int64)]
        for ax in perm:
            v.append(v[-1] + eye[ax])
        if perm in _ODD:
            v[1], v[2] = v[2], v[1]
        corners = [2 * cells + 2 * vi[None, :] for vi in v]          # refined coords
        nodes = corners + [(corners[a] + corners[b]) // 2 for a, b in T10_EDGES]
        conns.append(np.stack([nid(p) for p in nodes], axis=1))
    conn = np.stack(conns, axis=1).reshape(-1, 10).astype(np.int32)
    return Mesh(0, X, conn, name=f"kuhn{nx}x{ny}x{nz}")


def perturbed(mesh: Mesh, amp: float = 0.05, seed: int = SEED_BASE + 7) -> Mesh:
    """Unstructured variant: every node (mid-edge nodes included, so edges
    become curved) moved by U(-amp, amp) x node spacing. No two elements stay
    congruent, which exercises the per-(e,q) reference-table path."""
    X = mesh.X + np.random.default_rng(seed).uniform(-amp, amp, mesh.X.shape) * _node_spacing(mesh.X)
    return Mesh(mesh.element, X, mesh.conn.copy(), mesh.dims, name=mesh.name + "_perturbed")


def perturbed_straight(mesh: Mesh, amp: float = 0.2, seed: int = SEED_BASE + 8) -> Mesh:
    """Straight-sided unstructured T10 variant: the element corners move by
    U(-amp, amp) x node spacing and every mid-edge node is put back at the
    middle of its edge, so the elements stay affine but no two are congruent
    (the affine "min" layout path)."""
    X = mesh.X.copy()
    corners = np.unique(mesh.conn[:, :4])
    X[corners] += np.random.default_rng(seed).uniform(-amp, amp, (corners.size, 3)) * _node_spacing(mesh.X)
    for m, (a, b) in enumerate(T10_EDGES):
        X[mesh.conn[:, 4 + m]] = 0.5 * (X[mesh.conn[:, a]] + X[mesh.conn[:, b]])
    return Mesh(0, X, mesh.conn.copy(), None, name=mesh.name + "_straight")


def _morton3(c: np.ndarray) -> np.ndarray:
    code = np.zeros(c.shape[0], dtype=np.int64)
    for bit in range(21):
        for ax in range(3):
            code |= ((c[:, ax].astype(np.int64) >> bit) & 1) << (3 * bit + ax)
    return code


def ancf_plate(n: int, Lx: float = 4.0, Ly: float = 2.0, H: float = 0.1) -> Mesh:
    """n x n ANCF3443 plate (§5.4). Coefficients per node:
    r = (x, y, 0), r_x = e1, r_y = e2, r_z = e3 (flat reference, reading Q11)."""
    nn = n + 1
    xs = np.arange(nn) * (Lx / n)
    ys = np.arange(nn) * (Ly / n)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")          # node id = i*nn + j
    n_nodes = nn * nn
    X = np.zeros((n_nodes, 4, 3))
    X[:, 0, 0] = gx.ravel()
    X[:, 0, 1] = gy.ravel()
    X[:, 1, 0] = 1.0
    X[:, 2, 1] = 1.0
    X[:, 3, 2] = 1.0
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    nid = lambda a, b: a * nn + b
    conn = np.stack([nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)], axis=1)
    dims = np.tile(np.array([Lx / n, Ly / n, H]), (n * n, 1))
    return Mesh(1, X.reshape(-1, 3), conn.astype(np.int32), dims, name=f"ancf{n}x{n}")


def ancf_plate_graded(n: int, ratio: float = 1.15, Lx: float = 4.0, Ly: float = 2.0, H: float = 0.1) -> Mesh:
    """n x n ANCF3443 plate whose element lengths along x grow geometrically
    by `ratio` (total Lx): n distinct element sizes, so no geometry classes
    (the per-(e,q) table path). Flat reference as in ancf_plate."""
    nn = n + 1
    steps = ratio ** np.arange(n)
    xs = np.concatenate([[0.0], np.cumsum(steps)]) * (Lx / steps.sum())
    ys = np.arange(nn) * (Ly / n)
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    X = np.zeros((nn * nn, 4, 3))
    X[:, 0, 0] = gx.ravel()
    X[:, 0, 1] = gy.ravel()
    X[:, 1, 0] = 1.0
    X[:, 2, 1] = 1.0
    X[:, 3, 2] = 1.0
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    nid = lambda a, b: a * nn + b
    conn = np.stack([nid(i, j), nid(i + 1, j), nid(i + 1, j + 1), nid(i, j + 1)], axis=1)
    dims = np.stack([xs[i + 1] - xs[i], np.full(n * n, Ly / n), np.full(n * n, H)], axis=1)
    return Mesh(1, X.reshape(-1, 3), conn.astype(np.int32), dims, name=f"ancf{n}x{n}_graded")


def ancf_beam(n: int, L: float = 0.2, W: float = 0.1, H: float = 0.1) -> Mesh:
    """Chain of n ANCF3243 beam elements along x (§5.3):
    element e spans nodes e and e+1, uniform L, rectangular W x H section.
    Coefficients per node: r = (x, 0, 0), r_x = e1, r_y = e2, r_z = e3
    (straight reference, reading Q23)."""
    nn = n + 1
    X = np.zeros((nn, 4, 3))
    X[:, 0, 0] = np.arange(nn) * L
    X[:, 1, 0] = 1.0
    X[:, 2, 1] = 1.0
    X[:, 3, 2] = 1.0
    conn = np.stack([np.arange(n), np.arange(1, nn)], axis=1).astype(np.int32)
    dims = np.tile(np.array([L, W, H]), (n, 1))
    return Mesh(2, X.reshape(-1, 3), conn, dims, name=f"beam{n}")


def clamped_dofs_t10(mesh: Mesh, tol: float = 1e-12) -> int:
    """DOFs on the x = 0 face (the clamped end of the paper's beams)."""
    return int(3 * np.count_nonzero(np.abs(mesh.X[:, 0]) < tol))


def clamped_dofs_ancf(mesh: Mesh, tol: float = 1e-12) -> int:
    pos = mesh.X.reshape(-1, 4, 3)[:, 0, :]
    return int(12 * np.count_nonzero(np.abs(pos[:, 0]) < tol))


def constraint_set(mesh: Mesh, seed: int = SEED_BASE + 20, n_ties: int = 4, tol: float = 1e-12) -> dict:
    """Linear bilateral constraints c(q) = C q - b (NEXT-3, reading Q22) as a
    CSR over DOFs: clamp rows (C row = e_i, b = the reference coordinate)
    for every DOF of the x = 0 face (T10 nodes; ANCF position coefficients),
    then `n_ties` random linear ties between two DOFs of different nodes
    elsewhere (coefficients N(0,1), b = 0). Inputs only — no method arithmetic."""
    rng = np.random.default_rng(seed)
    X = mesh.X
    if mesh.element == 0:
        face = np.nonzero(np.abs(X[:, 0]) < tol)[0]
    else:
        face = 4 * np.nonzero(np.abs(X.reshape(-1, 4, 3)[:, 0, 0]) < tol)[0]
    rows, cols, vals, b = [0], [], [], []
    for I in face:
        for d in range(3):
            cols.append(3 * int(I) + d)
            vals.append(1.0)
            b.append(float(X[I, d]))
            rows.append(len(cols))
    n_dof = 3 * mesh.n_coef
    for _ in range(n_ties):
        i, j = rng.choice(n_dof, 2, replace=False)
        while i // 3 == j // 3:
            j = int(rng.integers(n_dof))
        lo, hi = sorted((int(i), int(j)))
        cols += [lo, hi]
        vals += list(rng.normal(size=2))
        b.append(0.0)
        rows.append(len(cols))
    return dict(rowptr=np.array(rows, np.int64), cols=np.array(cols, np.int64),
                vals=np.array(vals, np.float64), b=np.array(b, np.float64))


# ------------------------------------------------------------------ fields --

def t10_state(mesh: Mesh, seed: int = SEED_BASE, bend: float = 0.02,
              noise: float = 0.01, vel: float = 0.05, with_fext: bool = False):
    """x = X + u (cantilever bending + noise), v, v_n, f_ext (optional)."""
    X = mesh.X
    Lx = float(X[:, 0].max() - X[:, 0].min()) or 1.0
    ell = _node_spacing(X)
    s = (X[:, 0] - X[:, 0].min()) / Lx
    delta = bend * Lx
    u = np.zeros_like(X)
    u[:, 2] = -delta * s * s * (3.0 - s) / 2.0
    rng = np.random.default_rng(seed + 0)
    u += rng.normal(0.0, noise * ell, size=X.shape)
    x = (X + u).ravel()
    v = np.random.default_rng(seed + 1).normal(0.0, vel, size=x.shape)
    vn = np.random.default_rng(seed + 2).normal(0.0, vel, size=x.shape)
    fext = np.random.default_rng(seed + 3).normal(0.0, 1.0, size=x.shape) if with_fext else None
    return x, v, vn, fext


def ancf_state(mesh: Mesh, seed: int = SEED_BASE, delta: float = 0.04,
               noise: float = 1e-3, vel: float = 0.05, length: float = 4.0):
    """Coefficients = exact position and gradients of
    phi(X) = X + (0, 0, delta (x/length)^2) at the nodes, plus N(0, noise^2)
    relative noise (length = 4 for the 4 x 2 plate; the beam
    chain uses its own length, delta scaled with it)."""
    Xc = mesh.X.reshape(-1, 4, 3)
    pos = Xc[:, 0, :]
    q = Xc.copy()
    q[:, 0, 2] = pos[:, 2] + delta * (pos[:, 0] / length) ** 2
    q[:, 1, 2] = 2.0 * delta * pos[:, 0] / (length * length)
    L = float(mesh.dims[0, 0]) if mesh.dims is not None else 1.0
    rng = np.random.default_rng(seed + 0)
    q[:, 0, :] += rng.normal(0.0, noise * L, size=pos.shape)
    q[:, 1:, :] += rng.normal(0.0, noise, size=q[:, 1:, :].shape)
    x = q.reshape(-1)
    v = np.random.default_rng(seed + 1).normal(0.0, vel, size=x.shape)
    vn = np.random.default_rng(seed + 2).normal(0.0, vel, size=x.shape)
    return x, v, vn


def _node_spacing(X: np.ndarray) -> float:
    spans = X.max(axis=0) - X.min(axis=0)
    # refined-grid spacing along the shortest-resolved axis
    best = np.inf
    for d in range(3):
        u = np.unique(np.round(X[:, d], 12))
        if u.size > 1:
            best = min(best, float(np.min(np.diff(u))))
    return best if np.isfinite(best) else float(spans.max())


def random_rotation(rng) -> np.ndarray:
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def many_body(n_bodies: int = 2000, cells=(9, 6, 3), size=(0.3, 0.2, 0.1),
              layout=(20, 10, 10), pitch: float = 0.5, strain: float = 0.05,
              seed: int = SEED_BASE, vel: float = 0.05):
    """Config 5: independent Kuhn T10 bodies on a grid; each body's current
    state is a random rotation times a random 5% homogeneous strain of its
    reference shape plus node noise. Returns (mesh, x, v)."""
    body = kuhn_t10_box(*cells, *size)
    nb_nodes, nb_el = body.n_coef, body.n_el
    center = body.X.mean(axis=0)
    Xs, xs, conns = [], [], []
    ell = _node_spacing(body.X)
    for b in range(n_bodies):
        gi = b // (layout[1] * layout[2])
        gj = (b // layout[2]) % layout[1]
        gk = b % layout[2]
        off = pitch * np.array([gi, gj, gk], dtype=np.float64)
        Xb = body.X + off
        rng = np.random.default_rng(seed + 10 + b)
        R = random_rotation(rng)
        eps = rng.uniform(-strain, strain, size=(3, 3))
        Fh = R @ (np.eye(3) + 0.5 * (eps + eps.T))
        xb = (body.X - center) @ Fh.T + center + off
        xb += rng.normal(0.0, 0.01 * ell, size=xb.shape)
        Xs.append(Xb)
        xs.append(xb)
        conns.append(body.conn + b * nb_nodes)
    X = np.concatenate(Xs)
    conn = np.concatenate(conns).astype(np.int32)
    mesh = Mesh(0, X, conn, body_of_elem=np.repeat(np.arange(n_bodies), nb_el),
                name=f"manybody{n_bodies}")
    x = np.concatenate(xs).ravel()
    v = np.random.default_rng(seed + 1).normal(0.0, vel, size=x.shape)
    return mesh, x, v


# -------------------------------------------------------------- materials --

# tlfea_material field order: model, E, nu, C10, C01, kappa, rho0, eta, lambda_d
SVK_PAPER = dict(model=0, E=7.0e8, nu=0.33, C10=0.0, C01=0.0, kappa=0.0, rho0=2700.0,
                 eta_damp=0.0, lambda_damp=0.0)
MR_PAPER = dict(model=1, E=0.0, nu=0.0, C10=7.89e7, C01=5.26e7, kappa=1.03e9, rho0=2700.0,
                eta_damp=0.0, lambda_damp=0.0)
KV_TIRE = dict(eta_damp=5.0e3, lambda_damp=5.0e3)
TIRE_DROP = dict(model=0, E=5.0e6, nu=0.40, C10=0.0, C01=0.0, kappa=0.0, rho0=900.0,
                 eta_damp=0.0, lambda_damp=0.0)

Q_T10_4PT, Q_T10_KEAST5, Q_GL_443, Q_GL_322 = 0, 1, 2, 3
H_T10, H_ANCF = 1.0e-3, 5.0e-4
H_BEAM = 1.0e-3


@dataclasses.dataclass
class Config:
    name: str
    mesh: Mesh
    material: dict
    quadrature: int
    h: float
    force_only: bool = False


def config(idx: int, scale: str = "full") -> Config:
    """The five BASELINE.json configurations."""
    if idx == 1:
        m = kuhn_t10_box(8, 2, 2, 1.0, 0.25, 0.25)
        return Config("cfg1_t10_8x2x2_svk_4pt", m, dict(SVK_PAPER), Q_T10_4PT, H_T10)
    if idx == 2:
        m = kuhn_t10_box(42, 28, 14, 3.0, 2.0, 1.0)
        mat = dict(MR_PAPER)
        mat.update(KV_TIRE)
        return Config("cfg2_t10_42x28x14_mr_kv_keast5", m, mat, Q_T10_KEAST5, H_T10)
    if idx == 3:
        m = kuhn_t10_box(144, 96, 48, 3.0, 2.0, 1.0)
        return Config("cfg3_t10_144x96x48_svk_keast5", m, dict(SVK_PAPER), Q_T10_KEAST5, H_T10)
    if idx == 4:
        m = ancf_plate(200)
        return Config("cfg4_ancf3443_200x200_svk_gl443", m, dict(SVK_PAPER), Q_GL_443, H_ANCF)
    if idx == 5:
        m, _, _ = many_body()
        return Config("cfg5_manybody_2000x_t10_9x6x3_force_only", m, dict(TIRE_DROP),
                      Q_T10_KEAST5, H_T10, force_only=True)
    if idx == 6:
        # NEXT-1 measurement: the paper's largest ANCF3243 beam (RES32)
        m = ancf_beam(500000)
        return Config("cfg6_ancf3243_beam_res32_500k_svk_gl322", m, dict(SVK_PAPER), Q_GL_322, H_BEAM)
    raise ValueError(idx)
