"""GPU (libtlfea, sm_100a) vs CPU oracle parity, element by element, through
the C ABI. Bar (BASELINE.json north_star): CSR pattern and slot map bit-exact;
force, residual and Hessian values within 1e-11 normwise relative error;
bitwise run-to-run determinism."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-11


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_10357_b200 as T
    T.lib()
    return torch


def dev(torch, a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def gpu_eval(torch, mesh, mat, rule, x, v, vn=None, fext=None, h=1e-3, mass_rule=0, gravity=(0, 0, 0)):
    import paper_2604_10357_b200 as T
    ctx = T.Context.from_mesh(mesh, mat, rule, mass_rule=mass_rule, gravity=gravity)
    g, H, f = ctx.empty_outputs()
    ctx.eval(dev(torch, x), dev(torch, v), dev(torch, vn), dev(torch, fext), h, g, H, f)
    torch.cuda.synchronize()
    return ctx, g.cpu().numpy(), H.cpu().numpy(), f.cpu().numpy()


def check_pattern(ctx, pr):
    rowptr, cols, rowptr_c, cols_c, owned = [t.cpu().numpy() for t in ctx.export_pattern()]
    assert np.array_equal(rowptr.astype(np.int64), pr.rowptr)
    assert np.array_equal(cols.astype(np.int64), pr.cols)
    assert np.array_equal(rowptr_c.astype(np.int64), pr.rowptr_c)
    assert np.array_equal(cols_c.astype(np.int64), pr.cols_c)
    assert np.array_equal(owned, np.arange(pr.n_coef))


CASES = {
    "cfg1_svk_4pt": lambda: (synth.config(1).mesh, dict(synth.SVK_PAPER), 0),
    "t10_5x3x1_svk_keast5_ragged": lambda: (synth.kuhn_t10_box(5, 3, 1, 1.0, 0.6, 0.2), dict(synth.SVK_PAPER), 1),
    # 2,940 elements: the one-launch small-mesh path with warps taking several unit groups
    "t10_10x7x7_svk_keast5_small_fused": lambda: (synth.kuhn_t10_box(10, 7, 7, 1.0, 0.7, 0.7), dict(synth.SVK_PAPER), 1),
    "t10_4x3x2_mr_kv_keast5": lambda: (synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4),
                                       dict(synth.MR_PAPER, **synth.KV_TIRE), 1),
    "t10_3x2x2_svk_kv_4pt_morton": lambda: (synth.kuhn_t10_box(3, 2, 2, 0.3, 0.2, 0.2, order="morton"),
                                            dict(synth.SVK_PAPER, **synth.KV_TIRE), 0),
    "t10_single_element": lambda: (synth.Mesh(0, synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X,
                                              synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).conn[:1]), dict(synth.MR_PAPER), 1),
    # class-mode SVK (two-phase element group): a lone element and a tail that
    # ends inside a warp group (100 = 3 * 33 + 1) and inside a CTA tile
    "t10_single_element_svk": lambda: (synth.Mesh(0, synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).X,
                                                  synth.kuhn_t10_box(1, 1, 1, 1, 1, 1).conn[:1]),
                                       dict(synth.SVK_PAPER), 1),
    "t10_100el_svk_keast5_ragged": lambda: (synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                       synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100]),
                                            dict(synth.SVK_PAPER), 1),
    # two-phase SVK + KV and MR (+ KV) groups on a tail inside a warp group,
    # with classes and (perturbed) with staged per-element tables
    "t10_100el_svk_kv_keast5": lambda: (synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                   synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100]),
                                        dict(synth.SVK_PAPER, **synth.KV_TIRE), 1),
    "t10_100el_mr_kv_keast5": lambda: (synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                  synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100]),
                                       dict(synth.MR_PAPER, **synth.KV_TIRE), 1),
    "t10_100el_perturbed_mr_kv_4pt": lambda: (synth.perturbed(synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                                         synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100])),
                                              dict(synth.MR_PAPER, **synth.KV_TIRE), 0),
    "t10_100el_perturbed_svk_keast5": lambda: (synth.perturbed(synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                                          synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100])),
                                               dict(synth.SVK_PAPER), 1),
    "t10_4x3x2_perturbed_svk_kv_keast5": lambda: (synth.perturbed(synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4)),
                                                  dict(synth.SVK_PAPER, **synth.KV_TIRE), 1),
    "t10_3x3x2_perturbed_mr_4pt": lambda: (synth.perturbed(synth.kuhn_t10_box(3, 3, 2, 0.6, 0.6, 0.4)),
                                           dict(synth.MR_PAPER), 0),
    # straight-sided, non-congruent T10: the affine (min) layout, 13 fp64 per element
    "t10_5x3x2_straight_svk_keast5": lambda: (synth.perturbed_straight(synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4)),
                                              dict(synth.SVK_PAPER), 1),
    "t10_4x3x2_straight_svk_4pt": lambda: (synth.perturbed_straight(synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4)),
                                           dict(synth.SVK_PAPER), 0),
    "t10_4x3x2_straight_mr_kv_keast5": lambda: (synth.perturbed_straight(synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4)),
                                                dict(synth.MR_PAPER, **synth.KV_TIRE), 1),
    "t10_100el_straight_svk_keast5": lambda: (synth.perturbed_straight(synth.Mesh(0, synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).X,
                                                                                  synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4).conn[:100])),
                                              dict(synth.SVK_PAPER), 1),
    "ancf_3x3_svk": lambda: (synth.ancf_plate(3), dict(synth.SVK_PAPER), 2),
    "ancf_5x5_mr_kv": lambda: (synth.ancf_plate(5), dict(synth.MR_PAPER, **synth.KV_TIRE), 2),
    # ANCF3443 on the per-(e,q) table path (more than 4 element shapes: the
    # lane-per-node group without classes) and the SVK + KV tangent group
    "ancf_6x6_graded_svk": lambda: (synth.ancf_plate_graded(6), dict(synth.SVK_PAPER), 2),
    "ancf_4x4_perturbed_svk": lambda: (synth.perturbed(synth.ancf_plate(4), amp=0.02), dict(synth.SVK_PAPER), 2),
    "ancf_5x5_graded_svk_kv": lambda: (synth.ancf_plate_graded(5), dict(synth.SVK_PAPER, **synth.KV_TIRE), 2),
    "ancf_4x4_svk_kv": lambda: (synth.ancf_plate(4), dict(synth.SVK_PAPER, **synth.KV_TIRE), 2),
    # ANCF3243 beam (NEXT-1): 16 elements = one CTA tile; 9 = ragged tile
    "beam_16_svk": lambda: (synth.ancf_beam(16), dict(synth.SVK_PAPER), 3),
    "beam_9_mr_kv": lambda: (synth.ancf_beam(9), dict(synth.MR_PAPER, **synth.KV_TIRE), 3),
    "beam_5_perturbed_svk_kv": lambda: (synth.perturbed(synth.ancf_beam(5), amp=0.02),
                                        dict(synth.SVK_PAPER, **synth.KV_TIRE), 3),
}


def state(mesh, seed=synth.SEED_BASE):
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, seed=seed, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh, seed=seed)
        fext = np.random.default_rng(seed + 3).normal(size=x.shape)
    return x, v, vn, fext


@pytest.mark.parametrize("case", list(CASES))
def test_eval_parity(torch_cuda, case):
    mesh, mat, rule = CASES[case]()
    h = synth.H_T10 if mesh.element == 0 else synth.H_ANCF
    grav = (0.0, -9.81, 0.3)
    x, v, vn, fext = state(mesh)
    pr = oracle.Problem(mesh, mat, rule, gravity=grav)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    ctx, g, H, f = gpu_eval(torch_cuda, mesh, mat, rule, x, v, vn, fext, h, gravity=grav)
    check_pattern(ctx, pr)
    # congruent (Kuhn / uniform plate) meshes use shared-memory geometry classes,
    # perturbed meshes the per-(e,q) tables
    if "straight" in case:
        assert ctx.info["n_geometry_classes"] == 0 and ctx.info["reference_layout"] == 2
    elif "perturbed" in case or "graded" in case:
        assert ctx.info["n_geometry_classes"] == 0
        if mesh.element == 0:   # curved T10: the per-(e,q) J^-1 layout
            assert ctx.info["reference_layout"] == 3
    elif mesh.element == 0 and mesh.n_el >= 6:
        assert ctx.info["n_geometry_classes"] == 6
    else:
        assert ctx.info["n_geometry_classes"] >= 1
    assert rel(f, f0) <= TOL, rel(f, f0)
    assert rel(g, g0) <= TOL, rel(g, g0)
    assert rel(H, H0) <= TOL, rel(H, H0)
    # slot map bit-exact (reading Q16)
    assert np.array_equal(ctx.slot_map().astype(np.int64), pr.slot_map())
    # determinism: a second evaluation is bitwise identical
    _, g2, H2, f2 = gpu_eval(torch_cuda, mesh, mat, rule, x, v, vn, fext, h, gravity=grav)
    assert np.array_equal(g, g2) and np.array_equal(H, H2) and np.array_equal(f, f2)


@pytest.mark.parametrize("case", ["cfg1_svk_4pt", "t10_4x3x2_mr_kv_keast5", "ancf_5x5_mr_kv", "beam_9_mr_kv"])
def test_setup_exports(torch_cuda, case):
    mesh, mat, rule = CASES[case]()
    import paper_2604_10357_b200 as T
    grav = (0.1, 0.0, -9.81)
    ctx = T.Context.from_mesh(mesh, mat, rule, gravity=grav)
    pr = oracle.Problem(mesh, mat, rule, gravity=grav)
    gN, Jw = ctx.export_precompute()
    assert rel(gN.cpu().numpy(), pr.gradN) <= 1e-13
    assert rel(Jw.cpu().numpy(), pr.J0w) <= 1e-13
    M, fff = ctx.export_mass()
    assert rel(M.cpu().numpy(), pr.M) <= 1e-13
    assert rel(fff.cpu().numpy(), pr.fff) <= 1e-13


@pytest.mark.parametrize("case", ["cfg1_svk_4pt", "t10_4x3x2_mr_kv_keast5", "ancf_3x3_svk", "beam_16_svk",
                                  "t10_100el_perturbed_svk_keast5"])
def test_force_only_and_split_stages(torch_cuda, case):
    torch = torch_cuda
    mesh, mat, rule = CASES[case]()
    import paper_2604_10357_b200 as T
    x, v, vn, _ = state(mesh)
    pr = oracle.Problem(mesh, mat, rule)
    _, _, f0 = pr.eval(x, v, vn, None, 1e-3, hessian=False)
    ctx = T.Context.from_mesh(mesh, mat, rule)
    xd, vd = dev(torch, x), dev(torch, v)
    f = ctx.force_only(xd, vd)
    torch.cuda.synchronize()
    assert rel(f.cpu().numpy(), f0) <= TOL
    # Stage 1 alone (compute_p) and Stage 2 alone (compute_internal_force)
    P = ctx.compute_stress(xd, vd)
    P0 = pr.stress(x, v)
    assert rel(P.cpu().numpy(), P0) <= TOL
    f2 = ctx.internal_force_from_stress(P)
    assert rel(f2.cpu().numpy(), f0) <= TOL
    # residual alone from the oracle's f_int
    g = ctx.compute_gradient(dev(torch, f0), vd, dev(torch, vn), None, 1e-3)
    g0, _, _ = pr.eval(x, v, vn, None, 1e-3, hessian=False)
    assert rel(g.cpu().numpy(), g0) <= TOL
    # Hessian alone
    H = ctx.assemble_hessian(xd, 1e-3)
    _, H0, _ = pr.eval(x, v, vn, None, 1e-3)
    assert rel(H.cpu().numpy(), H0) <= TOL


@pytest.mark.parametrize("model", [0, 1])
def test_constitutive_hook(torch_cuda, model):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mat = dict(synth.SVK_PAPER if model == 0 else synth.MR_PAPER, **synth.KV_TIRE)
    rng = np.random.default_rng(31)
    n = 64
    F = np.eye(3)[None] + rng.uniform(-0.2, 0.2, (n, 3, 3))
    Fd = rng.normal(size=(n, 3, 3))
    P, A = T.tlfea_test_constitutive(mat, dev(torch, F.reshape(n, 9)), dev(torch, Fd.reshape(n, 9)))
    P, A = P.cpu().numpy(), A.cpu().numpy()
    for i in range(n):
        assert rel(P[i], oracle.pk1(model, mat, F[i], Fd[i]).ravel()) <= 1e-13
        assert rel(A[i], oracle.tangent(model, mat, F[i]).ravel()) <= 1e-12


@pytest.mark.parametrize("case", ["ancf_6x6_graded_svk", "ancf_4x4_perturbed_svk", "ancf_5x5_graded_svk_kv",
                                  "ancf_4x4_svk_kv", "ancf_3x3_svk", "t10_100el_perturbed_svk_keast5",
                                  "t10_5x3x2_straight_svk_keast5", "t10_4x3x2_straight_svk_4pt",
                                  "t10_5x3x1_svk_keast5_ragged", "cfg1_svk_4pt",
                                  "ancf_5x5_mr_kv", "ancf_6x6_graded_svk", "ancf_4x4_perturbed_svk",
                                  "ancf_5x5_graded_svk_kv", "beam_16_svk", "beam_9_mr_kv",
                                  "beam_5_perturbed_svk_kv", "t10_4x3x2_mr_kv_keast5", "t10_100el_perturbed_mr_kv_4pt",
                                  "t10_100el_svk_kv_keast5", "t10_4x3x2_perturbed_svk_kv_keast5",
                                  "t10_100el_mr_kv_keast5"])
def test_force_only_parity(torch_cuda, case):
    """tlfea_force_only (the AdamW inner evaluation) on the class and the
    per-(e,q) table paths, with and without Kelvin-Voigt."""
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule = CASES[case]()
    x, v, vn, fext = state(mesh)
    pr = oracle.Problem(mesh, mat, rule)
    _, _, f0 = pr.eval(x, v, vn, None, 1e-3, hessian=False)
    ctx = T.Context.from_mesh(mesh, mat, rule)
    f = ctx.force_only(dev(torch, x), dev(torch, v)).cpu().numpy()
    assert rel(f, f0) <= TOL, rel(f, f0)


def test_many_body_force_only(torch_cuda):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, x, v = synth.many_body(n_bodies=7, cells=(3, 2, 1), size=(0.3, 0.2, 0.1))
    mat = dict(synth.TIRE_DROP)
    pr = oracle.Problem(mesh, mat, 1)
    _, _, f0 = pr.eval(x, v, v, None, 1e-3, hessian=False)
    ctx = T.Context.from_mesh(mesh, mat, 1)
    f = ctx.force_only(dev(torch, x), dev(torch, v)).cpu().numpy()
    assert rel(f, f0) <= TOL


@pytest.mark.parametrize("rule", [0, 1])
def test_many_body_force_only_persistent(torch_cuda, rule):
    """Class-mode force-only kernel with persistent warps (several grid-stride
    sweeps: 58k elements > one resident wave) under both rules, and from a
    non-tile-aligned element offset (begin/interior/finish of a 2-part
    virtual partition would start mid-tile)."""
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, x, v = synth.many_body(n_bodies=60)
    mat = dict(synth.TIRE_DROP)
    pr = oracle.Problem(mesh, mat, rule)
    _, _, f0 = pr.eval(x, v, v, None, 1e-3, hessian=False)
    ctx = T.Context.from_mesh(mesh, mat, rule)
    assert ctx.info["n_geometry_classes"] > 0
    f = ctx.force_only(dev(torch, x), dev(torch, v)).cpu().numpy()
    assert rel(f, f0) <= TOL, rel(f, f0)


def test_eval_host_matches_device(torch_cuda):
    torch = torch_cuda
    import paper_2604_10357_b200 as T
    mesh, mat, rule = CASES["cfg1_svk_4pt"]()
    x, v, vn, fext = state(mesh)
    ctx, g, H, f = gpu_eval(torch, mesh, mat, rule, x, v, vn, fext, 1e-3)
    gh = np.zeros_like(g)
    Hh = np.zeros_like(H)
    fh = np.zeros_like(f)
    ctx.eval_host(x, v, vn, fext, 1e-3, gh, Hh, fh)
    assert np.array_equal(g, gh) and np.array_equal(H, Hh) and np.array_equal(f, fh)


def test_errors(torch_cuda):
    import paper_2604_10357_b200 as T
    mesh = synth.kuhn_t10_box(1, 1, 1, 1, 1, 1)
    c = mesh.conn.copy()
    c[3, [1, 2]] = c[3, [2, 1]]
    c[3, [4, 5, 6, 7, 8, 9]] = c[3, [6, 5, 4, 7, 9, 8]]
    with pytest.raises(T.TlfeaError, match="inverted element 3"):
        T.Context(0, c, mesh.X, synth.SVK_PAPER, 1)
    with pytest.raises(T.TlfeaError, match="INVALID"):
        T.Context(0, mesh.conn, mesh.X, dict(synth.SVK_PAPER, nu=0.5), 1)
    bad = mesh.conn.copy()
    bad[0, 1] = bad[0, 0]
    with pytest.raises(T.TlfeaError, match="repeats node"):
        T.Context(0, bad, mesh.X, synth.SVK_PAPER, 1)
    # Mooney-Rivlin inverted state is flagged with (element, qp)
    torch = torch_cuda
    ctx = T.Context(0, mesh.conn, mesh.X, synth.MR_PAPER, 1)
    x = mesh.X.copy()
    x[mesh.conn[2, 3]] = x[mesh.conn[2, 0]] - 0.5 * (x[mesh.conn[2, 3]] - x[mesh.conn[2, 0]])
    ctx.eval(dev(torch, x.ravel()), dev(torch, np.zeros(mesh.n_dof)), h=1e-3)
    bad = ctx.sync_status()
    assert bad is not None and bad[0] in set(np.nonzero((mesh.conn == mesh.conn[2, 3]).any(1))[0])
    with pytest.raises(T.TlfeaError, match="INVALID"):
        ctx.eval(dev(torch, mesh.X.ravel()), dev(torch, np.zeros(mesh.n_dof)), h=0.0)


@pytest.mark.parametrize("case", ["t10_5x3x1_svk_keast5_ragged", "cfg1_svk_4pt", "t10_4x3x2_mr_kv_keast5"])
def test_affine_layout_on_kuhn_boxes(torch_cuda, case):
    """options.reference_layout = 2 forces the affine (min) layout on a
    congruent Kuhn box: same results as the class tables (to rounding) and as
    the oracle."""
    import paper_2604_10357_b200 as T
    torch = torch_cuda
    mesh, mat, rule = CASES[case]()
    h = synth.H_T10
    x, v, vn, fext = state(mesh)
    ca = T.Context.from_mesh(mesh, mat, rule, reference_layout="affine")
    assert ca.info["reference_layout"] == 2
    g, H, f = ca.eval(dev(torch, x), dev(torch, v), dev(torch, vn), dev(torch, fext), h, f_int=ca.empty_outputs()[2])
    fo = ca.force_only(dev(torch, x), dev(torch, v)).cpu().numpy()
    torch.cuda.synchronize()
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    assert rel(g.cpu().numpy(), g0) <= TOL and rel(H.cpu().numpy(), H0) <= TOL and rel(f.cpu().numpy(), f0) <= TOL
    if not mat.get("eta_damp"):
        assert rel(fo, f0) <= TOL


@pytest.mark.parametrize("case", ["t10_100el_perturbed_svk_keast5", "t10_4x3x2_perturbed_svk_kv_keast5",
                                  "t10_3x3x2_perturbed_mr_4pt", "t10_100el_perturbed_mr_kv_4pt"])
def test_jinv_layout_vs_tables(torch_cuda, case):
    """Curved T10 (every node displaced): the per-(e,q) J^-1 layout (10 fp64 per
    point, grad N rebuilt from the T10 basis) against the paper's per-(e,q)
    tables forced by options.reference_layout = 1 (to rounding, 1e-12) and the oracle,
    for force + H + g and force only."""
    import paper_2604_10357_b200 as T
    torch = torch_cuda
    mesh, mat, rule = CASES[case]()
    h = synth.H_T10
    x, v, vn, fext = state(mesh)
    cj = T.Context.from_mesh(mesh, mat, rule)
    ct = T.Context.from_mesh(mesh, mat, rule, reference_layout="tables")
    assert cj.info["reference_layout"] == 3 and ct.info["reference_layout"] == 1
    outs = []
    for c in (cj, ct):
        g, H, f = c.eval(dev(torch, x), dev(torch, v), dev(torch, vn), dev(torch, fext), h, f_int=c.empty_outputs()[2])
        fo = c.force_only(dev(torch, x), dev(torch, v))
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (g, H, f, fo)])
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    for a, b in zip(outs[0], outs[1]):   # g carries cancellation (f - f_ext - f_ff + M dv/h)
        assert rel(a, b) <= 1e-12
    for a, b in zip(outs[0][:3], (g0, H0, f0)):
        assert rel(a, b) <= TOL
    assert rel(outs[0][3], f0) <= TOL


@pytest.mark.parametrize("case", ["cfg1_svk_4pt", "t10_5x3x1_svk_keast5_ragged", "t10_single_element_svk",
                                  "t10_100el_svk_keast5_ragged", "t10_5x3x2_straight_svk_keast5"])
def test_eval_parity_without_fint(torch_cuda, case):
    """tlfea_eval with f_int_out = NULL (the north star's outputs g and H
    only): g and H against the oracle at the same bar, bitwise repeatable, H
    bitwise equal to the f_int path's, and v_n = NULL."""
    import paper_2604_10357_b200 as T
    torch = torch_cuda
    mesh, mat, rule = CASES[case]()
    h = synth.H_T10
    grav = (0.0, -9.81, 0.3)
    x, v, vn, fext = state(mesh)
    pr = oracle.Problem(mesh, mat, rule, gravity=grav)
    g0, H0, _ = pr.eval(x, v, vn, fext, h)
    ctx = T.Context.from_mesh(mesh, mat, rule, gravity=grav)
    outs = []
    for _ in range(2):
        g, H, _ = ctx.eval(dev(torch, x), dev(torch, v), dev(torch, vn), dev(torch, fext), h)
        torch.cuda.synchronize()
        outs.append((g.cpu().numpy(), H.cpu().numpy()))
    (g, H), (g2, H2) = outs
    assert rel(g, g0) <= TOL, rel(g, g0)
    assert rel(H, H0) <= TOL, rel(H, H0)
    assert np.array_equal(g, g2) and np.array_equal(H, H2)
    _, gf, Hf, _ = gpu_eval(torch, mesh, mat, rule, x, v, vn, fext, h, gravity=grav)
    assert np.array_equal(H, Hf)
    # v_n = NULL (= 0) on the same path
    g0n, _, _ = pr.eval(x, v, None, fext, h)
    gn, _, _ = ctx.eval(dev(torch, x), dev(torch, v), None, dev(torch, fext), h)
    torch.cuda.synchronize()
    assert rel(gn.cpu().numpy(), g0n) <= TOL
