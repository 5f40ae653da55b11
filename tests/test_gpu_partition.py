"""Element-partitioned evaluation on ONE GPU:
P contexts (rank 0..P-1 of a P-way partition) live in one process and their
send/recv buffers are exchanged by device copies ("virtual partition"). The
union of the owned rows must reproduce the single-GPU pattern bit-exactly and
the oracle's values within 1e-11; results are deterministic run to run. The
NCCL transport of the same buffers is bench.py's `--gpus N` path."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-11


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def run_partitioned(torch, mesh, mat, rule, P, x, v, vn, fext, h, part=None, force_only=False):
    import paper_2604_10357_b200 as T
    d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    xd, vd, vnd, fed = d(x), d(v), d(vn), d(fext)
    ctxs = [T.Context.from_mesh(mesh, mat, rule, rank=r, nranks=P, elem_part=part) for r in range(P)]
    sizes = [c.exchange_sizes() for c in ctxs]
    sbufs = [torch.zeros(max(1, int(s.sum())), dtype=torch.float64, device="cuda") for s, _ in sizes]
    rbufs = [torch.zeros(max(1, int(r.sum())), dtype=torch.float64, device="cuda") for _, r in sizes]
    outs = []
    for c in ctxs:
        g, H, f = c.empty_outputs()
        outs.append((g, None if force_only else H, f))
    for r, c in enumerate(ctxs):
        c.eval_begin(xd, vd, h, outs[r][1], sbufs[r], force_only=force_only)
        c.eval_interior(xd, vd, h, outs[r][1], force_only=force_only)
    # the exchange: rank r's block for peer p -> rank p's block from r
    for r in range(P):
        soff = np.concatenate([[0], np.cumsum(sizes[r][0])])
        for p in range(P):
            n = int(sizes[r][0][p])
            if n == 0:
                continue
            roff = np.concatenate([[0], np.cumsum(sizes[p][1])])
            assert int(sizes[p][1][r]) == n
            rbufs[p][roff[r]:roff[r] + n].copy_(sbufs[r][soff[p]:soff[p] + n])
    for r, c in enumerate(ctxs):
        g, H, f = outs[r]
        c.eval_finish(rbufs[r], vd, vnd, fed, h, None if force_only else g, H, f, force_only=force_only)
    torch.cuda.synchronize()
    res = []
    for c, (g, H, f) in zip(ctxs, outs):
        rowptr, cols, _, _, owned = [t.cpu().numpy().astype(np.int64) for t in c.export_pattern()]
        res.append(dict(owned=owned, rowptr=rowptr, cols=cols, g=g.cpu().numpy(),
                        H=None if H is None else H.cpu().numpy(), f=f.cpu().numpy()))
    return res


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("case", ["t10_svk", "t10_mr_kv", "ancf"])
def test_virtual_partition_matches_oracle(torch_cuda, P, case):
    if case == "t10_svk":
        mesh, mat, rule = synth.kuhn_t10_box(6, 3, 2, 1.2, 0.6, 0.4), dict(synth.SVK_PAPER), 1
    elif case == "t10_mr_kv":
        mesh, mat, rule = synth.kuhn_t10_box(5, 3, 2, 1.0, 0.6, 0.4), dict(synth.MR_PAPER, **synth.KV_TIRE), 0
    else:
        mesh, mat, rule = synth.ancf_plate(6), dict(synth.SVK_PAPER), 2
    h = 1e-3
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = np.random.default_rng(3).normal(size=x.shape)
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    res = run_partitioned(torch_cuda, mesh, mat, rule, P, x, v, vn, fext, h)
    owned_all = np.concatenate([r["owned"] for r in res])
    assert np.array_equal(np.sort(owned_all), np.arange(mesh.n_coef))      # a partition of the rows
    g = np.zeros_like(g0)
    f = np.zeros_like(f0)
    H = np.zeros_like(H0)
    for r in res:
        for i, I in enumerate(r["owned"]):
            g[3 * I:3 * I + 3] = r["g"][3 * i:3 * i + 3]
            f[3 * I:3 * I + 3] = r["f"][3 * i:3 * i + 3]
            for dd in range(3):
                a0, a1 = r["rowptr"][3 * i + dd], r["rowptr"][3 * i + dd + 1]
                b0, b1 = pr.rowptr[3 * I + dd], pr.rowptr[3 * I + dd + 1]
                assert np.array_equal(r["cols"][a0:a1], pr.cols[b0:b1])      # global columns, bit-exact
                H[b0:b1] = r["H"][a0:a1]
    assert rel(f, f0) <= TOL and rel(g, g0) <= TOL and rel(H, H0) <= TOL
    # deterministic for a fixed partition
    res2 = run_partitioned(torch_cuda, mesh, mat, rule, P, x, v, vn, fext, h)
    for a, b in zip(res, res2):
        assert np.array_equal(a["H"], b["H"]) and np.array_equal(a["g"], b["g"])


def test_virtual_partition_force_only_custom_part(torch_cuda):
    mesh, x, v = synth.many_body(n_bodies=6, cells=(2, 2, 1), size=(0.2, 0.2, 0.1))
    mat = dict(synth.TIRE_DROP)
    part = (np.arange(mesh.n_el) % 4).astype(np.int32)        # scattered (worst-case) partition
    pr = oracle.Problem(mesh, mat, 1)
    _, _, f0 = pr.eval(x, v, v, None, 1e-3, hessian=False)
    res = run_partitioned(torch_cuda, mesh, mat, 1, 4, x, v, v, None, 1e-3, part=part, force_only=True)
    f = np.zeros_like(f0)
    for r in res:
        for i, I in enumerate(r["owned"]):
            f[3 * I:3 * I + 3] = r["f"][3 * i:3 * i + 3]
    assert rel(f, f0) <= TOL


@pytest.mark.parametrize("case", ["t10_svk", "t10_mr_kv", "beam"])
def test_virtual_partition_scattered_tangent(torch_cuda, case):
    """A scattered element partition (element e on rank e % 3): many element
    blocks have neither row owned by their rank, so they live only in the
    extra scratch positions and reach their owners through the pack lists."""
    if case == "t10_svk":
        mesh, mat, rule = synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4), dict(synth.SVK_PAPER), 1
    elif case == "t10_mr_kv":
        mesh, mat, rule = synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4), dict(synth.MR_PAPER, **synth.KV_TIRE), 1
    else:
        mesh, mat, rule = synth.ancf_beam(24), dict(synth.SVK_PAPER), 3
    P = 3
    part = (np.arange(mesh.n_el) % P).astype(np.int32)
    h = 1e-3
    if mesh.element == 0:
        x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    else:
        x, v, vn = synth.ancf_state(mesh)
        fext = np.random.default_rng(3).normal(size=x.shape)
    pr = oracle.Problem(mesh, mat, rule)
    g0, H0, f0 = pr.eval(x, v, vn, fext, h)
    res = run_partitioned(torch_cuda, mesh, mat, rule, P, x, v, vn, fext, h, part=part)
    g = np.zeros_like(g0)
    H = np.zeros_like(H0)
    for r in res:
        for i, I in enumerate(r["owned"]):
            g[3 * I:3 * I + 3] = r["g"][3 * i:3 * i + 3]
            for dd in range(3):
                a0, a1 = r["rowptr"][3 * i + dd], r["rowptr"][3 * i + dd + 1]
                b0, b1 = pr.rowptr[3 * I + dd], pr.rowptr[3 * I + dd + 1]
                assert np.array_equal(r["cols"][a0:a1], pr.cols[b0:b1])
                H[b0:b1] = r["H"][a0:a1]
    assert rel(g, g0) <= TOL and rel(H, H0) <= TOL


@pytest.mark.parametrize("scattered", [False, True])
def test_partitioned_slot_map_vs_global(torch_cuda, scattered):
    """Reading Q16 on partitioned contexts: a rank's slot map (its local
    elements, ascending global id) holds indices into ITS owned-row CSR (the H
    it writes) and -1 for rows another rank owns. Mapped through the owned
    rows' global CSR offsets, every entry equals the oracle's global slot map."""
    import paper_2604_10357_b200 as T
    mesh, mat, rule = synth.kuhn_t10_box(4, 3, 2, 0.8, 0.6, 0.4), dict(synth.SVK_PAPER), 1
    P = 3
    part = ((np.arange(mesh.n_el) % P) if scattered else (np.arange(mesh.n_el) * P // mesh.n_el)).astype(np.int32)
    pr = oracle.Problem(mesh, mat, rule)
    sm0 = pr.slot_map()
    cc = mesh.coef_conn().astype(np.int64)
    covered = np.zeros(sm0.shape, bool)
    for r in range(P):
        ctx = T.Context.from_mesh(mesh, mat, rule, rank=r, nranks=P, elem_part=part)
        rowptr, _, _, _, owned = [t.cpu().numpy().astype(np.int64) for t in ctx.export_pattern()]
        local = ctx.local_elements()   # boundary elements first (tlfea_local_elements)
        assert np.array_equal(np.sort(local), np.nonzero(part == r)[0])
        sm = ctx.slot_map().astype(np.int64)
        assert sm.shape[0] == local.size
        loc_row = -np.ones(mesh.n_coef, np.int64)
        loc_row[owned] = np.arange(owned.size)
        for k, e in enumerate(local):
            for a in range(10):
                i = loc_row[cc[e, a]]
                for d in range(3):
                    row = sm[k, 3 * a + d]
                    if i < 0:
                        assert np.all(row == -1)
                        continue
                    glob = pr.rowptr[3 * cc[e, a] + d] + (row - rowptr[3 * i + d])
                    assert np.array_equal(glob, sm0[e, 3 * a + d])
                    covered[e, 3 * a + d] = True
    assert covered.mean() > 0.3   # rows its own rank owns: all on a contiguous partition, fewer when scattered
