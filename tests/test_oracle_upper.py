"""Pins of the oracle's UPPER view of H (reading Q14):
the kept entries are exactly col >= row, their count is (nnz + n_dof)/2 for
the symmetric pattern, and the view plus its mirror rebuilds the full,
symmetric H. CPU only."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("mk,rule", [(lambda: synth.kuhn_t10_box(2, 2, 1, 0.4, 0.4, 0.2), 1),
                                     (lambda: synth.ancf_plate(3), 2),
                                     (lambda: synth.ancf_beam(5), 3)], ids=["t10", "ancf", "beam"])
def test_upper_view_rebuilds_full_h(mk, rule):
    mesh = mk()
    pr = oracle.Problem(mesh, dict(synth.SVK_PAPER), rule)
    if mesh.element == 0:
        x, v, vn, _ = synth.t10_state(mesh)
    else:
        x, v, vn = synth.ancf_state(mesh)
    _, H, _ = pr.eval(x, v, vn, None, 1e-3)
    rowptr_u, cols_u, idx = pr.upper_view()
    n = mesh.n_dof
    assert cols_u.size == (pr.nnz + n) // 2
    for i in range(n):
        c = cols_u[rowptr_u[i]:rowptr_u[i + 1]]
        assert c.size > 0 and c[0] == i and np.all(np.diff(c) > 0)
    full = np.zeros((n, n))
    for i in range(n):
        full[i, pr.cols[pr.rowptr[i]:pr.rowptr[i + 1]]] = H[pr.rowptr[i]:pr.rowptr[i + 1]]
    up = np.zeros((n, n))
    Hu = H[idx]
    for i in range(n):
        up[i, cols_u[rowptr_u[i]:rowptr_u[i + 1]]] = Hu[rowptr_u[i]:rowptr_u[i + 1]]
    rebuilt = up + np.triu(up, 1).T
    assert np.abs(rebuilt - full).max() <= 1e-12 * np.abs(full).max()
