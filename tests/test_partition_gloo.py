"""The N>1 path on CPU: two ranks over the gloo backend exercise the host
partition planner of libtlfea (tlfea_plan_partition, no GPU needed), the
product transport (paper_2604_10357_b200.dist.exchange) and the exchange
protocol (owner adds received partial blocks / forces in ascending peer
order). Partial values come from the oracle restricted to each rank's
elements; the assembled owned rows must equal the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dense_blocks(pr, H):
    """(I,J) -> 3x3 block of an oracle H on its DOF pattern."""
    out = {}
    for I in range(pr.n_coef):
        for k in range(pr.rowptr_c[I], pr.rowptr_c[I + 1]):
            J = int(pr.cols_c[k])
            blk = np.zeros((3, 3))
            for d in range(3):
                r0 = pr.rowptr[3 * I + d]
                deg = pr.rowptr_c[I + 1] - pr.rowptr_c[I]
                kk = k - pr.rowptr_c[I]
                blk[d] = H[r0 + 3 * kk:r0 + 3 * kk + 3]
            out[(I, J)] = blk
    return out


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2604_10357_b200 as T
    import synth
    from paper_2604_10357_b200 import dist as tdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "t10":
            mesh, mat, rule = synth.kuhn_t10_box(4, 2, 2, 0.8, 0.4, 0.4), dict(synth.SVK_PAPER), 1
            x, v, vn, _ = synth.t10_state(mesh)
        else:
            mesh, mat, rule = synth.ancf_plate(4), dict(synth.SVK_PAPER), 2
            x, v, vn = synth.ancf_state(mesh)
        h = 1e-3
        cc = mesh.coef_conn()
        part = tdist.contiguous_partition(mesh.n_el, world)
        plans = [T.tlfea_plan_partition(cc, mesh.n_coef, part, world, r) for r in range(world)]
        owner = plans[rank][0]
        # this rank's partial sums: oracle over its own elements only
        sub = synth.Mesh(mesh.element, mesh.X, mesh.conn[part == rank],
                         None if mesh.dims is None else mesh.dims[part == rank])
        prs = oracle.Problem(sub, dict(mat, rho0=0.0), rule)      # partial h K only
        _, Hs, fs = prs.eval(x, v, vn, None, h)
        blocks = _dense_blocks(prs, Hs)
        # pack per the planner's canonical send lists (peer, then (I,J) ascending)
        _, sb, sbp, sn, snp = plans[rank]
        send, scounts = [], np.zeros(world, np.int64)
        for p in range(world):
            for (I, J), pp in zip(sb, sbp):
                if pp == p:
                    send.append(blocks[(int(I), int(J))].ravel())
                    scounts[p] += 9
            for I, pp in zip(sn, snp):
                if pp == p:
                    send.append(fs[3 * I:3 * I + 3])
                    scounts[p] += 3
        # what each peer sends me = its send list restricted to peer == rank
        rcounts = np.zeros(world, np.int64)
        recv_lists = []
        for p in range(world):
            _, psb, psbp, psn, psnp = plans[p]
            bl = [tuple(map(int, k)) for k, pp in zip(psb, psbp) if pp == rank]
            nl = [int(k) for k, pp in zip(psn, psnp) if pp == rank]
            recv_lists.append((bl, nl))
            rcounts[p] = 9 * len(bl) + 3 * len(nl)
        sbuf = torch.tensor(np.concatenate(send) if send else np.zeros(1))
        rbuf = torch.zeros(max(1, int(rcounts.sum())), dtype=torch.float64)
        tdist.exchange(sbuf, rbuf, scounts, rcounts)
        # owner: own partial + received partials in ascending peer order
        rb = rbuf.numpy()
        roff = tdist.offsets(rcounts)
        pr = oracle.Problem(mesh, mat, rule)
        _, H0, f0 = pr.eval(x, v, vn, None, h)
        full = _dense_blocks(pr, H0)
        err_H = err_f = 0.0
        nrm_H = nrm_f = 0.0
        mine = {k: b.copy() for k, b in blocks.items() if owner[k[0]] == rank}
        fmine = {I: fs[3 * I:3 * I + 3].copy() for I in range(mesh.n_coef) if owner[I] == rank}
        for p in range(world):
            off = roff[p]
            bl, nl = recv_lists[p]
            for k in bl:
                mine[k] = mine.get(k, np.zeros((3, 3))) + rb[off:off + 9].reshape(3, 3)
                off += 9
            for I in nl:
                fmine[I] = fmine[I] + rb[off:off + 3]
                off += 3
        for (I, J), blk in full.items():
            if owner[I] != rank:
                continue
            got = mine.get((I, J), np.zeros((3, 3))) + M_over_h(pr, I, J, h)
            err_H += np.sum((got - blk) ** 2)
            nrm_H += np.sum(blk ** 2)
        for I in range(mesh.n_coef):
            if owner[I] == rank:
                err_f += np.sum((fmine[I] - f0[3 * I:3 * I + 3]) ** 2)
                nrm_f += np.sum(f0[3 * I:3 * I + 3] ** 2)
        q.put((rank, err_H, nrm_H, err_f, nrm_f, int(np.sum(owner == rank))))
    finally:
        dist.destroy_process_group()


def M_over_h(pr, I, J, h):
    k = np.searchsorted(pr.cols_c[pr.rowptr_c[I]:pr.rowptr_c[I + 1]], J)
    return np.eye(3) * pr.M[pr.rowptr_c[I] + k] / h


@pytest.mark.parametrize("case", ["t10", "ancf"])
def test_two_rank_exchange_protocol(case):
    import paper_2604_10357_b200 as T
    from paper_2604_10357_b200 import build
    build.build()
    T.lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    eH = sum(o[1] for o in out)
    nH = sum(o[2] for o in out)
    ef = sum(o[3] for o in out)
    nf = sum(o[4] for o in out)
    assert np.sqrt(eH / nH) <= 1e-12 and np.sqrt(ef / nf) <= 1e-12
    assert sum(o[5] for o in out) > 0 and all(o[5] > 0 for o in out)
