"""Partitioned evaluation across real processes (launched by
torch.distributed.run; tests/test_gpu_multirank.py): every rank builds its
partitioned context on GPU 0 (the ranks share it), runs
eval_begin -> dist.exchange_start -> eval_interior -> exchange_wait ->
eval_finish with the gloo transport (host-staged: NCCL refuses two ranks on one
device), and rank 0 checks the gathered owned rows against the oracle
(pattern bit-exact, values <= 1e-11). Prints one JSON line on rank 0.
--transport lib: the library's own NCCL transport instead (tlfea_nccl_attach +
tlfea_eval_exchange; rank r on GPU r, so it needs as many GPUs as ranks)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle  # noqa: E402
import paper_2604_10357_b200 as T  # noqa: E402
import synth  # noqa: E402
from paper_2604_10357_b200 import dist as tdist  # noqa: E402


def main():
    lib_transport = "--transport" in sys.argv and sys.argv[sys.argv.index("--transport") + 1] == "lib"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = rank if lib_transport else 0
    torch.cuda.set_device(dev)
    mesh, mat, rule, h = synth.kuhn_t10_box(6, 3, 2, 1.2, 0.6, 0.4), dict(synth.SVK_PAPER), 1, 1e-3
    x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    ctx = T.Context.from_mesh(mesh, mat, rule, rank=rank, nranks=world, device=dev)
    if lib_transport:
        uid = [T.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.nccl_attach(uid[0])
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    xd, vd, vnd, fed = d(x), d(v), d(vn), d(fext)
    sc, rc = ctx.exchange_sizes()
    sbuf = torch.zeros(max(1, int(sc.sum())), dtype=torch.float64, device="cuda")
    rbuf = torch.zeros(max(1, int(rc.sum())), dtype=torch.float64, device="cuda")
    g, H, f = ctx.empty_outputs()
    ctx.eval_begin(xd, vd, h, H, sbuf)
    if lib_transport:
        ctx.eval_exchange(sbuf, rbuf)   # NCCL on the context's stream; finish waits for it
        ctx.eval_interior(xd, vd, h, H)
    else:
        works = tdist.exchange_start(sbuf, rbuf, sc, rc, host_staging=True)
        ctx.eval_interior(xd, vd, h, H)
        tdist.exchange_wait(works)
    ctx.eval_finish(rbuf, vd, vnd, fed, h, g, H, f)
    torch.cuda.synchronize()
    rowptr, cols, _, _, owned = [t.cpu().numpy().astype(np.int64) for t in ctx.export_pattern()]
    mine = dict(owned=owned, rowptr=rowptr, cols=cols, g=g.cpu().numpy(), H=H.cpu().numpy(), f=f.cpu().numpy())
    allr = [None] * world if rank == 0 else None
    dist.gather_object(mine, allr, dst=0)
    if rank == 0:
        pr = oracle.Problem(mesh, mat, rule)
        g0, H0, f0 = pr.eval(x, v, vn, fext, h)
        G, Hh, F = np.zeros_like(g0), np.zeros_like(H0), np.zeros_like(f0)
        pattern_ok = True
        for r in allr:
            for i, I in enumerate(r["owned"]):
                G[3 * I:3 * I + 3] = r["g"][3 * i:3 * i + 3]
                F[3 * I:3 * I + 3] = r["f"][3 * i:3 * i + 3]
                for dd in range(3):
                    a0, a1 = r["rowptr"][3 * i + dd], r["rowptr"][3 * i + dd + 1]
                    b0, b1 = pr.rowptr[3 * I + dd], pr.rowptr[3 * I + dd + 1]
                    pattern_ok &= bool(np.array_equal(r["cols"][a0:a1], pr.cols[b0:b1]))
                    Hh[b0:b1] = r["H"][a0:a1]
        rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
        owned_all = np.sort(np.concatenate([r["owned"] for r in allr]))
        print(json.dumps({"world": world, "transport": "lib" if lib_transport else "gloo", "pattern_ok": pattern_ok,
                          "rows_partition": bool(np.array_equal(owned_all, np.arange(mesh.n_coef))),
                          "rel_g": rel(G, g0), "rel_H": rel(Hh, H0), "rel_f": rel(F, f0)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
