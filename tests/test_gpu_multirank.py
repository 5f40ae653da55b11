"""The partitioned path across real processes on one GPU:
torch.distributed.run starts P ranks of tools/multirank_check.py, each with its
own partitioned context; begin / exchange (gloo, host-staged) / interior /
finish; rank 0 compares the gathered owned rows with the oracle."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("P", [2, 3])
def test_multirank_processes_match_oracle(P):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "multirank_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == P and out["pattern_ok"] and out["rows_partition"]
    assert out["rel_g"] <= 1e-11 and out["rel_H"] <= 1e-11 and out["rel_f"] <= 1e-11, out


@pytest.mark.parametrize("P", [2])
def test_multirank_library_nccl_transport(P):
    """The library's own NCCL transport (tlfea_nccl_attach + tlfea_eval_exchange),
    one rank per GPU: needs P devices (NCCL refuses two ranks on one GPU)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} CUDA devices")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "multirank_check.py"),
           "--transport", "lib"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert out["transport"] == "lib" and out["pattern_ok"] and out["rows_partition"]
    assert out["rel_g"] <= 1e-11 and out["rel_H"] <= 1e-11 and out["rel_f"] <= 1e-11, out


def test_library_nccl_single_rank():
    """tlfea_nccl_attach on a one-rank communicator and the begin / exchange /
    interior / finish sequence: bitwise the plain evaluation (the dlopen'd NCCL,
    the communicator, the event ordering on one device)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import numpy as np

    import paper_2604_10357_b200 as T
    import synth
    mesh, mat = synth.kuhn_t10_box(3, 2, 2, 0.6, 0.4, 0.4), dict(synth.SVK_PAPER, **synth.KV_TIRE)
    x, v, vn, fext = synth.t10_state(mesh, with_fext=True)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ctx = T.Context.from_mesh(mesh, mat, 1)
    g0, H0, f0 = ctx.empty_outputs()
    ctx.eval(d(x), d(v), d(vn), d(fext), 1e-3, g0, H0, f0)
    ctx.nccl_attach(T.nccl_unique_id())
    with pytest.raises(T.TlfeaError, match="INVALID"):
        ctx.nccl_attach(T.nccl_unique_id())          # one communicator per context
    g, H, f = ctx.empty_outputs()
    buf = torch.zeros(1, dtype=torch.float64, device="cuda")
    ctx.eval_begin(d(x), d(v), 1e-3, H, buf)
    ctx.eval_exchange(buf, buf)
    ctx.eval_interior(d(x), d(v), 1e-3, H)
    ctx.eval_finish(buf, d(v), d(vn), d(fext), 1e-3, g, H, f)
    torch.cuda.synchronize()
    assert torch.equal(g, g0) and torch.equal(H, H0) and torch.equal(f, f0)


def test_bench_two_ranks_one_gpu():
    """bench.py's N>1 path (partitioned setup, begin / exchange / interior /
    finish, max-over-ranks timing, global accounting) under torch.distributed.run
    with 2 ranks sharing the GPU over gloo: the line is well formed (timings
    meaningless on one shared device)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, TLFEA_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "2", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert out["n_gpus"] == 2 and out["value"] > 0
    assert out["config"]["nnz_H"] == 34_979_121          # global accounting on a partitioned run
    assert abs(out["config"]["path_alg_bytes_per_el"] - out["roofline"]["alg_bytes_per_el"]) < 1e-6
