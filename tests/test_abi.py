"""The C-ABI library builds for sm_100a, loads without a GPU, exports every
symbol include/tlfea.h declares, and refuses to run without a device (no CPU
fallback). CPU-only."""
import os
import re
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    import paper_2604_10357_b200 as T
    from paper_2604_10357_b200 import build
    build.build()
    T.lib()
    return T


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tlfea.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tlfea_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(T):
    names = declared_symbols()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", T.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tlfea_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(T.EXPORTED) <= exported


def test_sm100a_code_in_library(T):
    out = subprocess.run(["cuobjdump", "--list-elf", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_no_cpu_fallback(T):
    assert T.lib().tlfea_abi_version() == 8
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the no-device path is exercised on CPU hosts")
    mesh = synth.kuhn_t10_box(1, 1, 1, 1, 1, 1)
    with pytest.raises(T.TlfeaError, match="no CUDA device"):
        T.Context.from_mesh(mesh, synth.SVK_PAPER, 1)


def test_plan_partition_host_only(T):
    mesh = synth.kuhn_t10_box(4, 2, 2, 1, 1, 1)
    part = (np.arange(mesh.n_el) * 2 // mesh.n_el).astype(np.int32)
    owner, sb, sbp, sn, snp = T.tlfea_plan_partition(mesh.conn, mesh.n_coef, part, 2, 1)
    # reading Q20: a node is owned by the lowest rank among its incident elements
    ref = np.full(mesh.n_coef, 2)
    for e in range(mesh.n_el):
        ref[mesh.conn[e]] = np.minimum(ref[mesh.conn[e]], part[e])
    assert np.array_equal(owner, ref)
    # rank 1 sends exactly the rows of rank-0-owned nodes its elements touch
    touched = set(mesh.conn[part == 1].ravel())
    assert set(sn) == {i for i in touched if owner[i] == 0}
    assert np.all(snp == 0) and np.all(sbp == 0)
    # blocks in canonical (peer, I, J) order, unique
    keys = [tuple(k) for k in sb]
    assert keys == sorted(set(keys))
    # rank 0 sends nothing (it owns every node it touches)
    _, sb0, _, sn0, _ = T.tlfea_plan_partition(mesh.conn, mesh.n_coef, part, 2, 0)
    assert len(sb0) == 0 and len(sn0) == 0


def test_nccl_unique_id_host_only(T):
    """tlfea_nccl_get_unique_id loads libnccl.so.2 at run time (no link-time
    NCCL dependency) and returns a 128-byte ncclUniqueId without a GPU."""
    uid = T.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
    out = subprocess.run(["ldd", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "libnccl" not in out
