"""Multi-GPU transport of the partitioned evaluation.

libtlfea packs, per peer, the partial 3x3 H blocks and partial nodal forces of
rows it touches but does not own (tlfea_eval_begin) and adds the received
partials in ascending peer order (tlfea_eval_finish); tlfea_eval_interior runs
the remaining elements while the buffers travel. This module only moves
the packed buffers between ranks with torch.distributed point-to-point
operations (NCCL over NVLink on a GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def offsets(counts) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.asarray(counts, np.int64))])


def exchange_start(send_buf, recv_buf, send_counts, recv_counts, group=None, host_staging: bool = False):
    """Start the transfer: send send_buf[soff[p]:soff[p+1]] to every peer p and
    receive recv_buf[roff[p]:roff[p+1]] from it, one batched group of P2P ops.
    With NCCL the operations run on the process group's own stream after the
    caller's stream reaches this point, so kernels the caller launches next
    (tlfea_eval_interior) overlap them. Returns the handles for exchange_wait.
    host_staging: move CUDA buffers through host memory, synchronously (gloo
    transport, used to run several ranks on one GPU in tests)."""
    import torch.distributed as dist
    if host_staging and send_buf.is_cuda:
        rh = recv_buf.new_empty(recv_buf.shape, device="cpu")
        exchange_wait(exchange_start(send_buf.cpu(), rh, send_counts, recv_counts, group))
        recv_buf.copy_(rh)
        return []
    soff, roff = offsets(send_counts), offsets(recv_counts)
    ops = []
    for p in range(len(send_counts)):
        if send_counts[p] > 0:
            ops.append(dist.P2POp(dist.isend, send_buf[int(soff[p]):int(soff[p + 1])], p, group))
        if recv_counts[p] > 0:
            ops.append(dist.P2POp(dist.irecv, recv_buf[int(roff[p]):int(roff[p + 1])], p, group))
    return dist.batch_isend_irecv(ops) if ops else []


def exchange_wait(works):
    """Order the caller's stream after the transfer (NCCL: a stream wait, not
    a host synchronization)."""
    for w in works:
        w.wait()


def exchange(send_buf, recv_buf, send_counts, recv_counts, group=None, host_staging: bool = False):
    """exchange_start + exchange_wait."""
    exchange_wait(exchange_start(send_buf, recv_buf, send_counts, recv_counts, group, host_staging))


def contiguous_partition(n_el: int, nranks: int) -> np.ndarray:
    """Default element partition: contiguous equal blocks of the element order
    (x-slabs for the lexicographic Kuhn meshes)."""
    return ((np.arange(n_el, dtype=np.int64) * nranks) // n_el).astype(np.int32)
