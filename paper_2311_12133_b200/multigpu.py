"""Batch compression of independent fields across GPUs.

The path shards only by field: a single field is never split (anchors and
edge stencils would change, so the archive would no longer match the
reference).  Field i belongs to rank i % world_size.  Every rank compresses
its own fields with the full B200 pipeline, then

Peers are addressed by group rank (``group_peer``), so subgroups work.

* all ranks learn every archive's size with one all-reduce of an int64
  vector (``ncclAllReduce`` over NVLink on GPUs, gloo on CPU), and
* rank 0 receives the archives with batched point-to-point transfers
  (``ncclSend/ncclRecv``), in field order.

Decompression mirrors this: rank 0 sends each archive to its owner.  The
reference's own batch mode is a process pool with one field per worker
(cli.py:183-193); this is the same decomposition with GPUs as workers.
"""

from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def owner(i: int, world: int) -> int:
    return i % world


def _comm_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_archives(local: dict, n_fields: int, group=None) -> list | None:
    """``local`` maps field index -> archive bytes for this rank's fields.
    Returns the ordered list of archives on rank 0, None elsewhere."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _comm_device(group)
    sizes = torch.zeros(n_fields, dtype=torch.int64, device=dev)
    for i, blob in local.items():
        sizes[i] = len(blob)
    dist.all_reduce(sizes, group=group)
    sizes_h = sizes.cpu().tolist()
    ops, recv = [], {}
    if rank == 0:
        for i in range(n_fields):
            src = owner(i, world)
            if src == 0:
                continue
            buf = torch.empty(sizes_h[i], dtype=torch.uint8, device=dev)
            recv[i] = buf
            ops.append(dist.P2POp(dist.irecv, buf, group=group, group_peer=src))
    else:
        for i in sorted(local):
            t = torch.frombuffer(bytearray(local[i]), dtype=torch.uint8).to(dev)
            ops.append(dist.P2POp(dist.isend, t, group=group, group_peer=0))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if rank != 0:
        return None
    out = []
    for i in range(n_fields):
        out.append(local[i] if owner(i, world) == 0 else recv[i].cpu().numpy().tobytes())
    return out


def scatter_archives(archives: Sequence[bytes] | None, n_fields: int, group=None) -> dict:
    """Rank 0 holds every archive; each rank receives the ones it owns."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _comm_device(group)
    sizes = torch.zeros(n_fields, dtype=torch.int64, device=dev)
    if rank == 0:
        for i, a in enumerate(archives):
            sizes[i] = len(a)
    dist.broadcast(sizes, group=group, group_src=0)
    sizes_h = sizes.cpu().tolist()
    mine, ops, recv = {}, [], {}
    for i in range(n_fields):
        dst = owner(i, world)
        if rank == 0:
            if dst == 0:
                mine[i] = archives[i]
            else:
                t = torch.frombuffer(bytearray(archives[i]), dtype=torch.uint8).to(dev)
                ops.append(dist.P2POp(dist.isend, t, group=group, group_peer=dst))
        elif dst == rank:
            buf = torch.empty(sizes_h[i], dtype=torch.uint8, device=dev)
            recv[i] = buf
            ops.append(dist.P2POp(dist.irecv, buf, group=group, group_peer=0))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for i, buf in recv.items():
        mine[i] = buf.cpu().numpy().tobytes()
    return mine


def compress_fields(make_field: Callable[[int], object], n_fields: int, bound, *,
                    codec: Callable | None = None, group=None, **kw) -> list | None:
    """Compress fields 0..n_fields-1 sharded over the process group.

    ``make_field(i)`` builds (or loads) field i on its owner only.  ``codec``
    defaults to the B200 ``pipeline.compress`` (returning ``.archive``)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = [i for i in range(n_fields) if owner(i, world) == rank]
    local = {}
    if codec is None:
        # B200 pipeline: field i's host zlib stage overlaps field i+1's GPU stage
        from .pipeline import compress_many
        for i, res in zip(mine, compress_many((make_field(i) for i in mine), bound, **kw)):
            local[i] = res.archive
    else:
        for i in mine:
            local[i] = codec(make_field(i), bound, **kw)
    return gather_archives(local, n_fields, group=group)


def decompress_fields(archives: Sequence[bytes] | None, n_fields: int, *,
                      codec: Callable | None = None, group=None) -> dict:
    """Inverse of compress_fields: returns {field index: grid} for this rank."""
    if codec is None:
        from .pipeline import decompress as codec
    mine = scatter_archives(archives, n_fields, group=group)
    return {i: codec(a) for i, a in mine.items()}
