"""Field sharding + archive gather/scatter logic, world size 2 over gloo on
CPU (the NCCL path runs the same code on GPUs).  A stand-in codec (zlib of
the field bytes) replaces the GPU pipeline so the test needs no device."""

import os
import socket
import zlib

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _field(i):
    return np.random.default_rng(100 + i).standard_normal(1000 + 37 * i).astype(np.float32)


def _codec(field, bound):
    return zlib.compress(field.tobytes() + np.float64(bound).tobytes(), 6)


def _worker(rank, world, port, n_fields, q):
    import torch.distributed as dist
    from paper_2311_12133_b200 import multigpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        arcs = multigpu.compress_fields(_field, n_fields, 0.5, codec=_codec)
        if rank == 0:
            expect = [_codec(_field(i), 0.5) for i in range(n_fields)]
            q.put(("gather", arcs == expect))
        back = multigpu.decompress_fields(arcs, n_fields, codec=lambda a: zlib.decompress(a))
        ok = all(back[i][:-8] == _field(i).tobytes() for i in back)
        owned = sorted(back) == [i for i in range(n_fields) if i % world == rank]
        q.put((f"scatter{rank}", ok and owned))
    finally:
        dist.destroy_process_group()


def test_shard_gather_scatter_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_fields = 7
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_fields, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(3))
    assert res == {"gather": True, "scatter0": True, "scatter1": True}


def _worker_sub(rank, world, port, n_fields, q):
    """World 3; the batch runs on the subgroup {1, 2} (group ranks 0, 1)."""
    import torch.distributed as dist
    from paper_2311_12133_b200 import multigpu
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sub = dist.new_group([1, 2])
        if rank in (1, 2):
            arcs = multigpu.compress_fields(_field, n_fields, 0.25, codec=_codec, group=sub)
            if rank == 1:  # group rank 0
                expect = [_codec(_field(i), 0.25) for i in range(n_fields)]
                q.put(("gather", arcs == expect))
            back = multigpu.decompress_fields(arcs, n_fields, codec=lambda a: zlib.decompress(a),
                                              group=sub)
            gr = rank - 1
            ok = sorted(back) == [i for i in range(n_fields) if i % 2 == gr]
            ok = ok and all(back[i][:-8] == _field(i).tobytes() for i in back)
            q.put((f"scatter{gr}", ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_subgroup_peers_world3():
    """Peers are group ranks: a subgroup whose members are not global ranks
    0..n-1 still gathers on its own rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sub, args=(r, 3, port, 5, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(3))
    assert res == {"gather": True, "scatter0": True, "scatter1": True}
