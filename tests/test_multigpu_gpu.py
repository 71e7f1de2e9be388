"""The real B200 pipeline under torch.distributed: world size 2 (gloo for the
host-side archive exchange, both ranks on cuda:0 -- independent fields, no
rank waits on another's kernels), multigpu.compress_fields / decompress_fields
against single-process pipeline.compress / decompress."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

DIMS = (72, 80, 96)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grid(i):
    import synthetic as syn
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    return ScalarGrid(DIMS, ElementKind.F32, syn.config_field(5, index=i, dims=DIMS))


def _worker(rank, world, port, n_fields, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_2311_12133_b200 import multigpu
    from paper_2311_12133_b200.grid import BoundMode, ErrorBoundSpec
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = ErrorBoundSpec(BoundMode.REL, 1e-3)
        arcs = multigpu.compress_fields(_grid, n_fields, spec)
        if rank == 0:
            q.put(("arcs", [bytes(a) for a in arcs]))
        back = multigpu.decompress_fields(arcs, n_fields)
        q.put((f"back{rank}", {i: g.data.tobytes() for i, g in back.items()}))
    finally:
        dist.destroy_process_group()


def test_compress_fields_real_pipeline_world2():
    from paper_2311_12133_b200.grid import BoundMode, ErrorBoundSpec
    from paper_2311_12133_b200.pipeline import compress
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    n_fields = 3
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_fields, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(3))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    spec = ErrorBoundSpec(BoundMode.REL, 1e-3)
    expect = [compress(_grid(i), spec) for i in range(n_fields)]
    assert res["arcs"] == [e.archive for e in expect]
    got = {**res["back0"], **res["back1"]}
    assert sorted(got) == list(range(n_fields))
    for i, e in enumerate(expect):
        assert got[i] == e.reconstruction.data.tobytes()
