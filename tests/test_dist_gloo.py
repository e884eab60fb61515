"""Host-side logic of the z-slab decomposition, multi-process on CPU
(torch.distributed gloo, world_size 2 and 3): every rank builds its local
grid (slab + ghosts) with the product's slab initialisers, exchanges ghost
planes with the same partition / ghost rules st_dist_* uses
(st_dist_partition), and must end up holding exactly its window of the
global grid.  Also checks the timing protocol the bench uses for N > 1
(max over ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CF.get(5).scaled((12 * world, 10, 14), 4)
        spec = P.StencilSpec.make("w", 3, [P.StencilTerm(c, dt, o) for c, dt, o in cfg.terms], model=1)
        r = cfg.radius
        ghost = r * 2
        gext = cfg.extents
        z0, nzs, glo, ghi = P.dist_partition(gext[0], world, rank, ghost)
        lext = (nzs + glo + ghi,) + tuple(gext[1:])
        centre = [e // 2 for e in gext]
        # local grid: global Gaussian evaluated on global planes [z0-glo, z0+nzs+ghi)
        loc = P.init_gaussian(spec, P.IterationSpace(4, lext), 3, cfg.sigma, centre, z_begin=z0 - glo)
        full = P.init_gaussian(spec, P.IterationSpace(4, gext), 3, cfg.sigma, centre)
        lv = loc.view()
        # wipe the ghosts, then refill them by exchange (plane blocks, z slowest)
        lv[:, r:r + glo] = 0
        lv[:, r + glo + nzs: r + glo + nzs + ghi] = 0
        reqs = []
        if rank > 0:
            send = torch.from_numpy(np.ascontiguousarray(lv[:2, r + glo: r + glo + glo]))
            recv = torch.empty_like(send)
            reqs += [dist.isend(send, rank - 1), dist.irecv(recv, rank - 1)]
        if rank < world - 1:
            send2 = torch.from_numpy(np.ascontiguousarray(lv[:2, r + glo + nzs - ghi: r + glo + nzs]))
            recv2 = torch.empty_like(send2)
            reqs += [dist.isend(send2, rank + 1), dist.irecv(recv2, rank + 1)]
        for rq in reqs:
            rq.wait()
        if rank > 0:
            lv[:2, r: r + glo] = recv.numpy()
        if rank < world - 1:
            lv[:2, r + glo + nzs: r + glo + nzs + ghi] = recv2.numpy()
        fv = full.view()
        ok = bool(np.array_equal(lv[:2, r: r + lext[0]], fv[:2, r + z0 - glo: r + z0 - glo + lext[0]]))
        # bench timing protocol: max over ranks
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok, float(t.item()), (z0, nzs, glo, ghi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_ghost_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    assert all(t == float(world) for _, _, t, _ in res)
    # partition covers the global grid exactly, ghosts only at interior faces
    spans = [part for *_, part in res]
    assert spans[0][2] == 0 and spans[-1][3] == 0
    assert sum(s[1] for s in spans) == 12 * world
    for a, b in zip(spans, spans[1:]):
        assert a[0] + a[1] == b[0]


def test_partition_rules():
    assert P.dist_partition(512, 1, 0, 16) == (0, 512, 0, 0)
    assert P.dist_partition(1024, 2, 1, 16) == (512, 512, 16, 0)
    assert P.dist_partition(1030, 4, 2, 8)[2:] == (8, 8)
    with pytest.raises(P.Error):
        P.dist_partition(10, 4, 1, 8)          # ghost deeper than a slab
    with pytest.raises(P.Error):
        P.dist_partition(10, 2, 2, 1)          # bad rank
