"""Batch sharding (bench.py's data-parallel path) on CPU with gloo, world
size 2: each rank runs its contiguous slice of the batch, the logits are
all-gathered, and the result is bit-identical to the single-process run
(per-sample detector state makes samples independent, quant.cpp:477-481)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

DIMS = dict(image=16, channels=3, patch=4, embed=16, state=4, blocks=2, classes=7, conv_width=3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    chk = O.Checker(O.ORACLE_SO)
    d = O.Dims(**DIMS)
    m = chk.model(d, 9)
    B = 6
    imgs = chk.normal(3, B * d.pix).reshape(B, -1)
    cal = m.calibrate(chk.normal(4, 3 * d.pix), O.Spec(abits=4, obits=8, n_refresh=3, rho=0.1))
    per = B // world
    mine = m.forward(imgs[rank * per:(rank + 1) * per], cal, 1, threads=1)
    parts = [torch.empty(per, d.classes, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(mine))
    if rank == 0:
        full = m.forward(imgs, cal, 1, threads=1)
        q.put(bool(np.array_equal(torch.cat(parts).numpy(), full)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_forward_matches_single_process(oracle_checker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
