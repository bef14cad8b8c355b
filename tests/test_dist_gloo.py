"""bench.py's data-parallel path on CPU with gloo, world size 2.

Drives bench.py's own multi-GPU plumbing — `shard_bounds` (contiguous batch
slices), `timed_steps` (barrier + sync on both sides), `max_over_ranks` and
`gather_logits` (the forward's only collective) — with the CPU oracle standing
in for the device forward (no GPU here). The gathered logits must equal the
single-process forward of the whole batch bit for bit: samples are independent
(fresh detector state per sample, quant.cpp:477-481). Also checks that
`bench.py --gpus 2` outside torchrun re-launches itself as two ranks.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS = dict(image=16, channels=3, patch=4, embed=16, state=4, blocks=2, classes=7, conv_width=3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import time
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    chk = O.Checker(O.ORACLE_SO)
    d = O.Dims(**DIMS)
    m = chk.model(d, 9)
    B = 7  # uneven split: ranks get 3 and 4 samples
    imgs = chk.normal(3, B * d.pix).reshape(B, -1)
    cal = m.calibrate(chk.normal(4, 3 * d.pix), O.Spec(abits=4, obits=8, n_refresh=3, rho=0.1))
    s0, s1 = bench.shard_bounds(B, rank, world)
    state = {}

    def step():  # the device forward's stand-in on this rank's shard
        state["mine"] = torch.from_numpy(m.forward(imgs[s0:s1], cal, 1, threads=1))

    def wall_timer():
        t = {}
        return (lambda: t.__setitem__(0, time.perf_counter())), (lambda: t.__setitem__(1, time.perf_counter())), \
            (lambda: 1e3 * (t[1] - t[0]))

    ms = bench.timed_steps(step, 2, world, dist, lambda: None, wall_timer)
    ms_max = bench.max_over_ranks(dist, ms, world, "cpu")
    # gather_logits needs equal shard sizes (all_gather); pad to the largest shard
    per = max(bench.shard_bounds(B, r, world)[1] - bench.shard_bounds(B, r, world)[0] for r in range(world))
    mine = torch.zeros(per, d.classes, dtype=torch.float64)
    mine[:s1 - s0] = state["mine"]
    allg = bench.gather_logits(dist, mine, world)
    sizes = [bench.shard_bounds(B, r, world)[1] - bench.shard_bounds(B, r, world)[0] for r in range(world)]
    got = torch.cat([allg[r * per:r * per + sizes[r]] for r in range(world)]).numpy()
    if rank == 0:
        full = m.forward(imgs, cal, 1, threads=1)
        q.put((bool(np.array_equal(got, full)), ms_max >= ms, sizes))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_forward_matches_single_process(oracle_checker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, max_ok, sizes = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok and max_ok and sizes == [3, 4]


def test_shard_bounds_cover_batch():
    sys.path.insert(0, ROOT)
    import bench
    for B in (1, 7, 256, 1000):
        for world in (1, 2, 3, 8):
            cuts = [bench.shard_bounds(B, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == B
            assert all(cuts[r][1] == cuts[r + 1][0] for r in range(world - 1))


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2 --impl reference` outside torchrun runs as two
    torchrun ranks: rank 0 prints the line, rank 1 exits 0 without work."""
    from oracle import oracle as O
    if not O.ref_available():
        import pytest
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--embed", "32", "--blocks", "2", "--image", "32", "--steps", "1", "--warmup", "0",
                        "--batch", "2"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    import json
    assert json.loads(lines[0])["n_gpus"] == 2
