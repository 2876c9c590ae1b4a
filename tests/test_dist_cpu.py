"""N > 1 host logic on CPU: world_size-2 gloo process groups (127.0.0.1).

Covers what bench.py --gpus N runs around the kernels: cube sharding across
ranks, max-over-ranks timing and the whole-job rate; plus the pixel-sharded
Gram all-reduce named by the north_star (each rank's Gram of its pixel rows,
summed, equals the full Gram -- checked with the fp64 oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from harness import dist as hd
from harness import synth
from oracle import hyres_ref as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = hd.env_rank()
        own = hd.shard(64, r, w)
        # every rank's local "time" differs; the reported one is the max
        t_max = hd.max_over_ranks(1.0 + r)
        n_units = hd.sum_over_ranks(len(own))
        # pixel-sharded Gram: rank r owns pixel rows r, r + w, ... of the tiny cube
        s = synth.make_cube("tiny", 0)
        b, rows, cols = s.noisy.shape
        mine = s.noisy[:, r::w, :]
        g = torch.from_numpy(O.gram(np.ascontiguousarray(mine)))
        dist.all_reduce(g, op=dist.ReduceOp.SUM)
        q.put((r, own, t_max, n_units, g.numpy()))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_sharding_timing_and_gram_allreduce():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    owned = sorted(u for _, own, *_ in res for u in own)
    assert owned == list(range(64))                       # every cube exactly once
    assert all(abs(len(own) - 32) <= 1 for _, own, *_ in res)
    assert all(t == 2.0 for _, _, t, _, _ in res)          # max over ranks
    assert all(n == 64 for _, _, _, n, _ in res)
    full = O.gram(synth.make_cube("tiny", 0).noisy)
    for *_, g in res:
        assert np.allclose(g, full, rtol=1e-12, atol=1e-9 * np.abs(full).max())


def test_shard_and_rate_single_process():
    assert hd.shard(5, 0, 1) == [0, 1, 2, 3, 4]
    assert hd.shard(5, 1, 2) == [1, 3]
    with pytest.raises(ValueError):
        hd.shard(5, 2, 2)
    assert hd.max_over_ranks(3.5) == 3.5                   # no process group: identity
    assert hd.whole_job_rate(10.0, 2.0) == 5.0
    with pytest.raises(ValueError):
        hd.whole_job_rate(1.0, 0.0)
