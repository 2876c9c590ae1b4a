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


# ------------------------------------------------------------------------------
# E1 decomposition (include/hyde.h hyde_hyres_sharded) on CPU: world-size-2 gloo
# ranks run the library's partition -- slab rows and component ownership from
# libhyde's own host functions (hyde_shard_rows / hyde_shard_owner, no GPU) --
# with the fp64 oracle's arithmetic in every step, exchanging exactly the
# messages the library exchanges (Gram all-reduce; slab -> component sends in
# ascending component order; per-subband SURE statistics all-reduced; component
# -> slab rows).  The gathered result must equal the oracle on the whole cube:
# the partition, the message matching and the shared rank decision are right.
def _e1_worker(rank, world, port, name, q):
    import ctypes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_06979_b200 import _lib
        L = _lib.lib()

        def rows_of(g, rows):
            r0, nr = ctypes.c_int(0), ctypes.c_int(0)
            assert L.hyde_shard_rows(rows, world, g, ctypes.byref(r0), ctypes.byref(nr)) == 0
            return r0.value, r0.value + nr.value

        s = synth.make_cube(name, 0)
        cube = s.noisy
        b, rows, cols = cube.shape
        n = rows * cols
        r0, r1 = rows_of(rank, rows)
        y_loc = cube[:, r0:r1, :].reshape(b, -1).astype(np.float64)
        g = torch.from_numpy(y_loc @ y_loc.T)
        dist.all_reduce(g)                                          # A1
        g = g.numpy()
        m = np.linalg.inv(g + 1e-6 * np.eye(b))
        sigma = np.sqrt(1.0 / (n * np.diag(m)))
        lam, v, _ = O.whiten_eig(g, sigma, n)                        # A2 replicated
        lv = O.auto_levels(rows, cols)
        nc = O.coeff_count(rows, cols, lv)
        first = min(16, max(4, world))
        k0, c, rank_star, den_loc = 0, 0, None, {}
        while rank_star is None:
            cnt = min(b - k0, min(16, first << c))
            e_loc = (v[:, k0:k0 + cnt] / sigma[:, None]).T @ y_loc    # A3 on the slab
            owner = [L.hyde_shard_owner(k0 + k, world) for k in range(cnt)]
            mine = [k for k in range(cnt) if owner[k] == rank]
            full = {k: np.zeros((rows, cols)) for k in mine}
            for k in range(cnt):                                     # slab -> component
                for gsrc in range(world):
                    a0, a1 = rows_of(gsrc, rows)
                    if gsrc == rank and owner[k] == rank:
                        full[k][a0:a1] = e_loc[k].reshape(a1 - a0, cols)
                    elif gsrc == rank:
                        dist.send(torch.from_numpy(np.ascontiguousarray(e_loc[k])), owner[k])
                    elif owner[k] == rank:
                        t = torch.empty((a1 - a0) * cols, dtype=torch.float64)
                        dist.recv(t, gsrc)
                        full[k][a0:a1] = t.numpy().reshape(a1 - a0, cols)
            stats = torch.zeros(cnt, dtype=torch.float64)
            soft = {}
            for k in mine:                                           # A4/A5 of owned images
                co = O.dwt2(full[k], lv)
                subs = O.flatten_coeffs(co)
                sb = [O.soft_threshold(x, O.sure_threshold(x).t) for x in subs]
                stats[k] = float(sum(np.sum(x * x) for x in sb))
                soft[k] = (sb, co)
            dist.all_reduce(stats)                                   # every rank: all E_post
            kept = cnt
            for k in range(cnt):                                     # first-failure rule
                if stats[k] <= nc:
                    rank_star = max(1, k0 + k)
                    kept = rank_star - k0
                    break
            for k in range(kept):                                    # IDWT owned kept -> slab rows
                if owner[k] == rank:
                    sb, co = soft[k]
                    img = O.idwt2(O.unflatten_coeffs(sb, co))
                    for gdst in range(world):
                        a0, a1 = rows_of(gdst, rows)
                        if gdst == rank:
                            den_loc[k0 + k] = img[a0:a1].ravel()
                        else:
                            dist.send(torch.from_numpy(np.ascontiguousarray(img[a0:a1].ravel())), gdst)
                else:
                    t = torch.empty((r1 - r0) * cols, dtype=torch.float64)
                    dist.recv(t, owner[k])
                    den_loc[k0 + k] = t.numpy()
            if rank_star is None and k0 + cnt >= b:
                rank_star = b
            k0 += cnt
            c += 1
        u = v[:, :rank_star] * sigma[:, None]
        out_loc = (u @ np.stack([den_loc[k] for k in range(rank_star)])).reshape(b, r1 - r0, cols)
        q.put((rank, r0, out_loc.astype(np.float32), rank_star))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("tiny", 2), ("small", 3)])
def test_e1_partition_gloo_equals_oracle(name, world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_e1_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([x[2] for x in res], axis=1)
    ref = O.hyres(synth.make_cube(name, 0).noisy)
    assert all(x[3] == ref.rank for x in res)
    assert np.max(np.abs(got - ref.out)) <= 1e-5 * np.max(np.abs(ref.out))
