"""E1 pixel-sharded single-cube path (include/hyde.h hyde_hyres_sharded) on ONE
GPU: G ranks are emulated by G host threads, each with its own handle and
stream, exchanging through an in-process communicator (the same hyde_comm
callbacks torch.distributed / NCCL implements on a multi-GPU box).  The
gathered result must equal the whole-cube hyres up to the summation order of
the Gram partials."""
import ctypes
import threading

import numpy as np
import pytest
import torch

from harness import metrics, synth
from oracle import hyres_ref as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hy():
    import paper_2204_06979_b200 as hy
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return hy


class ThreadComm:
    """In-process collectives among `world` threads on one GPU (host-synchronised
    copies: no kernel ever waits on another rank's kernel)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slot = [None] * world

    def _publish(self, rank, item, stream):
        torch.cuda.ExternalStream(stream).synchronize()   # the producing kernels are done
        self.slot[rank] = item
        self.bar.wait()
        return list(self.slot)

    def for_rank(self, hy, rank):
        def asum(t, stream):
            parts = self._publish(rank, t, stream)
            res = torch.zeros_like(t)
            for p in parts:                                   # fixed rank order
                res += p
            self.bar.wait()
            t.copy_(res)
            torch.cuda.synchronize()
            self.bar.wait()

        def sendrecv(sends, recvs, stream):
            parts = self._publish(rank, sends, stream)
            for peer in range(self.world):
                mine = [buf for (p, buf) in recvs if p == peer]
                theirs = [buf for (p, buf) in parts[peer] if p == rank]
                assert len(mine) == len(theirs), (rank, peer, len(mine), len(theirs))
                for dst, src in zip(mine, theirs):            # i-th send matches i-th receive
                    assert dst.numel() == src.numel()
                    dst.copy_(src)
            torch.cuda.synchronize()
            self.bar.wait()

        return hy.make_comm(rank, self.world, asum, sendrecv)


def run_sharded(hy, cube, world):
    b, rows, cols = cube.shape
    comm = ThreadComm(world)
    outs, infos, errs = [None] * world, [None] * world, []
    dev = torch.device("cuda", 0)

    def rank_main(r):
        try:
            hv = ctypes.c_void_p()
            hy._lib.check(hy._lib.lib().hyde_create(ctypes.byref(hv), 0))
            st = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(st):
                r0, r1 = hy.slab_rows(rows, r, world)
                local = torch.from_numpy(np.ascontiguousarray(cube[:, r0:r1, :])).to(dev)
                c = comm.for_rank(hy, r)
                out, info = hy.hyres_sharded(local, rows, c, handle_id=hv.value, return_info=True)
                st.synchronize()
            outs[r], infos[r] = out.cpu().numpy(), info
            hy._lib.lib().hyde_destroy(hv.value)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    return np.concatenate(outs, axis=1), infos


@pytest.mark.parametrize("name,world", [("tiny", 2), ("small", 3), ("wide", 2), ("small", 5), ("tiny", 8)])
def test_sharded_equals_whole_cube(hy, name, world):
    s = synth.make_cube(name, 0)
    whole, winfo = hy.hyres(torch.from_numpy(s.noisy).cuda(), return_info=True)
    whole = whole.cpu().numpy()
    got, infos = run_sharded(hy, s.noisy, world)
    assert all(i["rank"] == winfo["rank"] for i in infos)
    assert metrics.rel_l2(whole, got) < 1e-5
    if name != "wide":                       # the fp64 oracle is slow at the Houston shape
        ref = O.hyres(s.noisy)
        assert infos[0]["rank"] == ref.rank
        assert metrics.rel_l2(ref.out, got) < 1e-4
        assert abs(metrics.mpsnr(s.clean, got) - metrics.mpsnr(s.clean, ref.out)) < 0.01


def test_sharded_rejects_wrong_slab(hy):
    s = synth.make_cube("tiny", 0)
    comm = ThreadComm(2).for_rank(hy, 0)
    bad = torch.from_numpy(np.ascontiguousarray(s.noisy[:, :10, :])).cuda()   # rank 0 of 2 owns 32 rows
    with pytest.raises(hy.HydeError):
        hy.hyres_sharded(bad, 64, comm)


def test_sharded_nccl_world1_equals_whole_cube(hy):
    """World-size-1 NCCL communicator: every collective call site of hyde_hyres_sharded
    (Gram all-reduce, slab <-> component exchange as self copies, SURE statistics
    all-reduce) runs through libhyde's NCCL on one GPU."""
    assert hy._lib.lib().hyde_nccl_version() >= 22000
    for name in ("tiny", "small"):
        s = synth.make_cube(name, 0)
        x = torch.from_numpy(s.noisy).cuda()
        whole, winfo = hy.hyres(x, return_info=True)
        comm = hy.nccl_comm_single()
        try:
            got, info = hy.hyres_sharded(x, s.noisy.shape[1], comm, return_info=True)
            torch.cuda.synchronize()
        finally:
            comm.close()
        assert info["rank"] == winfo["rank"]
        assert metrics.rel_l2(whole.cpu().numpy(), got.cpu().numpy()) < 1e-6


def test_sharded_nonfinite_on_one_rank_stops_every_rank(hy):
    """a NaN in ONE rank's slab must return HYDE_EDATA on every rank
    (no rank left waiting in a collective)."""
    s = synth.make_cube("tiny", 0)
    cube = s.noisy.copy()
    cube[3, 50, 7] = np.nan                      # rows 32..63: rank 1 of 2
    with pytest.raises(hy.HydeError) as ei:
        run_sharded(hy, cube, 2)
    assert ei.value.status == 3


def test_shard_plan_covers_rows_and_components(hy):
    for rows, world in [(64, 2), (349, 8), (7, 7), (1024, 3)]:
        spans = [hy.slab_rows(rows, g, world) for g in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == rows
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        own = [hy.component_owner(k, world) for k in range(40)]
        assert own == [k % world for k in range(40)]
