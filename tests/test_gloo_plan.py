"""World-size-2 host logic of the multi-rank path on CPU (gloo): each rank
counts its own row, the rows are all-gathered (the count exchange),
and rafi_plan on every rank yields the oracle's receive plan and the same G
and overflow decision."""
import os
import tempfile
import uuid

import numpy as np
import pytest


def _free_port():
    """A fresh file:// rendezvous for the gloo group (no TCP port to race for:
    a port probed free and then bound by the workers can be taken in between)."""
    return "file://" + os.path.join(tempfile.gettempdir(), "rafi_pg_%d_%s" % (os.getpid(), uuid.uuid4().hex))


def _worker(rank, world, port, cap, n):
    import torch
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2605_30294_b200 import build, rafi

    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    ds = synth.make_dests("skewed", 3, rank, 0, n, world)
    row = torch.from_numpy(np.bincount(ds, minlength=world).astype(np.int64))
    rows = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(rows, row)
    Cm = torch.stack(rows).numpy().astype(np.uint64)
    build.build()
    p = rafi.plan(Cm, cap, rank)
    # oracle: all ranks simulated in one world
    w = oracle.World(world, cap, 16)
    for s in range(world):
        d = synth.make_dests("skewed", 3, s, 0, n, world)
        it = synth.make_items(s, 0, n, 16)
        for i in range(n):
            w.emit(s, it[i].tobytes(), int(d[i]))
    G = w.forward()
    if G < 0:
        assert p["overflow"]
    else:
        assert not p["overflow"] and p["G"] == G
        assert list(p["recv_off"]) == list(w.recv_off()[rank])
        assert list(p["src_off"]) == list(w.send_off()[:, rank])
        assert p["total"] == w.num_incoming(rank)
    dist.destroy_process_group()


@pytest.mark.parametrize("cap", [2000, 1100])   # 1100: some rank overflows (Z3)
def test_gloo_world2_plan(cap):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), cap, 1000), nprocs=2, join=True)


def _worker_allgather(rank, world, port):
    import ctypes

    import torch.distributed as dist

    from paper_2605_30294_b200 import rafi

    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    fn = rafi.torch_allgather()
    for nbytes in (0, 1, 13, 4096):
        send = (ctypes.c_uint8 * max(nbytes, 1))(*[(rank * 31 + i) & 0xFF for i in range(max(nbytes, 1))])
        recv = (ctypes.c_uint8 * max(world * nbytes, 1))()
        assert fn(None, ctypes.addressof(send), ctypes.addressof(recv), nbytes) == 0
        for p in range(world):
            got = bytes(recv[p * nbytes:(p + 1) * nbytes])
            assert got == bytes((p * 31 + i) & 0xFF for i in range(nbytes)), (p, nbytes)
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_allgather():
    """rafi.torch_allgather -- the host all-gather behind rafi_create_boot and
    HOST control (the paper's MPI host transport) -- on a gloo
    world of 2: every process receives every process's bytes in rank order,
    for empty, odd-sized and page-sized payloads."""
    import torch.multiprocessing as mp
    mp.spawn(_worker_allgather, args=(2, _free_port()), nprocs=2, join=True)
