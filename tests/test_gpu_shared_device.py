"""Cross-process forwarding on ONE GPU: two processes share cuda:0.

The multi-GPU suite (test_gpu_multiproc.py) needs >= 2 GPUs; this module runs
the cross-process machinery on the single GPU the round-end tests get:

  * rafi_create_boot with a gloo host bootstrap (no NCCL: NCCL refuses two
    ranks on one device): CUDA-IPC handles of every queue travel through the
    host all-gather, together with (item_bytes, capacity, local_ranks), which
    must agree;
  * RAFI_CONTROL_HOST, the paper's host-side count exchange: count
    rows to the host, host all-gather, device plan, scatter, host barrier;
  * the FUSED exchange pushing every destination run straight into the other
    process's incoming queue through its CUDA-IPC mapping, and the staged PEER
    exchange pulling from the other process's send batch.

No kernel ever waits on a flag another process raises (PEER control is
refused when processes share a device: nothing co-schedules their kernels),
so the two processes' kernels may time-slice freely.  Every round is checked
bit-exactly against the oracle run on both processes' snapshots (P1).
"""
import os
import tempfile
import uuid

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)


def _free_port():
    """A fresh file:// rendezvous for the gloo group (no TCP port to race for:
    a port probed free and then bound by the workers can be taken in between)."""
    return "file://" + os.path.join(tempfile.gettempdir(), "rafi_pg_%d_%s" % (os.getpid(), uuid.uuid4().hex))


def _worker(rank, world, port, B, L, n, pattern, exchange, rounds, resize_round):
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2605_30294_b200 import rafi

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    R = world * L
    cap = R * n  # any pattern fits (all_to_one sends everything to one rank)
    stream = torch.cuda.Stream()
    ctx = rafi.Context(B, cap, stream=stream, local_ranks=L, bootstrap=(world, rank, rafi.torch_allgather()))
    assert ctx.num_ranks == R and ctx.rank_of(0) == rank * L
    # processes share the device: AUTO control is HOST, PEER control is refused
    assert ctx.get_option(rafi.OPT_CONTROL) == rafi.CONTROL_HOST
    with pytest.raises(rafi.RafiError):
        ctx.set_option(rafi.OPT_CONTROL, rafi.CONTROL_PEER)
    assert ctx.get_option(rafi.OPT_CONTROL) == rafi.CONTROL_HOST
    ctx.set_option(rafi.OPT_EXCHANGE, exchange)
    assert ctx.get_option(rafi.OPT_EXCHANGE) == exchange
    with pytest.raises(rafi.RafiError):        # HOST control synchronises with the host: not capturable
        ctx.forward_async(torch.zeros(1, dtype=torch.int64, device="cuda"))
    for rnd in range(rounds):
        if rnd == resize_round:
            cap = R * n + 1000
            ctx.resize(cap)                    # collective; old queues freed after every process unmapped them
            assert ctx.capacity == cap
        m = n if rnd % 2 == 0 else n // 3 + rnd
        for l in range(L):
            g = rank * L + l
            it = synth.make_items(g, rnd, m, max(B, 16))[:, :B].copy()
            ds = synth.make_dests(pattern, 31 + rnd, g, rnd, m, R, invalid_frac=0.01)
            ctx.emit_bulk(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), m, local=l)
        snaps = [ctx.read_outgoing(l) for l in range(L)]
        allsnaps = [None] * world
        dist.all_gather_object(allsnaps, snaps)
        w = oracle.World(R, cap, B)
        for p, sn in enumerate(allsnaps):
            for l, (items, dests, ctr, inv) in enumerate(sn):
                w.load_snapshot(p * L + l, items, dests, ctr, inv)
        G_o = w.forward()
        G = ctx.forward_rc()
        assert G == G_o, (rank, rnd, G, G_o)
        assert np.array_equal(ctx.matrix(), w.C())
        for l in range(L):
            g = rank * L + l
            st = ctx.stats(l)
            assert st["num_in"] == w.num_incoming(g)
            if exchange == rafi.EXCHANGE_PEER:
                assert np.array_equal(ctx.read_binned(l, st["n_out"]), w.binned(g, st["n_out"]))
            assert np.array_equal(ctx.read_incoming(l), w.incoming(g)), (rank, rnd, l)
    assert ctx.forward() == 0                  # termination on both processes
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", [3, 2])   # FUSED (push over IPC), PEER (staged pull over IPC)
@pytest.mark.parametrize("B,L,n,pattern", [(48, 1, 30011, "uniform"), (44, 2, 20000, "skewed"),
                                           (16, 3, 5000, "all_to_one")])
def test_two_processes_one_gpu_host_control(B, L, n, pattern, exchange):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), B, L, n, pattern, exchange, 4, 2), nprocs=2, join=True)


def _worker_mismatch(rank, world, port):
    import torch.distributed as dist

    from paper_2605_30294_b200 import rafi

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    # the processes disagree on the capacity: creation fails on BOTH
    with pytest.raises(rafi.RafiError) as e:
        rafi.Context(32, 1000 + rank, bootstrap=(world, rank, rafi.torch_allgather()))
    assert e.value.status == rafi.ERR_INVALID_ARG
    ctx = rafi.Context(32, 1000, bootstrap=(world, rank, rafi.torch_allgather()))
    with pytest.raises(rafi.RafiError) as e:
        ctx.resize(2000 + rank)                # and so does a resize, before anything changes
    assert e.value.status == rafi.ERR_INVALID_ARG and ctx.capacity == 1000
    assert ctx.forward() == 0
    ctx.close()
    dist.destroy_process_group()


def test_two_processes_disagreeing_parameters():
    import torch.multiprocessing as mp
    mp.spawn(_worker_mismatch, args=(2, _free_port()), nprocs=2, join=True)
