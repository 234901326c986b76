"""Multi-GPU parity: one process per GPU, NCCL communicator, both payload
transports (PEER copy kernel over CUDA-IPC NVLink pointers; NCCL grouped
send/recv).  Every rank checks its own outputs bit-exactly against the oracle
run on all ranks' snapshots (P1)."""
import os
import tempfile
import uuid

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 CUDA GPUs", allow_module_level=True)


def _need(world):
    """Skip unless `world` GPUs are visible (and, when RAFI_TEST_WORLDS is set,
    e.g. "2", unless world is one of the listed sizes)."""
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs" % world)
    only = os.environ.get("RAFI_TEST_WORLDS")
    if only and str(world) not in only.split(","):
        pytest.skip("world %d not selected by RAFI_TEST_WORLDS" % world)


def _free_port():
    """A fresh file:// rendezvous for the gloo group (no TCP port to race for:
    a port probed free and then bound by the workers can be taken in between)."""
    return "file://" + os.path.join(tempfile.gettempdir(), "rafi_pg_%d_%s" % (os.getpid(), uuid.uuid4().hex))


def _worker(rank, world, port, B, n, pattern, exchange, rounds, scatter=1, control=0, comm_mode="nccl"):
    """comm_mode: "nccl" (rafi_create_ex with an NCCL communicator), "both"
    (NCCL communicator + gloo bootstrap) or "boot" (gloo bootstrap only, no
    NCCL in the library)."""
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2605_30294_b200 import rafi

    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    comm = None
    if comm_mode in ("nccl", "both"):
        obj = [rafi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = rafi.nccl_comm_init(world, rank, obj[0], rank)
    boot = (world, rank, rafi.torch_allgather()) if comm_mode in ("both", "boot") else None
    cap = n * world
    ctx = rafi.Context(B, cap, comm=comm, stream=torch.cuda.current_stream(), bootstrap=boot)
    ctx.set_option(rafi.OPT_EXCHANGE, exchange)
    assert ctx.get_option(rafi.OPT_EXCHANGE) == (exchange or rafi.EXCHANGE_FUSED)
    ctx.set_option(rafi.OPT_SCATTER, scatter)
    assert ctx.get_option(rafi.OPT_SCATTER) == (scatter or rafi.SCATTER_BULK)
    ctx.set_option(rafi.OPT_CONTROL, control)
    if control:
        assert ctx.get_option(rafi.OPT_CONTROL) == control
    assert ctx.num_ranks == world and ctx.rank_of(0) == rank
    for rnd in range(rounds):
        m = n if rnd % 2 == 0 else n // 3
        it = synth.make_items(rank, rnd, m, max(B, 16))[:, :B].copy()
        ds = synth.make_dests(pattern, 7 + rnd, rank, rnd, m, world, invalid_frac=0.01)
        ctx.emit_bulk(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), m)
        snap = ctx.read_outgoing(0)
        snaps = [None] * world
        dist.all_gather_object(snaps, snap)
        w = oracle.World(world, cap, B)
        for s, (items, dests, ctr, inv) in enumerate(snaps):
            w.load_snapshot(s, items, dests, ctr, inv)
        G_o = w.forward()
        G = ctx.forward_rc()
        assert G == G_o, (rank, G, G_o)
        assert np.array_equal(ctx.matrix(), w.C())
        st = ctx.stats()
        assert st["num_in"] == w.num_incoming(rank)
        if exchange in (rafi.EXCHANGE_NCCL, rafi.EXCHANGE_PEER):  # staged: the send batch is readable
            assert np.array_equal(ctx.read_binned(0, st["n_out"]), w.binned(rank, st["n_out"]))
        assert np.array_equal(ctx.read_incoming(0), w.incoming(rank))
    # termination: nothing emitted anywhere -> 0 on every rank
    assert ctx.forward() == 0
    ctx.close()
    if comm:
        rafi.nccl_comm_destroy(comm)
    dist.destroy_process_group()


@pytest.mark.parametrize("scatter", [1, 2])  # THREADS, BULK (TMA bulk stores, to NVLink peers)
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", [1, 2, 3])  # NCCL, PEER, FUSED
@pytest.mark.parametrize("B,pattern", [(48, "uniform"), (44, "skewed"), (16, "all_to_one")])
def test_multigpu_snapshot_parity(world, exchange, B, pattern, scatter):
    _need(world)
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), B, 30011, pattern, exchange, 3, scatter), nprocs=world, join=True)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("control", [1, 2, 3])  # NCCL collectives, PEER mailboxes over NVLink, HOST
@pytest.mark.parametrize("exchange", [3])  # FUSED
def test_multigpu_control_modes(world, control, exchange):
    """Count exchange + completion barrier through NCCL or through the peer
    mailboxes: same bytes, same G, several rounds (epochs) in a row."""
    _need(world)
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), 48, 20011, "skewed", exchange, 5, 1, control,
                                  "both" if control == 3 else "nccl"), nprocs=world,
             join=True)


@pytest.mark.parametrize("world", [2, 4])
def test_multigpu_large_default_path(world):
    """The bench's own configuration (AUTO: FUSED exchange, BULK pushes, peer
    control) at 2M x 48-B items per rank, two rounds: P1 bit-exact."""
    _need(world)
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), 48, 2 * 1024 * 1024, "uniform", 0, 2, 0, 0), nprocs=world,
             join=True)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", [2, 3])  # PEER (staged pull), FUSED
def test_multigpu_bootstrap_without_nccl(world, exchange):
    """rafi_create_boot with a gloo bootstrap and no NCCL communicator: CUDA-IPC
    handles travel through the host all-gather; AUTO control is PEER (mailboxes
    over NVLink) for FUSED, the host all-gather for the staged counts."""
    _need(world)
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), 44, 20011, "uniform", exchange, 3, 1, 0, "boot"), nprocs=world,
             join=True)


def _worker_hybrid(rank, world, port, L, B, n, graph, scatter=1):
    """P processes x L logical ranks each (R = P*L), FUSED exchange over
    local HBM and NVLink peer mappings; optionally the forward captured in a
    CUDA graph (NCCL collectives inside the capture, device-side G)."""
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2605_30294_b200 import rafi

    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", init_method=port, rank=rank, world_size=world)
    obj = [rafi.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = rafi.nccl_comm_init(world, rank, obj[0], rank)
    R = world * L
    cap = 2 * n
    s = torch.cuda.Stream()
    ctx = rafi.Context(B, cap, comm=comm, stream=s, local_ranks=L)
    assert ctx.num_ranks == R and ctx.get_option(rafi.OPT_EXCHANGE) == rafi.EXCHANGE_FUSED
    ctx.set_option(rafi.OPT_SCATTER, scatter)
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    ex = None
    for rnd in range(3):
        for l in range(L):
            g = rank * L + l
            it = synth.make_items(g, rnd, n, max(B, 16))[:, :B].copy()
            ds = synth.make_dests("uniform", 11 + rnd, g, rnd, n, R)
            ctx.emit_bulk(it, ds, n, local=l)
        snaps = []
        for l in range(L):
            snaps.append(ctx.read_outgoing(l))
        allsnaps = [None] * world
        dist.all_gather_object(allsnaps, snaps)
        w = oracle.World(R, cap, B)
        for p, sn in enumerate(allsnaps):
            for l, (items, dests, ctr, inv) in enumerate(sn):
                w.load_snapshot(p * L + l, items, dests, ctr, inv)
        G_o = w.forward()
        if graph:
            if ex is None:
                ctx.capture_begin()
                ctx.forward_async(G_dev)
                ex = ctx.capture_end()
            ctx.graph_launch(ex)
            s.synchronize()
            G = int(G_dev.item())
            ctx.sync_host()
        else:
            G = ctx.forward_rc()
        assert G == G_o, (rank, rnd, G, G_o)
        assert np.array_equal(ctx.matrix(), w.C())
        for l in range(L):
            assert np.array_equal(ctx.read_incoming(l), w.incoming(rank * L + l)), (rank, l)
    if ex is not None:
        rafi.Context.graph_destroy(ex)
    ctx.close()
    rafi.nccl_comm_destroy(comm)
    dist.destroy_process_group()


@pytest.mark.parametrize("scatter", [1, 2])
@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("world,L", [(2, 2), (2, 4), (4, 2)])
def test_multigpu_hybrid_local_ranks(world, L, graph, scatter):
    _need(world)
    import torch.multiprocessing as mp
    mp.spawn(_worker_hybrid, args=(world, _free_port(), L, 44, 20011, graph, scatter), nprocs=world,
             join=True)


@pytest.mark.parametrize("scatter", [1, 2])  # THREADS (warp tiles), BULK
def test_diag_redirect_to_peer_device(scatter):
    """One process, two GPUs: rank 1's incoming queue of a 2-rank context on
    cuda:0 is redirected to a buffer on cuda:1 (rafi_diag_redirect_incoming
    enables peer access), so the scatter pushes rank 1's block over NVLink
    -- the bytes that land on cuda:1 are exactly the oracle's incoming queue
    of rank 1, and rank 0's own queue is untouched."""
    from helpers import make_inputs, snapshot_world
    from paper_2605_30294_b200 import rafi
    B, L, n = 48, 2, 200003
    inputs = make_inputs(L, n, B, "uniform", 77)
    torch.cuda.set_device(0)
    with rafi.Context(B, L * n, local_ranks=L, device=0) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, scatter)
        buf = torch.zeros(L * n * B + 16, dtype=torch.uint8, device="cuda:1")
        ctx.diag_redirect_incoming(1, buf)
        for l, (it, ds) in enumerate(inputs):
            ctx.emit_bulk(torch.from_numpy(it).cuda(0), torch.from_numpy(ds).cuda(0), n, local=l)
        w, _ = snapshot_world(ctx, L, B)
        assert ctx.forward() == w.forward()
        m = ctx.num_incoming(1)
        assert m == w.num_incoming(1)
        torch.cuda.synchronize(1)
        assert np.array_equal(buf[: m * B].cpu().numpy().reshape(m, B), w.incoming(1))
        assert np.array_equal(ctx.read_incoming(0), w.incoming(0))
        ctx.diag_redirect_incoming(1, None)
