"""NEXT-3: device-side termination (rafi_forward_async) and CUDA-graph-captured
rounds, bit-exact against the oracle round by round."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2605_30294_b200 import rafi  # noqa: E402
from helpers import canonical  # noqa: E402


def _canon_id0(items):
    ids = items[:, 0:4].copy().view(np.uint32).ravel()
    return items[np.argsort(ids, kind="stable")]


def test_forward_async_equals_forward():
    L, n, B = 4, 5000, 48
    s = torch.cuda.Stream()
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    with torch.cuda.stream(s):
        with rafi.Context(B, 2 * n, local_ranks=L, stream=s) as ctx:
            w = oracle.World(L, 2 * n, B)
            for l in range(L):
                ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], 3, 0, n, local=l)
                w.emit_many(l, synth.make_items(l, 0, n, B), synth.make_dests("uniform", 3, l, 0, n, L))
            ctx.forward_async(G_dev)
            s.synchronize()
            assert int(G_dev.item()) == w.forward() == L * n
            ctx.sync_host()
            for l in range(L):
                assert ctx.num_incoming(l) == w.num_incoming(l)
                assert np.array_equal(canonical(ctx.read_incoming(l)), canonical(w.incoming(l)))


def test_forward_async_overflow_flag():
    B, cap = 16, 100
    s = torch.cuda.Stream()
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    with rafi.Context(B, cap, local_ranks=2, stream=s) as ctx:
        for l in range(2):
            ctx.emit_bulk(synth.make_items(l, 0, 60, B), np.ones(60, np.int32), local=l)
        ctx.forward_async(G_dev)
        s.synchronize()
        assert int(G_dev.item()) == -1            # ~0ull: nothing moved
        with pytest.raises(rafi.RafiError):
            ctx.sync_host()                      # collective overflow surfaces here
        assert ctx.forward_rc() == rafi.ERR_STATE


@pytest.mark.parametrize("R,n", [(8, 20000), (2, 10000)])
def test_graph_captured_advection_rounds(R, n):
    """One captured graph = app step (advect) + rafi_forward_async; replayed
    until the device-side G reaches 0; every round matches the oracle."""
    g = oracle.grid_dims(R)
    omega, eps, h, maxr = 2 * math.pi / 64, 1.0 / 64, 1.0, 10**6
    s = torch.cuda.Stream()
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    w = oracle.World(R, 2 * n, 16)
    with rafi.Context(16, 2 * n, local_ranks=R, stream=s) as ctx:
        for r in range(R):
            ctx.drv_advect_seed(n, 5, g, local=r)
            w.advect_seed(r, n, 5, g)
        assert ctx.forward() == w.forward()
        ctx.capture_begin()
        ctx.drv_advect_step(1, maxr, omega, eps, h, g)
        ctx.forward_async(G_dev)
        ex = ctx.capture_end()
        try:
            rounds = 0
            while True:
                ctx.graph_launch(ex)
                for r in range(R):
                    w.advect_step(r, 1, maxr, omega, eps, h, g)
                G_o = w.forward()
                s.synchronize()
                G = int(G_dev.item())
                assert G == G_o, (rounds, G, G_o)
                rounds += 1
                if rounds % 7 == 0 or G == 0:      # host refresh is optional between replays
                    ctx.sync_host()
                    for r in range(R):
                        assert np.array_equal(_canon_id0(ctx.read_incoming(r)), _canon_id0(w.incoming(r)))
                if G == 0:
                    break
            assert rounds > 10
        finally:
            rafi.Context.graph_destroy(ex)


@pytest.mark.parametrize("path", ["forward_async", "graph"])
def test_async_read_not_torn_by_a_later_forward(path):
    """rafi_read_incoming_async copies the incoming queue out on the copy-out
    stream; a forward enqueued right after it (rafi_forward_async, or a graph
    replay of one) rewrites that queue.  The library makes the context stream
    wait for the read first, so the host copy holds exactly the old round."""
    L, n, B, seed = 2, 4 * 1024 * 1024, 48, 91
    s = torch.cuda.Stream()
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    with rafi.Context(B, 2 * n, local_ranks=L, stream=s) as ctx:
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], seed, 0, n, local=l)
        assert ctx.forward() == L * n
        expect = [ctx.read_incoming(l) for l in range(L)]
        pins = [torch.empty((len(e), B), dtype=torch.uint8).pin_memory() for e in expect]
        ex = None
        if path == "graph":
            ctx.capture_begin()
            ctx.drv_random_walk(seed, 1, 5)
            ctx.forward_async(G_dev)
            ex = ctx.capture_end()
        for l in range(L):
            ctx.read_incoming_async(pins[l], local=l)
        if path == "graph":
            ctx.graph_launch(ex)
        else:
            ctx.drv_random_walk(seed, 1, 5)
            ctx.forward_async(G_dev)
        s.synchronize()
        ctx.read_wait()
        assert int(G_dev.item()) == L * n
        for l in range(L):
            assert np.array_equal(pins[l].numpy(), expect[l]), l
        ctx.sync_host()
        assert sum(ctx.num_incoming(l) for l in range(L)) == L * n
        if ex is not None:
            rafi.Context.graph_destroy(ex)


def test_capture_after_blocking_forward_covers_empty_rank():
    """A graph captured right after a blocking forward that left a local rank
    with no items must still contain that rank's app-step kernel (sized from
    the capacity, reading numIncoming on the device): later replays bring it
    items, and none may be dropped."""
    L, n, B, seed = 2, 3000, 32, 17
    s = torch.cuda.Stream()
    G_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    w = oracle.World(L, 2 * n * L, B)
    with rafi.Context(B, 2 * n * L, local_ranks=L, stream=s) as ctx:
        for l in range(L):  # everything to rank 0: rank 1 starts empty
            ctx.drv_emit_synthetic(synth.PATTERNS["all_to_one"], seed, 0, n, local=l, target=0)
            w.emit_many(l, synth.make_items(l, 0, n, B), synth.make_dests("all_to_one", seed, l, 0, n, L, target=0))
        assert ctx.forward() == w.forward() == L * n
        assert ctx.num_incoming(1) == 0
        ctx.capture_begin()
        ctx.drv_random_walk(seed, 1, 10 ** 6)
        ctx.forward_async(G_dev)
        ex = ctx.capture_end()
        try:
            for rnd in range(4):
                ctx.graph_launch(ex)
                for l in range(L):
                    inc = w.incoming(l).copy()
                    inc[:, 4:8] = np.frombuffer(np.uint32(1).tobytes(), np.uint8)
                    w.emit_many(l, inc, synth.walk_dests(seed, 1, synth.item_id_of(inc), L))
                G_o = w.forward()
                s.synchronize()
                assert int(G_dev.item()) == G_o == L * n, (rnd, int(G_dev.item()), G_o)
            ctx.sync_host()
            assert ctx.num_incoming(1) > 0
            for l in range(L):
                assert np.array_equal(canonical(ctx.read_incoming(l)), canonical(w.incoming(l)))
        finally:
            rafi.Context.graph_destroy(ex)
