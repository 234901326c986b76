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
