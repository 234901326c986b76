"""Full-size R=8 parity on one GPU (BASELINE configs[1] and configs[4]).

The whole 8-rank world of cfg2 (8 x 16,777,216 x 48-B items, uniform) and of
cfg5 (8 x 33,554,432 items at 64 B and at the paper's 44 B, uniform
all-to-all) runs as 8 logical ranks of one context on one B200 -- the same
kernels, launch configuration and FUSED exchange the bench times, the ranks'
incoming queues being local HBM instead of NVLink peers.

Check (P1 semantics through the oracle's streaming-digest mode, P3): after
the device-side emission (rafi::Queue<T>::emitOutgoing, warp-aggregated
atomics), every rank's outgoing queue is read back once, in ascending rank
order, and fed to oracle.Digest -- which digests each destination's incoming
queue as the plain definition builds it (sources ascending, slot order) and
counts the R x R matrix exactly, without materialising 19-60 GiB of state.
Then the GPU forwards; its count matrix and G must equal the oracle's
exactly, and the digest of each incoming queue read back from the GPU must
equal the oracle's digest.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2605_30294_b200 import rafi  # noqa: E402

SCATTERS = {"threads": rafi.SCATTER_THREADS, "bulk": rafi.SCATTER_BULK}


def _full_world(L, n, B, seed, scatter, pattern="uniform"):
    cap = n + n // 8
    with rafi.Context(B, cap, local_ranks=L) as ctx:
        if scatter != "auto":
            ctx.set_option(rafi.OPT_SCATTER, SCATTERS[scatter])
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS[pattern], seed, 0, n, local=l)
        dg = oracle.Digest(L, cap, B)
        for s in range(L):                       # sources ascending, each queue in slot order
            items, dests, ctr, inv = ctx.read_outgoing(s)
            assert ctr == n and inv == 0 and len(dests) == n
            dg.feed(s, items, dests)
            del items, dests
        G_o = dg.finish()
        G = ctx.forward()
        assert G == G_o == L * n
        assert np.array_equal(ctx.matrix(), dg.C())
        for d in range(L):
            st = ctx.stats(d)
            assert st["n_out"] == n and st["dropped"] == 0 and st["num_in"] == int(dg.C()[:, d].sum())
            got = ctx.read_incoming(d)
            assert oracle.digest_items(got, B) == dg.value(d), "incoming queue %d differs" % d
            del got
        dg.close()


@pytest.mark.parametrize("scatter", ["threads", "bulk"])
def test_cfg2_full_world_r8(scatter):
    """cfg2: 8 ranks x 16M x 48-B items, uniform destinations, one round."""
    _full_world(8, 16 * 1024 * 1024, 48, synth.CONFIG_SEEDS[2], scatter)


@pytest.mark.parametrize("B,scatter", [(64, "threads"), (44, "threads"), (44, "bulk")])
def test_cfg5_full_world_r8(B, scatter):
    """cfg5: 8 ranks x 32M items, uniform all-to-all, at the headline 64 B
    and the paper's 44-B payload (4-byte units: the 16-B chunk gather and
    the bulk-store path)."""
    _full_world(8, 32 * 1024 * 1024, B, synth.CONFIG_SEEDS[5], scatter)


@pytest.mark.parametrize("B", [16, 128])
def test_cfg5_sweep_ends_full_world_r8(B):
    """The ends of cfg5's 16-128 B item-size sweep at full size."""
    _full_world(8, 32 * 1024 * 1024, B, synth.CONFIG_SEEDS[5], "auto")
