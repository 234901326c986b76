"""Shared test helpers: parity checks of the CUDA path against the oracle.

P1 (snapshot parity): read back the GPU's outgoing queue after emission (the
slot order the atomics chose), run the oracle's forward on exactly that
snapshot, and require every output -- count matrix, sender batches, incoming
queues, counters, G -- to be bit-identical in raw order.
P2 (canonical parity): the oracle emits sequentially in input order; the GPU
result must match after sorting each incoming queue by logical item id
(bytes 8..15), because the atomic append order is nondeterministic (Z17).
"""
import numpy as np

import oracle
import synth


def snapshot_world(ctx, L, B):
    w = oracle.World(L, ctx.capacity, B)
    snaps = []
    for l in range(L):
        items, dests, ctr, inv = ctx.read_outgoing(l)
        w.load_snapshot(l, items, dests, ctr, inv)
        snaps.append((items, dests, ctr, inv))
    return w, snaps


def p1_forward(ctx, L, B, check_binned=True):
    """One forward of a single-process context with L local ranks, checked
    bit-exactly against the oracle run on the GPU's own snapshot.  The send
    batch is compared too unless the FUSED exchange (which writes none) ran."""
    from paper_2605_30294_b200 import rafi
    if ctx.get_option(rafi.OPT_EXCHANGE) == rafi.EXCHANGE_FUSED:
        check_binned = False
    w, snaps = snapshot_world(ctx, L, B)
    G_o = w.forward()
    G_g = ctx.forward_rc()
    if G_o == oracle.ERR_RECV_OVERFLOW:   # Z3: both sides refuse the round (status codes differ by library)
        assert G_g == rafi.ERR_RECV_OVERFLOW, G_g
        return w, G_o
    assert G_g == G_o, (G_g, G_o)
    assert np.array_equal(ctx.matrix(), w.C())
    for l in range(L):
        st = ctx.stats(l)
        items, dests, ctr, inv = snaps[l]
        n = min(ctr, ctx.capacity)
        assert st["n_out"] == n and st["dropped"] == ctr - n and st["invalid"] == inv
        assert st["num_in"] == w.num_incoming(l) == ctx.num_incoming(l)
        if check_binned:
            assert np.array_equal(ctx.read_binned(l, n), w.binned(l, n)), "binned mismatch rank %d" % l
        assert np.array_equal(ctx.read_incoming(l), w.incoming(l)), "incoming mismatch rank %d" % l
    return w, G_o


def canonical(items):
    """Sort rows by logical id (bytes 8..15); ids are unique per item."""
    if len(items) == 0:
        return items
    ids = synth.item_id_of(items)
    return items[np.argsort(ids, kind="stable")]


def make_inputs(L, n, B, pattern, seed, rnd=0, invalid_frac=0.0, target=0):
    out = []
    for s in range(L):
        it = synth.make_items(s, rnd, n, max(B, 16))[:, :B].copy()
        ds = synth.make_dests(pattern, seed, s, rnd, n, L, invalid_frac=invalid_frac, target=target)
        out.append((it, ds))
    return out


def oracle_sequential(L, cap, B, inputs):
    w = oracle.World(L, cap, B)
    for s, (it, ds) in enumerate(inputs):
        w.emit_many(s, it, ds)
    return w
