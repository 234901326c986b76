"""Pins of the oracle's streaming-digest mode (oracle/digest.c, SURVEY §8(c)
P3) and of the snapshot / sequential-emit entry points every P1 and P2 test
routes through.  CPU only.

The digest mode is pinned against the MATERIALISED plain forward
(orc_forward_plain, itself pinned by SPEC's worked examples, closed forms and
brute force in test_oracle.py): same count matrix, same G, and the digest of
each materialised incoming queue equals the streamed digest.  Its
sensitivity is pinned too: a swapped pair, a flipped bit, a dropped or a
duplicated item all change the digest.
"""
import numpy as np
import pytest

import oracle
import synth

PATTERNS = ["uniform", "skewed", "ring", "all_to_one", "round_robin", "self"]


def _world(R, n, B, pattern, seed, cap, invalid_frac=0.0):
    w = oracle.World(R, cap, B)
    for s in range(R):
        it = synth.make_items(s, 0, n, max(B, 16))[:, :B].copy()
        ds = synth.make_dests(pattern, seed, s, 0, n, R, invalid_frac=invalid_frac)
        w.emit_many(s, it, ds)
    return w


def _stream(w, R, B, chunks):
    """Feed every source's queued items (slot order, sources ascending) in chunks."""
    g = oracle.Digest(R, w.cap, B)
    for s in range(R):
        items, dests = w.out_items(s), w.out_dests(s)
        cuts = [0] + sorted(chunks.integers(0, len(dests) + 1, 3).tolist()) + [len(dests)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            g.feed(s, items[a:b], dests[a:b])
    return g


@pytest.mark.parametrize("trial", range(24))
def test_digest_mode_equals_materialised_forward(trial):
    rng = np.random.default_rng(1000 + trial)
    R = int(rng.choice([1, 2, 3, 5, 8]))
    B = int(rng.choice([3, 16, 24, 44, 48, 64, 130]))
    n = int(rng.integers(0, 30000))
    pattern = str(rng.choice(PATTERNS))
    cap = max(1, int(n * rng.choice([0.7, 1.0, R])))  # some queues overflow (Z1 drops)
    w = _world(R, n, B, pattern, trial, cap, invalid_frac=float(rng.choice([0.0, 0.03])))
    g = _stream(w, R, B, rng)
    G = w.forward()
    assert g.finish() == G
    if G < 0:
        return  # Z3: both detect the receive overflow
    assert np.array_equal(g.C(), w.C())
    for d in range(R):
        assert g.value(d) == oracle.digest_items(w.incoming(d), B), d


def test_digest_mode_detects_receive_overflow():
    R, n, B = 3, 1000, 16
    w = _world(R, n, B, "all_to_one", 5, cap=2 * n)
    g = _stream(w, R, B, np.random.default_rng(0))
    assert g.finish() == w.forward() == oracle.ERR_RECV_OVERFLOW


def test_digest_self_pattern_closed_form():
    """Everything to self: in_r == out_r byte for byte, so the streamed digest
    equals the digest of the outgoing queue itself."""
    R, n, B = 4, 5000, 44
    w = _world(R, n, B, "self", 3, cap=n)
    outs = [w.out_items(s) for s in range(R)]
    g = _stream(w, R, B, np.random.default_rng(1))
    assert g.finish() == R * n
    for r in range(R):
        assert g.value(r) == oracle.digest_items(outs[r], B)


def test_digest_feed_order_and_bounds_enforced():
    g = oracle.Digest(2, 10, 16)
    it = synth.make_items(0, 0, 4, 16)
    g.feed(1, it, np.zeros(4, np.int32))
    with pytest.raises(ValueError):
        g.feed(0, it, np.zeros(4, np.int32))          # sources must ascend
    with pytest.raises(ValueError):
        g.feed(1, it, np.full(4, 2, np.int32))        # dest outside [0, R)
    with pytest.raises(ValueError):
        g.feed(1, synth.make_items(1, 0, 7, 16), np.zeros(7, np.int32))  # more than cap queued


@pytest.mark.parametrize("B", [1, 7, 8, 44, 64])
def test_digest_is_sensitive(B):
    rng = np.random.default_rng(B)
    items = rng.integers(0, 256, size=(50, B), dtype=np.uint8)
    base = oracle.digest_items(items, B)
    assert oracle.digest_items(items.copy(), B) == base
    seen = {base}
    sw = items.copy()
    sw[[10, 11]] = sw[[11, 10]]
    if not np.array_equal(sw, items):
        seen.add(oracle.digest_items(sw, B))
    for pos in range(B):                              # every byte position, one bit
        fl = items.copy()
        fl[17, pos] ^= 1 << (pos % 8)
        seen.add(oracle.digest_items(fl, B))
    seen.add(oracle.digest_items(np.delete(items, 30, axis=0), B))
    seen.add(oracle.digest_items(np.insert(items, 30, items[30], axis=0), B))
    expected = 1 + (0 if np.array_equal(sw, items) else 1) + B + 2
    assert len(seen) == expected


# ---- snapshot and sequential-emit entry points (orc_load_snapshot, orc_emit_many)

@pytest.mark.parametrize("R,n,B,cap", [(3, 700, 16, 1000), (2, 1200, 44, 1000), (4, 50, 8, 10)])
def test_load_snapshot_round_trip(R, n, B, cap):
    """Emit sequentially, read the queues back (items, dests, raw counters),
    load them into a fresh world: the two forwards are identical, output for
    output -- the P1 path's entry point reproduces the state it was given."""
    a = _world(R, n, B, "uniform", 9, cap, invalid_frac=0.05)
    b = oracle.World(R, cap, B)
    for s in range(R):
        b.load_snapshot(s, a.out_items(s), a.out_dests(s), a.emitted(s), a.invalid(s))
        assert b.emitted(s) == a.emitted(s) and b.invalid(s) == a.invalid(s)
    Ga, Gb = a.forward(), b.forward()
    assert Ga == Gb
    assert np.array_equal(a.C(), b.C())
    for r in range(R):
        assert np.array_equal(a.incoming(r), b.incoming(r))
        assert a.dropped_last(r) == b.dropped_last(r) and a.invalid_last(r) == b.invalid_last(r)


def test_load_snapshot_rejects_invalid_dest():
    w = oracle.World(2, 10, 16)
    with pytest.raises(ValueError):
        w.load_snapshot(0, synth.make_items(0, 0, 3, 16), np.array([0, 2, 1], np.int32), 3)


def test_emit_many_equals_single_emits():
    """orc_emit_many is n calls of orc_emit in array order:
    same queue, counters and return value (accepted count) as the loop."""
    R, n, B, cap = 3, 400, 20, 300
    it = synth.make_items(1, 0, n, 24)[:, :B].copy()
    ds = synth.make_dests("uniform", 4, 1, 0, n, R, invalid_frac=0.1)
    a, b = oracle.World(R, cap, B), oracle.World(R, cap, B)
    acc = a.emit_many(1, it, ds)
    acc_b = sum(b.emit(1, it[i].tobytes(), int(ds[i])) for i in range(n))
    assert acc == acc_b == min(cap, int(((ds >= 0) & (ds < R)).sum()))
    assert a.emitted(1) == b.emitted(1) and a.invalid(1) == b.invalid(1)
    assert np.array_equal(a.out_items(1), b.out_items(1)) and np.array_equal(a.out_dests(1), b.out_dests(1))
