"""Pins for the CPU oracle (oracle/): SPEC worked examples, closed forms,
brute force and the paper's invariants.  CPU only.

Each check pins the oracle to something other than itself:
  * SPEC.md's printed examples (tests/golden/spec_examples.json, cited);
  * closed forms (round-robin counts, self/ring/all-to-one exchanges);
  * exhaustive brute force on tiny inputs against Python's stable ``sorted``;
  * the two independent oracle pipelines (plain definition vs paper-literal)
    against each other;
  * invariants stated by the paper (conservation and exactly-once, PAPER:86;
    contiguity/stability of the sort; the reduce-add total,
    PAPER:136; the drop rule).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _item(ch, B=4):
    b = ch.encode() if isinstance(ch, str) else bytes(ch)
    return (b * B)[:B]


# ---------------------------------------------------------------- SPEC examples

@pytest.mark.parametrize("ex", GOLD["pack_keys"], ids=lambda e: e["cite"])
def test_spec_pack_keys(ex):
    got = oracle.pack_keys(ex["dests"])
    assert [int(k) for k in got] == [int(k, 16) for k in ex["keys"]]


@pytest.mark.parametrize("ex", GOLD["sort_and_gather"], ids=lambda e: e["cite"])
def test_spec_sort_and_gather(ex):
    B = 4
    items = np.array([list(_item(c, B)) for c in ex["items"]], np.uint8).reshape(-1, B)
    s, sd = oracle.sort_and_gather(items, ex["dests"], B)
    assert [bytes(r) for r in s] == [_item(c, B) for c in ex["sorted"]]
    assert list(sd) == ex["sorted_dests"]
    # the plain-definition forward bins the same way (rank 0 holding the batch)
    w = oracle.World(ex["R"], max(len(ex["dests"]), 1), B)
    for c, d in zip(ex["items"], ex["dests"]):
        assert w.emit(0, _item(c, B), d)
    w.forward()
    assert [bytes(r) for r in w.binned(0, len(ex["dests"]))] == [_item(c, B) for c in ex["sorted"]]


@pytest.mark.parametrize("ex", GOLD["compute_segments"], ids=lambda e: e["cite"])
def test_spec_compute_segments(ex):
    cnt, off = oracle.compute_segments(ex["sorted_dests"], ex["R"])
    assert list(map(int, cnt)) == ex["counts"]
    assert list(map(int, off)) == ex["offsets"]


@pytest.mark.parametrize("ex", GOLD["alltoall_counts"], ids=lambda e: e["cite"])
def test_spec_alltoall(ex):
    got = oracle.alltoall_u64(np.array(ex["send"], np.uint64))
    assert got.tolist() == ex["recv"]


@pytest.mark.parametrize("ex", GOLD["alltoallv_bytes"], ids=lambda e: e["cite"])
def test_spec_alltoallv(ex):
    R = len(ex["send"])
    sb = [np.frombuffer(s.encode(), np.uint8).copy() for s in ex["send"]]
    plan = np.array(ex["plan"], np.uint64)            # plan[s][d] = bytes s -> d
    sdispl = np.zeros((R, R), np.uint64)
    rdispl = np.zeros((R, R), np.uint64)
    for s in range(R):
        sdispl[s] = np.concatenate([[0], np.cumsum(plan[s])[:-1]])
    for d in range(R):
        rdispl[d] = np.concatenate([[0], np.cumsum(plan[:, d])[:-1]])
    rb = [np.zeros(len(r), np.uint8) for r in ex["recv"]]
    oracle.alltoallv_bytes(sb, plan, sdispl, rb, rdispl)
    assert [bytes(r).decode() for r in rb] == ex["recv"]


@pytest.mark.parametrize("ex", GOLD["emit"], ids=lambda e: e["cite"])
def test_spec_emit(ex):
    B = 4
    w = oracle.World(ex["R"], ex["cap"], B)
    if "emits" in ex:
        acc = [w.emit(0, _item(c, B), d) for c, d in ex["emits"]]
        assert acc == ex["accepted"]
        n = len(ex["slots"])
        assert [bytes(r) for r in w.out_items(0, n)] == [_item(c, B) for c, _ in ex["slots"]]
        assert list(w.out_dests(0, n)) == [d for _, d in ex["slots"]]
    else:
        for i in range(ex["n_emits"]):
            w.emit(0, _item(bytes([i]), B), 0)
    assert w.emitted(0) == ex["emitted"]
    w.forward()
    assert w.dropped_last(0) == ex["dropped"]


@pytest.mark.parametrize("ex", GOLD["forward"], ids=lambda e: e["cite"])
@pytest.mark.parametrize("literal", [False, True])
def test_spec_forward(ex, literal):
    B = 8
    w = oracle.World(ex["R"], 16, B)
    for k, (s, d) in enumerate(ex["emits"]):
        assert w.emit(s, _item(bytes([k + 1]), B), d)
    G = w.forward(literal=literal)
    assert G == ex["G"]
    assert [w.num_incoming(r) for r in range(ex["R"])] == ex["n_in"]


def test_spec_allreduce_sum():
    ex = GOLD["allreduce_sum"][0]
    R = len(ex["locals"])
    w = oracle.World(R, 8, 4)
    for d, c in enumerate(ex["locals"]):   # rank d receives ex.locals[d] items
        for k in range(c):
            w.emit((d + k) % R, _item(bytes([k]), 4), d)
    assert w.forward() == ex["sum"]
    assert [w.num_incoming(r) for r in range(R)] == ex["locals"]


# ---------------------------------------------------------------- emit rules

def test_invalid_dest_rejected_and_counted():
    w = oracle.World(3, 4, 4)
    assert not w.emit(0, b"aaaa", -1)
    assert not w.emit(0, b"bbbb", 3)
    assert w.emit(0, b"cccc", 2)
    assert w.emitted(0) == 1 and w.invalid(0) == 2
    assert list(w.out_dests(0)) == [2]
    w.forward()
    assert w.invalid_last(0) == 2 and w.dropped_last(0) == 0
    assert w.invalid(0) == 0 and w.emitted(0) == 0       # wrap-up resets
    assert w.incoming(2)[0].tobytes() == b"cccc"


def test_drop_accounting_invariant():
    rng = np.random.default_rng(1)
    for _ in range(20):
        R, cap = int(rng.integers(1, 5)), int(rng.integers(0, 12))
        w = oracle.World(R, cap, 4)
        attempts_valid = [0] * R
        for _ in range(int(rng.integers(0, 30))):
            s, d = int(rng.integers(0, R)), int(rng.integers(-1, R + 1))
            w.emit(s, b"xxxx", d)
            attempts_valid[s] += 0 <= d < R
        rc = w.forward()
        if rc == oracle.ERR_RECV_OVERFLOW:
            continue
        for s in range(R):  # accepted + dropped = valid attempts
            assert int(w.C()[s].sum()) + w.dropped_last(s) == attempts_valid[s]
            assert int(w.C()[s].sum()) == min(attempts_valid[s], cap)


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("R,N", [(1, 7), (2, 9), (3, 10), (4, 4), (5, 23), (8, 100)])
def test_round_robin_closed_form(R, N):
    B = 16
    w = oracle.World(R, N, B)
    items = synth.make_items(0, 0, N, B)
    for i in range(N):
        w.emit(0, items[i].tobytes(), i % R)
    w.forward()
    C = w.C()
    for d in range(R):
        assert C[0, d] == -(-(N - d) // R)          # ceil((N-d)/R)
    perm = [i for d in range(R) for i in range(d, N, R)]   # stride permutation
    assert np.array_equal(w.binned(0, N), items[perm])


def _emit_pattern(w, R, n, B, pattern, seed=7, target=0):
    outs = []
    for s in range(R):
        it = synth.make_items(s, 0, n, B)
        ds = synth.make_dests(pattern, seed, s, 0, n, R, target=target)
        for i in range(n):
            w.emit(s, it[i].tobytes(), int(ds[i]))
        outs.append(it)
    return outs


@pytest.mark.parametrize("literal", [False, True])
@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_self_ring_all_to_one_closed_forms(R, literal):
    B, n = 24, 13
    w = oracle.World(R, n * R, B)
    outs = _emit_pattern(w, R, n, B, "self")
    assert w.forward(literal) == R * n
    for r in range(R):
        assert np.array_equal(w.incoming(r), outs[r])     # in_r == out_r
    outs = _emit_pattern(w, R, n, B, "ring")
    w.forward(literal)
    for d in range(R):
        assert np.array_equal(w.incoming(d), outs[(d - 1) % R])   # in_d == out_{d-1}
    outs = _emit_pattern(w, R, n, B, "all_to_one", target=0)
    assert w.forward(literal) == R * n
    assert np.array_equal(w.incoming(0), np.concatenate(outs))  # out_0 || out_1 || ...
    for d in range(1, R):
        assert w.num_incoming(d) == 0


# ---------------------------------------------------------------- brute force

def _expected(R, B, per_rank):
    """Python-only statement of the result: stable sort by dest per source
    (Python's sorted() is stable), then per destination concatenate sources
    in rank order."""
    binned, C = [], np.zeros((R, R), np.uint64)
    for s, (items, dests) in enumerate(per_rank):
        order = sorted(range(len(dests)), key=lambda i: dests[i])
        binned.append([items[i] for i in order])
        for d in dests:
            C[s, d] += 1
    incoming = []
    for d in range(R):
        inc = []
        for s, (items, dests) in enumerate(per_rank):
            inc += [items[i] for i in range(len(dests)) if dests[i] == d]
        incoming.append(inc)
    return binned, C, incoming


@pytest.mark.parametrize("R,Nmax", [(2, 10), (3, 6), (4, 5)])
def test_exhaustive_brute_force(R, Nmax):
    """Every dest vector in R^N on rank 0 (N <= Nmax); a fixed small batch on
    the other ranks; plain == literal == Python statement."""
    B = 4
    others = [[(bytes([100 + s, k, 0, 0]), (s + k) % R) for k in range(2)] for s in range(1, R)]
    for N in range(Nmax + 1):
        for dv in itertools.product(range(R), repeat=N):
            items0 = [bytes([0, k, 1, 2]) for k in range(N)]
            per_rank = [(items0, list(dv))] + [([i for i, _ in o], [d for _, d in o]) for o in others]
            exp_binned, exp_C, exp_in = _expected(R, B, per_rank)
            for literal in (False, True):
                w = oracle.World(R, 16, B)
                for s, (its, ds) in enumerate(per_rank):
                    for it, d in zip(its, ds):
                        w.emit(s, it, d)
                G = w.forward(literal)
                assert G == sum(len(p[1]) for p in per_rank)
                assert np.array_equal(w.C(), exp_C)
                for s in range(R):
                    assert [bytes(r) for r in w.binned(s, len(per_rank[s][1]))] == exp_binned[s]
                for d in range(R):
                    assert [bytes(r) for r in w.incoming(d)] == exp_in[d]
                w.close()


# ---------------------------------------------------------------- invariants

def _check_invariants(w, R, B, emitted_by_src):
    """Paper invariants after one forward, given what each source emitted
    (list of (item bytes, dest) in slot order, accepted only)."""
    C, so, ro = w.C(), w.send_off(), w.recv_off()
    G = w.G()
    # row sums = accepted emits; column sums = n_in; total = G
    for s in range(R):
        assert int(C[s].sum()) == len(emitted_by_src[s])
        assert list(so[s]) == list(np.concatenate([[0], np.cumsum(C[s])[:-1]]).astype(np.uint64))
    for d in range(R):
        assert int(C[:, d].sum()) == w.num_incoming(d)
        assert list(ro[d]) == list(np.concatenate([[0], np.cumsum(C[:, d])[:-1]]).astype(np.uint64))
    assert G == int(C.sum())
    # contiguity + stability of the sender's sort
    for s in range(R):
        b = w.binned(s, len(emitted_by_src[s]))
        for d in range(R):
            seg = b[int(so[s, d]): int(so[s, d] + C[s, d])]
            exp = [it for it, dd in emitted_by_src[s] if dd == d]
            assert [bytes(r) for r in seg] == exp
    # exactly-once delivery to the named rank, source-major (Z5)
    for d in range(R):
        inc = w.incoming(d)
        for s in range(R):
            seg = inc[int(ro[d, s]): int(ro[d, s] + C[s, d])]
            exp = [it for it, dd in emitted_by_src[s] if dd == d]
            assert [bytes(r) for r in seg] == exp


@pytest.mark.parametrize("trial", range(60))
def test_randomized_plain_vs_literal(trial):
    rng = np.random.default_rng(1000 + trial)
    R = int(rng.integers(1, 9))
    B = int(rng.choice([1, 3, 4, 8, 12, 16, 24, 44, 48, 64, 128]))
    n = int(rng.integers(0, 400))
    cap = int(n * R) + 1
    pattern = str(rng.choice(["uniform", "skewed", "ring", "round_robin", "self", "all_to_one"]))
    worlds = [oracle.World(R, cap, B) for _ in range(2)]
    emitted = [[] for _ in range(R)]
    for s in range(R):
        its = synth.make_items(s, trial, n, max(B, 16))[:, :B]
        ds = synth.make_dests(pattern, 99 + trial, s, 0, n, R, invalid_frac=0.05)
        for i in range(n):
            for w in worlds:
                w.emit(s, its[i].tobytes(), int(ds[i]))
            if 0 <= ds[i] < R:
                emitted[s].append((its[i].tobytes(), int(ds[i])))
    G0 = worlds[0].forward(literal=False)
    G1 = worlds[1].forward(literal=True)
    assert G0 == G1 == sum(len(e) for e in emitted)
    a, b = worlds
    assert np.array_equal(a.C(), b.C()) and np.array_equal(a.send_off(), b.send_off())
    assert np.array_equal(a.recv_off(), b.recv_off())
    for r in range(R):
        assert np.array_equal(a.incoming(r), b.incoming(r))
        assert np.array_equal(a.binned(r, len(emitted[r])), b.binned(r, len(emitted[r])))
        assert a.invalid_last(r) == b.invalid_last(r)
    _check_invariants(a, R, B, emitted)


def test_receive_overflow_state_unchanged():
    """Z3: a rank that would receive more than its capacity fails the forward
    on every rank, before any payload moves."""
    for literal in (False, True):
        w = oracle.World(2, 3, 4)
        for k in range(3):
            w.emit(0, bytes([k] * 4), 1)
            w.emit(1, bytes([9, k, 0, 0]), 1)
        w.set_incoming(1, np.zeros(4, np.uint8))
        assert w.forward(literal) == oracle.ERR_RECV_OVERFLOW
        assert w.emitted(0) == 3 and w.emitted(1) == 3       # queues untouched
        assert w.num_incoming(1) == 1


# ---------------------------------------------------------------- termination

def _run_rounds(w, R, step, max_rounds=100):
    """host loop: do { step; G = forward } while (G > 0)."""
    rounds = 0
    while True:
        for r in range(R):
            step(r, rounds)
        G = w.forward()
        rounds += 1
        if G == 0 or rounds >= max_rounds:
            return rounds, G


@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_ring_walk_rounds(R):
    """items seeded with R hops, each forwarded to (rank+1) mod R
    once per round and retired after R hops -> exactly R item-carrying rounds
    (+1 terminating forward that returns 0), identical on all ranks."""
    B = 16
    w = oracle.World(R, 8, B)
    for s in range(R):
        hdr = np.zeros(B, np.uint8)
        hdr[0] = R  # hops left
        hdr[1] = s  # origin
        w.set_incoming(s, hdr)
    carrying = []

    def step(r, k):
        for i in range(w.num_incoming(r)):
            it = bytearray(w.incoming(r)[i].tobytes())
            if it[0] > 0:
                it[0] -= 1
                w.emit(r, bytes(it), (r + 1) % R)

    rounds = 0
    while True:
        for r in range(R):
            step(r, rounds)
        G = w.forward()
        rounds += 1
        carrying.append(G)
        if G == 0:
            break
    assert rounds == R + 1 and carrying[:R] == [R] * R and carrying[R] == 0
    # after R hops every item is back at its origin: no premature exit of any rank


# ---------------------------------------------------------------- emit_many / load_snapshot / set_incoming

@pytest.mark.parametrize("cap", [0, 1, 7, 64, 500])
def test_emit_many_is_the_drop_rule(cap):
    """orc_emit_many against the drop and reject rules written out (Z1, Z2,
    PAPER:71): the queue holds exactly the first min(cap, #valid) valid
    (item, dest) pairs in array order, the counter counts every valid
    attempt, the reject counter every invalid one -- and a world fed by
    single orc_emit calls ends in the same state and forwards alike."""
    rng = np.random.default_rng(cap + 3)
    R, B, n = 3, 12, 300
    items = rng.integers(0, 256, (n, B), dtype=np.uint8)
    dests = rng.integers(-2, R + 2, n).astype(np.int32)
    valid = [i for i in range(n) if 0 <= dests[i] < R]
    kept = valid[:cap]
    a, b = oracle.World(R, cap, B), oracle.World(R, cap, B)
    assert a.emit_many(1, items, dests) == len(kept)
    for i in range(n):
        b.emit(1, items[i].tobytes(), int(dests[i]))
    for w in (a, b):
        assert w.emitted(1) == len(valid) and w.invalid(1) == n - len(valid)
        assert np.array_equal(w.out_items(1), items[kept].reshape(len(kept), B))
        assert np.array_equal(w.out_dests(1), dests[kept])
    ga, gb = a.forward(), b.forward()
    if ga == oracle.ERR_RECV_OVERFLOW:
        assert gb == ga
        return
    assert ga == gb == len(kept)
    for r in range(R):
        assert np.array_equal(a.incoming(r), b.incoming(r))
        assert np.array_equal(a.incoming(r), items[[i for i in kept if dests[i] == r]].reshape(-1, B))


@pytest.mark.parametrize("literal", [False, True])
def test_load_snapshot_round_trip(literal):
    """A queue state read back from one world (items in slot order, dests,
    raw counters) and loaded into a fresh world with orc_load_snapshot
    forwards to the same incoming queues, count matrix and G -- including an
    over-capacity counter (only cap items are loaded, the rest count as
    dropped) -- and a snapshot with an out-of-range dest is refused."""
    rng = np.random.default_rng(9)
    R, cap, B = 4, 50, 20
    src = oracle.World(R, cap, B)
    for s in range(R):
        n = int(rng.integers(0, 70))
        src.emit_many(s, rng.integers(0, 256, (n, B), dtype=np.uint8), rng.integers(-1, R + 1, n).astype(np.int32))
    dst = oracle.World(R, cap, B)
    for s in range(R):
        dst.load_snapshot(s, src.out_items(s), src.out_dests(s), src.emitted(s), src.invalid(s))
        assert dst.emitted(s) == src.emitted(s) and dst.invalid(s) == src.invalid(s)
    g1, g2 = src.forward(literal=literal), dst.forward(literal=literal)
    assert g1 == g2
    if g1 == oracle.ERR_RECV_OVERFLOW:
        return
    assert np.array_equal(src.C(), dst.C())
    for r in range(R):
        assert np.array_equal(src.incoming(r), dst.incoming(r))
        assert dst.dropped_last(r) == src.dropped_last(r)
    bad = oracle.World(2, 4, 4)
    with pytest.raises(ValueError):
        bad.load_snapshot(0, np.zeros((2, 4), np.uint8), np.array([0, 2], np.int32), 2, 0)


def test_set_incoming_is_what_get_incoming_reads():
    """orc_set_incoming seeds a rank's input queue: numIncoming and
    getIncoming read back exactly the seeded items; more than
    capacity is refused; a forward replaces the queue (Z12)."""
    w = oracle.World(2, 8, 6)
    seed = np.arange(5 * 6, dtype=np.uint8).reshape(5, 6)
    w.set_incoming(1, seed)
    assert w.num_incoming(1) == 5 and np.array_equal(w.incoming(1), seed)
    with pytest.raises(ValueError):
        w.set_incoming(0, np.zeros((9, 6), np.uint8))
    assert w.emit(0, b"abcdef", 1)
    assert w.forward() == 1
    assert w.num_incoming(1) == 1 and w.incoming(1)[0].tobytes() == b"abcdef"
