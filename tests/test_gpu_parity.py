"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Single-process cases, including R logical ranks hosted on one GPU
(local_ranks = R), which run the same kernels and the PEER copy path with
local pointers.  Every comparison is bit-exact (integer/byte work).
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import canonical, make_inputs, oracle_sequential, p1_forward, snapshot_world

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2605_30294_b200 import rafi  # noqa: E402


def _ctx(B, cap, L=1, **kw):
    return rafi.Context(B, cap, local_ranks=L, **kw)


def _emit_all(ctx, inputs, device=True):
    for l, (it, ds) in enumerate(inputs):
        if device:
            ctx.emit_bulk(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), len(ds), local=l)
        else:
            ctx.emit_bulk(it, ds, len(ds), local=l)


# ------------------------------------------------------------------ emission

@pytest.mark.parametrize("B", [3, 4, 16, 44, 48, 128, 520])
@pytest.mark.parametrize("device", [True, False])
def test_emit_bulk_queue_contents(B, device):
    n, L = 10007, 3
    inputs = make_inputs(L, n, B, "uniform", 11, invalid_frac=0.03)
    with _ctx(B, 2 * n, L) as ctx:
        _emit_all(ctx, inputs, device)
        for l, (it, ds) in enumerate(inputs):
            items, dests, ctr, inv = ctx.read_outgoing(l)
            ok = (ds >= 0) & (ds < L)
            assert ctr == ok.sum() and inv == (~ok).sum()
            # the queue holds exactly the accepted (item, dest) pairs (a permutation of 2048-blocks)
            got = np.concatenate([items, dests.view(np.uint8).reshape(-1, 4)], axis=1)
            exp = np.concatenate([it[ok], ds[ok].view(np.uint8).reshape(-1, 4)], axis=1)
            gv = np.sort(got.view(np.dtype((np.void, got.shape[1]))).ravel())
            ev = np.sort(exp.view(np.dtype((np.void, exp.shape[1]))).ravel())
            assert np.array_equal(gv, ev)


def test_emit_drop_rule():
    """Z1: capacity 5000, 3 bulk emits of 2000 -> ctr 6000, 5000 stored, 1000 dropped."""
    B = 16
    with _ctx(B, 5000, 1) as ctx:
        for k in range(3):
            it = synth.make_items(0, 0, 2000, B, seq0=2000 * k)
            ctx.emit_bulk(it, np.zeros(2000, np.int32))
        items, dests, ctr, inv = ctx.read_outgoing(0)
        assert ctr == 6000 and len(items) == 5000
        w, G = p1_forward(ctx, 1, B)
        assert G == 5000 and ctx.stats()["dropped"] == 1000


# ------------------------------------------------------------------ forward, P1

CASES = [
    # (B, L, n per rank, pattern)
    (4, 1, 5000, "uniform"), (16, 1, 0, "uniform"), (48, 1, 100000, "uniform"),
    (8, 2, 7777, "uniform"), (12, 3, 4099, "skewed"), (16, 2, 4096, "ring"),
    (24, 4, 20001, "uniform"), (32, 2, 4096, "uniform"), (40, 5, 3333, "round_robin"),
    (44, 4, 50000, "uniform"), (48, 8, 30000, "uniform"), (64, 8, 12345, "skewed"),
    (96, 3, 9000, "all_to_one"), (128, 4, 7000, "uniform"), (3, 2, 6000, "uniform"),
    (20, 7, 5001, "uniform"), (520, 3, 2000, "uniform"), (200, 2, 3000, "self"),
    (32, 20, 2000, "skewed"), (16, 40, 1000, "uniform"), (8, 64, 700, "round_robin"),
]


EXCHANGES = {"fused": 3, "peer": 2}
SCATTERS = {"threads": rafi.SCATTER_THREADS, "bulk": rafi.SCATTER_BULK}


def _bulk_ok(B):
    """BULK needs item_bytes % 4 == 0 and a 256-item tile in shared memory
    (test_bulk_unsupported checks that it is refused otherwise)."""
    return B % 4 == 0 and B <= 256


@pytest.mark.parametrize("scatter,exchange,B,L,n,pattern",
                         [(sc, ex) + case for sc in sorted(SCATTERS) for ex in sorted(EXCHANGES) for case in CASES
                          if sc == "threads" or _bulk_ok(case[0])])
def test_forward_snapshot_parity(B, L, n, pattern, exchange, scatter):
    inputs = make_inputs(L, n, B, pattern, 1234 + B, invalid_frac=0.01)
    cap = max(n * L, 1)
    with _ctx(B, cap, L) as ctx:
        ctx.set_option(rafi.OPT_EXCHANGE, EXCHANGES[exchange])
        ctx.set_option(rafi.OPT_SCATTER, SCATTERS[scatter])
        assert ctx.get_option(rafi.OPT_SCATTER) == SCATTERS[scatter]
        _emit_all(ctx, inputs)
        p1_forward(ctx, L, B)
        # a second round on the same context (counters reset, buffers reused)
        inputs2 = make_inputs(L, n // 2, B, pattern, 99 + B, rnd=1)
        _emit_all(ctx, inputs2)
        p1_forward(ctx, L, B)


@pytest.mark.parametrize("tile", [128, 256, 512, 1024, 4096])
@pytest.mark.parametrize("B", [4, 12, 20, 24, 44, 48, 64, 128])
def test_tile_sizes(tile, B):
    """Every tile on every path: 128/256 are the warp-tile kernels at R <= 8
    (16-byte units, or the 16-byte chunk gather at 4, 12, 20, 24 and 44 B,
    where a chunk spans up to four items), larger tiles the block-tile ones."""
    L, n = 4, 20011
    inputs = make_inputs(L, n, B, "uniform", 5 + B)
    with _ctx(B, n * L, L) as ctx:
        ctx.set_option(rafi.OPT_TILE, tile)
        assert ctx.get_option(rafi.OPT_TILE) == tile
        _emit_all(ctx, inputs)
        p1_forward(ctx, L, B)


def test_tile_128_needs_the_warp_tile_path():
    """RAFI_OPT_TILE 128 exists only on the warp-tile path (THREADS, R <= 8,
    item_bytes % 4 == 0)."""
    with _ctx(42, 1000, 2) as ctx:          # 2-byte units: block tiles only
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_TILE, 128)
    with _ctx(48, 1000, 9) as ctx:          # R = 9
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_TILE, 128)
    with _ctx(48, 1000, 2) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, rafi.SCATTER_BULK)
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_TILE, 128)


@pytest.mark.parametrize("B,tile", [(16, 256), (16, 1024), (16, 2048), (48, 256), (48, 512), (44, 1024),
                                    (128, 256), (4, 4096), (36, 512), (256, 256), (200, 256), (64, 1024)])
@pytest.mark.parametrize("mode", ["bulk"])
def test_perm_tile_sizes(B, tile, mode):
    """The permuting (TMA bulk-store) scatter at every tile that fits, ragged
    last tiles and runs whose global start is not 16-byte aligned (B % 16 != 0)."""
    L, n = 4, 20011
    inputs = make_inputs(L, n, B, "uniform", 6 + B)
    with _ctx(B, n * L, L) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, SCATTERS[mode])
        ctx.set_option(rafi.OPT_TILE, tile)
        _emit_all(ctx, inputs)
        p1_forward(ctx, L, B)


def test_bulk_unsupported():
    """BULK is refused (not silently replaced) where it cannot run."""
    with _ctx(6, 1000, 1) as ctx:
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_SCATTER, rafi.SCATTER_BULK)
        assert ctx.get_option(rafi.OPT_SCATTER) == rafi.SCATTER_THREADS
    with _ctx(520, 1000, 1) as ctx:
        with pytest.raises(rafi.RafiError):  # 2 stages + 1 output tile of 256 x 520 B > 227 KiB
            ctx.set_option(rafi.OPT_SCATTER, rafi.SCATTER_BULK)
    with _ctx(48, 100000, 1) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, rafi.SCATTER_BULK)
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_TILE, 4096)  # 2 stages + 1 output tile of 4096 x 48 B > 227 KiB


@pytest.mark.parametrize("B,L,n,pattern", [(16, 1, 3000, "uniform"), (32, 2, 4096, "uniform"),
                                           (48, 4, 5000, "skewed"), (44, 3, 2500, "all_to_one"),
                                           (64, 8, 1500, "uniform")])
def test_forward_canonical_parity(B, L, n, pattern):
    """P2: GPU result == sequential oracle after canonical ordering by id."""
    inputs = make_inputs(L, n, B, pattern, 77, invalid_frac=0.02)
    cap = n * L
    w = oracle_sequential(L, cap, B, inputs)
    G_o = w.forward()
    with _ctx(B, cap, L) as ctx:
        _emit_all(ctx, inputs)
        assert ctx.forward() == G_o
        assert np.array_equal(ctx.matrix(), w.C())
        for l in range(L):
            assert np.array_equal(canonical(ctx.read_incoming(l)), canonical(w.incoming(l)))
            assert ctx.stats(l)["invalid"] == w.invalid_last(l)


# ------------------------------------------------------------------ edge cases

def test_default_exchange_is_fused_and_nccl_single_rank():
    with _ctx(16, 1000, 1) as ctx:
        assert ctx.get_option(rafi.OPT_EXCHANGE) == rafi.EXCHANGE_FUSED
        ctx.set_option(rafi.OPT_EXCHANGE, rafi.EXCHANGE_NCCL)   # R=1: the self run is a local copy
        ctx.emit_bulk(synth.make_items(0, 0, 777, 16), np.zeros(777, np.int32))
        p1_forward(ctx, 1, 16)
    with _ctx(16, 1000, 2) as ctx:   # NCCL staging needs one local rank per process
        with pytest.raises(rafi.RafiError):
            ctx.set_option(rafi.OPT_EXCHANGE, rafi.EXCHANGE_NCCL)


def test_empty_forward_is_termination():
    with _ctx(32, 100, 3) as ctx:
        assert ctx.forward() == 0
        assert all(ctx.num_incoming(l) == 0 for l in range(3))
        assert ctx.forward() == 0


def test_receive_overflow_collective_and_state_unchanged():
    B, cap = 16, 100
    with _ctx(B, cap, 2) as ctx:
        for l in range(2):
            ctx.emit_bulk(synth.make_items(l, 0, 60, B), np.ones(60, np.int32), local=l)
        assert ctx.forward_rc() == rafi.ERR_RECV_OVERFLOW
        for l in range(2):
            _, _, ctr, _ = ctx.read_outgoing(l)
            assert ctr == 60 and ctx.num_incoming(l) == 0
        assert ctx.forward_rc() == rafi.ERR_STATE


def test_exact_capacity_receive():
    B, cap = 16, 128
    with _ctx(B, cap, 2) as ctx:
        for l in range(2):
            ctx.emit_bulk(synth.make_items(l, 0, 64, B), np.ones(64, np.int32), local=l)
        p1_forward(ctx, 2, B)
        assert ctx.num_incoming(1) == 128


def test_device_view_and_resize():
    B = 32
    with _ctx(B, 1000, 2) as ctx:
        v = ctx.device_view(1)
        assert v.capacity == 1000 and v.item_bytes == B and v.num_ranks == 2 and v.my_rank == 1
        inputs = make_inputs(2, 700, B, "uniform", 3)
        _emit_all(ctx, inputs)
        w, _ = p1_forward(ctx, 2, B)
        before = [ctx.read_incoming(l) for l in range(2)]
        ctx.resize(5000)
        assert ctx.capacity == 5000
        for l in range(2):
            assert np.array_equal(ctx.read_incoming(l), before[l])
        inputs = make_inputs(2, 2400, B, "uniform", 4, rnd=1)
        _emit_all(ctx, inputs)
        p1_forward(ctx, 2, B)


# ------------------------------------------------------------------ device-side emit

@pytest.mark.parametrize("B", [16, 32, 44, 48, 64, 128])
@pytest.mark.parametrize("pattern", ["uniform", "skewed", "round_robin"])
def test_device_emit_matches_generator(B, pattern):
    """rafi::Queue<T>::emitOutgoing (warp-aggregated) from the proxy emitter:
    the queue holds exactly synth's items/dests (the generator's two
    implementations agree), invalid dests rejected and counted."""
    L, n, seed = 3, 9001, 42
    thr = synth.invalid_threshold(0.02)
    with _ctx(B, 2 * n, L) as ctx:
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS[pattern], seed, 5, n, local=l, invalid_threshold=thr)
        for l in range(L):
            items, dests, ctr, inv = ctx.read_outgoing(l)
            exp_it = synth.make_items(l, 5, n, B)
            exp_d = synth.make_dests(pattern, seed, l, 5, n, L, invalid_frac=0.02)
            ok = (exp_d >= 0) & (exp_d < L)
            assert ctr == ok.sum() and inv == (~ok).sum()
            order = np.argsort(synth.item_id_of(items))
            assert np.array_equal(items[order], exp_it[ok])
            assert np.array_equal(dests[order], exp_d[ok])
        p1_forward(ctx, L, B)


def test_random_walk_cfg1_shape():
    """cfg1 (BASELINE configs[0]): 2 ranks, 4096 x 32-B items each, uniform
    destinations, 3 forwarding rounds, then termination; canonical parity of
    every round against the sequential oracle."""
    L, n, B, seed = 2, 4096, 32, synth.CONFIG_SEEDS[1]
    w = oracle.World(L, n * L, B)
    with _ctx(B, n * L, L) as ctx:
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], seed, 0, n, local=l)
            w.emit_many(l, synth.make_items(l, 0, n, B), synth.make_dests("uniform", seed, l, 0, n, L))
        Gs = []
        for k in range(1, 5):
            G = ctx.forward()
            assert G == w.forward()
            Gs.append(G)
            for l in range(L):
                assert np.array_equal(canonical(ctx.read_incoming(l)), canonical(w.incoming(l)))
            # app step k: re-emit every incoming item (rounds 1..3), then stop
            ctx.drv_random_walk(seed, k, 3)
            if k <= 3:
                for l in range(L):
                    inc = w.incoming(l).copy()
                    inc[:, 4:8] = np.frombuffer(np.uint32(k).tobytes(), np.uint8)
                    w.emit_many(l, inc, synth.walk_dests(seed, k, synth.item_id_of(inc), L))
        assert Gs[:3] == [2 * n] * 3
        assert ctx.forward() == w.forward() == 0


# ------------------------------------------------------------------ full size (bench shape)

@pytest.mark.parametrize("exchange", ["fused", "peer"])
@pytest.mark.parametrize("L,n", [(1, 16 * 1024 * 1024), (8, 2 * 1024 * 1024)])
def test_full_size_cfg2_shape(L, n, exchange):
    """BASELINE configs[1] per-rank shape (16M x 48-B items, uniform) at R=1,
    and 8 logical ranks x 2M on one GPU; P1 bit-exact on everything."""
    B = 48
    cap = n if L == 1 else n + n // 8
    with _ctx(B, cap, L) as ctx:
        ctx.set_option(rafi.OPT_EXCHANGE, EXCHANGES[exchange])
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], synth.CONFIG_SEEDS[2], 0, n, local=l)
        p1_forward(ctx, L, B)


@pytest.mark.parametrize("B,scatter", [(44, "threads"), (64, "threads"), (48, "bulk"), (24, "threads")])
def test_full_size_item_sizes(B, scatter):
    """16M items of the cfg5 sweep sizes at R=4 logical ranks, in the launch
    configuration the benches use (auto tile), including the 16-B chunk
    gather (44 B) and the bulk-store path: P1 bit-exact."""
    L, n = 4, 4 * 1024 * 1024
    with _ctx(B, n + n // 8, L) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, SCATTERS[scatter])
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS["uniform"], synth.CONFIG_SEEDS[5], 0, n, local=l)
        p1_forward(ctx, L, B)


def test_host_io_overlap_rounds():
    """rafi_emit_bulk from pinned host memory (copy-in stream, double-buffered
    staging) and rafi_read_incoming_async (copy-out stream) over several
    rounds with no host waits in between: each read must capture its own
    round (the next forward waits for it), matching the oracle."""
    B, L, n, rounds = 48, 2, 30000, 4
    pins = [torch.empty((2 * n, B), dtype=torch.uint8).pin_memory() for _ in range(rounds)]
    host_in = []
    sizes, exp = [], []
    with _ctx(B, 2 * n, L) as ctx:
        for rnd in range(rounds):
            inputs = make_inputs(L, n - 1000 * rnd, B, "uniform", 5 + rnd, rnd=rnd)
            w = oracle_sequential(L, 2 * n, B, inputs)
            w.forward()
            exp.append(w.incoming(1))
            for l, (it, ds) in enumerate(inputs):
                hi, hd = torch.from_numpy(it).pin_memory(), torch.from_numpy(ds).pin_memory()
                host_in.append((hi, hd))  # keep alive until the copies ran
                ctx.emit_bulk(hi, hd, len(ds), local=l)
            ctx.forward()
            m = ctx.num_incoming(1)
            sizes.append(m)
            ctx.read_incoming_async(pins[rnd][:m], local=1)
        ctx.read_wait()
    for rnd in range(rounds):
        assert np.array_equal(canonical(pins[rnd][: sizes[rnd]].numpy()), canonical(exp[rnd])), rnd


@pytest.mark.parametrize("graph", [0, 1])
def test_forward_graph_rounds_with_option_changes(graph):
    """The blocking forward replayed from its cached CUDA graph (default) or
    launched kernel by kernel: P1 bit-exact over rounds of changing sizes,
    with tile / scatter / timing changes between rounds (each forces a
    re-capture)."""
    B, L = 44, 3
    with _ctx(B, 60000, L) as ctx:
        ctx.set_option(rafi.OPT_FORWARD_GRAPH, graph)
        assert ctx.get_option(rafi.OPT_FORWARD_GRAPH) == graph
        steps = [(20000, None), (7, None), (15000, (rafi.OPT_TILE, 1024)), (0, None),
                 (19999, (rafi.OPT_TIMING, 1)), (12345, (rafi.OPT_SCATTER, rafi.SCATTER_BULK)),
                 (20000, (rafi.OPT_TILE, 0))]
        for rnd, (n, opt) in enumerate(steps):
            if opt:
                ctx.set_option(*opt)
            inputs = make_inputs(L, n, B, "skewed", 300 + rnd, rnd=rnd)
            _emit_all(ctx, inputs)
            p1_forward(ctx, L, B)
            if ctx.get_option(rafi.OPT_TIMING) and n:
                st = ctx.stats()  # phase events are recorded by the graph replay too
                assert st["ms_scatter"] > 0 and st["ms_hist"] > 0 and st["ms_total"] > 0, st
        assert ctx.forward() == 0


# ------------------------------------------------------------------ device emit: drop rule and re-emit

@pytest.mark.parametrize("pattern", ["uniform", "self"])
@pytest.mark.parametrize("B", [16, 24, 44, 48, 64, 128])
@pytest.mark.parametrize("cap", [1, 31, 1000, 4133])
def test_device_emit_overflow_drop_rule(B, cap, pattern):
    """Z1/Z2 through rafi::Queue<T>::emitOutgoing (warp-aggregated): more
    emits than capacity (cap not a multiple of 32, so a warp's slot range
    straddles it), mixed invalid destinations.  The counter is not clamped and
    equals the valid emits; invalid ones are counted and take no slot; exactly
    min(ctr, cap) items are kept, each one a distinct generator item with its
    own destination; the forward reports the drops and is P1-exact."""
    L, n, seed = 3, 9001, 23
    thr = synth.invalid_threshold(0.05)
    with _ctx(B, cap, L) as ctx:
        for l in range(L):
            ctx.drv_emit_synthetic(synth.PATTERNS[pattern], seed, 2, n, local=l, invalid_threshold=thr)
        ctrs = []
        for l in range(L):
            items, dests, ctr, inv = ctx.read_outgoing(l)
            ctrs.append(int(ctr))
            exp_it = synth.make_items(l, 2, n, B)
            exp_d = synth.make_dests(pattern, seed, l, 2, n, L, invalid_frac=0.05)
            ok = (exp_d >= 0) & (exp_d < L)
            assert ctr == ok.sum() and inv == (~ok).sum()
            assert len(items) == min(ctr, cap)
            seq = (synth.item_id_of(items) & np.uint64((1 << 40) - 1)).astype(np.int64)
            assert len(np.unique(seq)) == len(seq)               # no item kept twice
            assert np.all(ok[seq])                               # only valid emits take slots
            assert np.array_equal(items, exp_it[seq])            # each slot holds a whole generator item
            assert np.array_equal(dests, exp_d[seq])             # ... with its own destination
        # uniform: a receiver may get more than cap (Z3, refused alike by both sides);
        # self: every rank receives its own cap items, and the stats report the drops
        w, G = p1_forward(ctx, L, B)  # checks dropped == ctr - min(ctr, cap) per rank, then every byte
        if pattern == "self":
            assert G == sum(min(cap, c) for c in ctrs)


@pytest.mark.parametrize("batch", [1, 8])
@pytest.mark.parametrize("B", [4, 8, 12, 16, 20, 44, 48, 64, 128])
def test_device_reemit_of_resident_batch(B, batch):
    """rafi_drv_emit_items: a resident (items, dests) batch re-emitted through
    emitOutgoing (single or batched) with vector loads/stores; the queue holds
    exactly the valid (item, dest) pairs (as a multiset: warp order follows
    the atomics), then P1."""
    L, n = 2, 50001
    inputs = make_inputs(L, n, B, "uniform", 5 + B, invalid_frac=0.02)
    with _ctx(B, n, L) as ctx:
        for l, (it, ds) in enumerate(inputs):
            ctx.drv_emit_items(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), n, local=l, batch=batch)
        for l, (it, ds) in enumerate(inputs):
            items, dests, ctr, inv = ctx.read_outgoing(l)
            ok = (ds >= 0) & (ds < L)
            assert ctr == ok.sum() and inv == (~ok).sum()
            got = np.concatenate([items, dests.view(np.uint8).reshape(-1, 4)], axis=1)
            exp = np.concatenate([it[ok], ds[ok].view(np.uint8).reshape(-1, 4)], axis=1)
            gv = np.sort(got.view(np.dtype((np.void, got.shape[1]))).ravel())
            ev = np.sort(exp.view(np.dtype((np.void, exp.shape[1]))).ravel())
            assert np.array_equal(gv, ev)
        p1_forward(ctx, L, B)


@pytest.mark.parametrize("batch", [1, 8])
@pytest.mark.parametrize("cap", [1, 1000, 30001])
def test_device_reemit_drop_rule(batch, cap):
    """Z1/Z2 for the single and the batched device emit: over capacity (cap
    not a multiple of the 32- or 256-item warp reservation), with invalid
    destinations.  ctr = valid emits, invalid counted, min(ctr, cap) kept,
    every kept slot a distinct input pair with its own destination."""
    B, n = 48, 50001
    (it, ds), = make_inputs(1, n, B, "self", 77, invalid_frac=0.03)
    with _ctx(B, cap, 1) as ctx:
        ctx.drv_emit_items(torch.from_numpy(it).cuda(), torch.from_numpy(ds).cuda(), n, batch=batch)
        items, dests, ctr, inv = ctx.read_outgoing(0)
        ok = (ds >= 0) & (ds < 1)
        assert ctr == ok.sum() and inv == (~ok).sum() and len(items) == min(ctr, cap)
        seq = (synth.item_id_of(items) & np.uint64((1 << 40) - 1)).astype(np.int64)
        assert len(np.unique(seq)) == len(seq) and np.all(ok[seq])
        assert np.array_equal(items, it[seq]) and np.array_equal(dests, ds[seq])
        w, G = p1_forward(ctx, 1, B)
        assert G == min(ctr, cap)


@pytest.mark.parametrize("scatter", [1, 2])  # THREADS (warp tiles at R <= 8), BULK
@pytest.mark.parametrize("B", [16, 44, 48])
def test_diag_redirect_incoming(B, scatter):
    """rafi_diag_redirect_incoming: the FUSED scatter writes rank 1's block
    into a caller buffer instead of the context's queue -- exactly the bytes
    the oracle delivers to rank 1 (P1 on the redirected queue); the other
    ranks' queues are untouched by the redirect, and restoring it brings
    the default back."""
    L, n = 3, 30001
    inputs = make_inputs(L, n, B, "uniform", 21 + B)
    with _ctx(B, L * n, L) as ctx:
        ctx.set_option(rafi.OPT_SCATTER, scatter)
        buf = torch.zeros(L * n * B + 16, dtype=torch.uint8, device="cuda")
        ctx.diag_redirect_incoming(1, buf)
        _emit_all(ctx, inputs)
        w, _ = snapshot_world(ctx, L, B)
        G_o = w.forward()
        assert ctx.forward() == G_o
        m = ctx.num_incoming(1)
        assert m == w.num_incoming(1)
        got = buf[: m * B].cpu().numpy().reshape(m, B)
        assert np.array_equal(got, w.incoming(1))
        for l in (0, 2):
            assert np.array_equal(ctx.read_incoming(l), w.incoming(l))
        ctx.diag_redirect_incoming(1, None)
        _emit_all(ctx, inputs)
        p1_forward(ctx, L, B)
    with _ctx(B, n, 1) as ctx:
        with pytest.raises(rafi.RafiError):
            ctx.diag_redirect_incoming(1, buf)   # not a local rank


@pytest.mark.parametrize("R", [1, 3, 8])
def test_warp_tiles_many_rounds_empty_ranks_and_resize(R):
    """The warp-tile path (128/256-item tiles, R <= 8: k_hist_w, k_scan,
    k_scatter_w) over many forwards on one context: sizes that change every
    round (empty ranks, partial scan blocks and tiles), a resize between
    rounds (new H/O arrays), every round P1-exact against the oracle."""
    B = 48 if R != 3 else 256   # 256- and 128-item warp tiles
    sizes = [[5000, 0, 70001], [0, 0, 0], [2048, 2047, 1], [300000, 4096, 0], [1, 0, 123457]]
    with _ctx(B, 300000, R) as ctx:
        assert ctx.get_option(rafi.OPT_TILE) == (256 if B == 48 else 128)
        for rnd, ns in enumerate(sizes * 2):
            if rnd == len(sizes):
                ctx.resize(400000)
            inputs = [(synth.make_items(s, rnd, ns[s % 3], B)[:, :B].copy(),
                       synth.make_dests("uniform", 40 + rnd, s, rnd, ns[s % 3], R)) for s in range(R)]
            _emit_all(ctx, inputs)
            p1_forward(ctx, R, B)


@pytest.mark.parametrize("B,L,tile", [(16, 8, 256), (44, 8, 256), (48, 8, 256), (64, 8, 256), (96, 8, 128),
                                      (128, 8, 256), (256, 8, 128), (48, 1, 256), (48, 9, None), (42, 4, None),
                                      (520, 2, None)])
def test_automatic_tile_choice(B, L, tile):
    """The automatic binning tile: warp tiles of 256
    items while >= 6 warp regions fit (two TMA stages per warp up to 96 B,
    one above: 16-64 B and 128 B), 128 otherwise; block tiles (256 * 2^k) for
    R > 8, items over 256 B or item sizes that are not a multiple of 4 B."""
    with _ctx(B, 50000, L) as ctx:
        assert ctx.get_option(rafi.OPT_SCATTER) == rafi.SCATTER_THREADS
        t = ctx.get_option(rafi.OPT_TILE)
        if tile is None:
            assert t >= 256 and t & (t - 1) == 0
        else:
            assert t == tile
