"""Full-size R=8 parity on one GPU (BASELINE configs[1] to configs[4]).

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


# ------------------------------------------------------------------ cfg3 / cfg4 at full size, sampled twin
#
# The proxies' per-item dynamics are independent of the other items (each
# ray's marching and scattering hashes only its own id and state; each
# particle's RK4 step only its own position), and forwarding only routes
# them.  So the full-size GPU run (the whole 8-rank world on one B200) is
# checked item by item against the CPU twin run on a 1-in-SAMPLE subset of the
# same seeds: the twin's queues hold exactly the sampled items, and the
# GPU's queues, restricted to the sampled ids, must equal them bit for bit.

SAMPLE = 32


def _sampled_twin(R, cap_full, cap, B, seed_fn, key_off):
    """A twin world (capacity cap) whose outgoing queues hold the sampled
    seeds only (the full seeding, capacity cap_full, filtered by id in slot
    order)."""
    full = oracle.World(R, cap_full, B)
    for r in range(R):
        seed_fn(full, r)
    w = oracle.World(R, cap, B)
    for r in range(R):
        items, dests = full.out_items(r), full.out_dests(r)
        ids = items[:, key_off:key_off + 4].copy().view(np.uint32).ravel()
        keep = ids % SAMPLE == 0
        w.emit_many(r, items[keep], dests[keep])
    full.close()
    return w


def _sampled_sorted(items, key_off):
    ids = items[:, key_off:key_off + 4].copy().view(np.uint32).ravel()
    sub = items[ids % SAMPLE == 0]
    sid = sub[:, key_off:key_off + 4].copy().view(np.uint32).ravel()
    return sub[np.argsort(sid, kind="stable")]


def test_cfg3_full_size_ray_march_sampled_twin():
    """configs[2]: 2x2x2 bricks, 8 ranks x 4,194,304 48-B rays, p_scatter
    0.01, marched and forwarded until G = 0 -- every ray retires on the GPU,
    and every sampled ray retires with the twin's integral, bit for bit (its
    whole trajectory: steps, scatter events, brick crossings, forwards)."""
    R, n, B = 8, 4 * 1024 * 1024, 48
    g = oracle.grid_dims(R)
    p_thr, max_b, max_s, seed = int(0.01 * 2**32), 4, 256, 0x5EED0003
    res_g = torch.full((R * n,), -1.0, dtype=torch.float32, device="cuda")
    with rafi.Context(B, 2 * n, local_ranks=R) as ctx:
        for r in range(R):
            ctx.drv_march_seed(n, seed, g, local=r)
        rounds_g = 0
        while True:
            if ctx.forward() == 0:
                break
            rounds_g += 1
            ctx.drv_march_step(rounds_g, seed, p_thr, max_b, max_s, g, res_g)
            assert rounds_g < 64
    res_g = res_g.cpu().numpy()
    assert np.all(res_g >= 0)                          # every ray retired exactly once
    w = _sampled_twin(R, n, R * n // SAMPLE, B, lambda wl, r: wl.march_seed(r, n, seed, g), 28)
    res_c = np.full(R * n, -1.0, np.float32)
    rounds_c = 0
    while True:
        if w.forward() == 0:
            break
        rounds_c += 1
        for r in range(R):
            w.march_step(r, seed, p_thr, max_b, max_s, g, res_c)
    w.close()
    sampled = np.arange(0, R * n, SAMPLE)
    assert np.all(res_c[sampled] >= 0) and rounds_c <= rounds_g
    assert np.array_equal(res_g[sampled].view(np.uint32), res_c[sampled].view(np.uint32))


def test_cfg4_full_size_advection_sampled_twin():
    """configs[3]: 2x2x2 macrocells, 8 ranks x 1,048,576 16-B seeds, 64 RK4
    rounds -- at rounds 1, 8, 32 and 63 every rank's incoming queue,
    restricted to the sampled ids, equals the twin's bit for bit; the run
    ends after exactly 64 rounds."""
    R, n, B = 8, 1024 * 1024, 16
    g = oracle.grid_dims(R)
    omega, eps, h, max_rounds, seed = 2 * np.pi / 64, 1.0 / 128, 1.0, 64, 0x5EED0004
    w = _sampled_twin(R, n, R * n // SAMPLE, B, lambda wl, r: wl.advect_seed(r, n, seed, g), 0)
    checks = {1, 8, 32, 63}
    with rafi.Context(B, 2 * n, local_ranks=R) as ctx:
        for r in range(R):
            ctx.drv_advect_seed(n, seed, g, local=r)
        k = 0
        while True:
            G = ctx.forward()
            Gw = w.forward()
            assert (G == 0) == (Gw == 0)
            if k in checks:
                for r in range(R):
                    got = _sampled_sorted(ctx.read_incoming(r), 0)
                    exp = _sampled_sorted(w.incoming(r), 0)
                    assert np.array_equal(got, exp), (k, r)
            if G == 0:
                break
            k += 1
            ctx.drv_advect_step(k, max_rounds, omega, eps, h, g)
            for r in range(R):
                w.advect_step(r, k, max_rounds, omega, eps, h, g)
        assert k == max_rounds
    w.close()
