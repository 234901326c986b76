"""NEXT-2: several RaFI contexts with different item types on one
communicator -- the N-body exchange pattern: particle
migration (40 B), root-multipole broadcast and subtree responses (24 B),
refinement requests (4 B).  CPU: invariants of the CPU twin; GPU: the driver
kernels + three librafi contexts against the twin + oracle forwarding."""
import numpy as np
import pytest

import oracle

PART = np.dtype([("p", "<f4", 3), ("v", "<f4", 3), ("f", "<f4", 3), ("mass", "<f4")])
VIRT = np.dtype([("c", "<f4", 3), ("mass", "<f4"), ("smax", "<f4"), ("src", "<i4")])


def _as(items, dt):
    return np.frombuffer(np.ascontiguousarray(items).tobytes(), dt)


def _canon(items):
    """multiset order: sort rows by their bytes"""
    if len(items) == 0:
        return items
    v = np.ascontiguousarray(items).view(np.dtype((np.void, items.shape[1]))).ravel()
    return items[np.argsort(v, kind="stable")]


def _morton_py(x, y, z, R):
    q = [min(int(np.float32(c) * np.float32(1024.0)), 1023) for c in (x, y, z)]
    code = 0
    for b in range(10):
        for a in range(3):
            code |= ((q[a] >> b) & 1) << (3 * b + a)
    return (code * R) >> 30


def _step(nb, dt=1.0 / 16, theta2=0.25, check=True):
    nb.migrate(dt)
    assert nb.P.forward() >= 0
    nb.compute_stats()
    nb.root()
    nb.V.forward()
    nb.refine(theta2)
    nb.Q.forward()
    nb.respond()
    nb.V.forward()


def test_morton_owner_matches_bit_interleaving():
    rng = np.random.default_rng(0)
    for R in (1, 2, 3, 4, 8, 16):
        for x, y, z in rng.random((200, 3), dtype=np.float32):
            assert oracle.morton_owner(float(x), float(y), float(z), R) == _morton_py(x, y, z, R)
    assert oracle.morton_owner(0.0, 0.0, 0.0, 8) == 0
    assert oracle.morton_owner(0.9999, 0.9999, 0.9999, 8) == 7


def test_nbody_pattern_invariants():
    R, n = 8, 3000
    nb = oracle.NBody(R, 4 * n, 64 * R, 4 * R)
    for r in range(R):
        nb.seed(r, n, 77)
    assert nb.P.forward() == R * n
    for step in range(3):
        nb.migrate(1.0 / 16)
        assert nb.P.forward() == R * n                     # particles are conserved
        for r in range(R):
            p = _as(nb.P.incoming(r), PART)
            assert all(oracle.morton_owner(*map(float, q), R) == r for q in p["p"][:200])
        nb.compute_stats()
        st = nb.stats
        counts = st[:, 0].astype(np.int64)
        assert counts.sum() == R * n
        assert np.array_equal(st[:, 10::4].sum(axis=1), st[:, 0])  # octants partition each rank
        nb.root()
        G = nb.V.forward()
        nonempty = int((counts > 0).sum())
        assert G == nonempty * (nonempty - 1)              # every non-empty rank hears every other root
        for r in range(R):
            roots = _as(nb.V.incoming(r), VIRT)
            assert sorted(roots["src"]) == [s for s in range(R) if s != r and counts[s] > 0]
            assert all(int(m) == counts[s] for m, s in zip(roots["mass"], roots["src"]))
        nb.refine(0.25)
        Gq = nb.Q.forward()
        nb.respond()
        Gv = nb.V.forward()
        # each request is answered by every non-empty octant of the requested rank
        octs = (st[:, 10::4] > 0).sum(axis=1)
        exp = 0
        for r in range(R):
            for s in _as(nb.Q.incoming(r), np.dtype("<i4")):
                exp += int(octs[r])
        assert Gv == exp and Gq >= 0


@pytest.mark.gpu
@pytest.mark.parametrize("R,n", [(8, 4000), (4, 6000)])
def test_gpu_nbody_three_contexts_match_twin(R, n):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2605_30294_b200 import rafi
    s = torch.cuda.Stream()
    stats = torch.zeros((R, oracle.NB_STATS), dtype=torch.int64, device="cuda")
    nb = oracle.NBody(R, 4 * n, 64 * R, 4 * R)
    P = rafi.Context(40, 4 * n, local_ranks=R, stream=s)
    V = rafi.Context(24, 64 * R, local_ranks=R, stream=s)
    Q = rafi.Context(4, 4 * R, local_ranks=R, stream=s)
    try:
        def same(ctx, w, tag):
            for r in range(R):
                assert np.array_equal(_canon(ctx.read_incoming(r)), _canon(w.incoming(r))), (tag, r)

        for r in range(R):
            P.drv_nbody_seed(n, 77, local=r)
            nb.seed(r, n, 77)
        assert P.forward() == nb.P.forward()
        same(P, nb.P, "seed")
        for step in range(3):
            P.drv_nbody_migrate(1.0 / 16)
            nb.migrate(1.0 / 16)
            assert P.forward() == nb.P.forward()
            same(P, nb.P, "migrate")
            P.drv_nbody_stats(stats)
            nb.compute_stats()
            s.synchronize()
            assert np.array_equal(stats.cpu().numpy().astype(np.uint64), nb.stats)
            V.drv_nbody_root(stats)
            nb.root()
            assert V.forward() == nb.V.forward()
            same(V, nb.V, "root")
            V.drv_nbody_refine(Q, stats, 0.25)
            nb.refine(0.25)
            assert Q.forward() == nb.Q.forward()
            same(Q, nb.Q, "refine")
            Q.drv_nbody_respond(V, stats)
            nb.respond()
            assert V.forward() == nb.V.forward()
            same(V, nb.V, "respond")
    finally:
        P.close(); V.close(); Q.close()
