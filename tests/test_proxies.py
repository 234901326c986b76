"""Proxy applications (cfg3 ray marcher, cfg4 particle advector).

CPU part: the oracle's twins (oracle/proxies.c) pinned by properties the
mathematics fixes -- exact invariants of special cases and error bounds
against exact (float64) solutions.  GPU part: the drivers
(csrc/drivers.cu, through librafi's C ABI and the device header) against the
CPU twins + oracle forwarding, round by round, bit for bit after canonical
ordering by item id.
"""
import math

import numpy as np
import pytest

import oracle

GRID8 = oracle.grid_dims(8)
PART = np.dtype([("id", "<u4"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4")])
RAY = np.dtype([("o", "<f4", 3), ("d", "<f4", 3), ("t", "<f4"), ("id", "<u4"), ("integral", "<f4"),
                ("rng", "<u4"), ("bounces", "<u4"), ("pad", "<u4")])


def _parts(items):
    return np.frombuffer(np.ascontiguousarray(items).tobytes(), PART)


def _rays(items):
    return np.frombuffer(np.ascontiguousarray(items).tobytes(), RAY)


def _seed_world(R, n, B, kind, seed):
    g = oracle.grid_dims(R)
    w = oracle.World(R, 2 * n * R, B)
    for r in range(R):
        (w.advect_seed if kind == "advect" else w.march_seed)(r, n, seed, g)
    assert w.forward() == R * n
    return w, g


# ------------------------------------------------------------------ CPU pins

def test_grid_owner_is_the_containing_cell():
    g = GRID8
    for x, y, z in [(0.1, 0.1, 0.1), (0.9, 0.1, 0.1), (0.1, 0.9, 0.1), (0.9, 0.9, 0.9), (0.5, 0.49, 0.75)]:
        cx, cy, cz = int(x >= 0.5), int(y >= 0.5), int(z >= 0.5)
        assert oracle.grid_owner(x, y, z, g) == (cz * 2 + cy) * 2 + cx


def test_seeds_are_in_their_own_cell():
    w, g = _seed_world(8, 500, 16, "advect", 3)
    for r in range(8):
        p = _parts(w.incoming(r))
        assert len(p) == 500     # every seed lies in its rank's own cell: nothing moved
        cx, cy, cz = r % 2, (r // 2) % 2, r // 4
        assert np.all((p["x"] >= cx / 2) & (p["x"] < (cx + 1) / 2))
        assert np.all((p["z"] >= cz / 2) & (p["z"] < (cz + 1) / 2))


def test_advection_pure_drift_is_exact():
    """omega = 0, h = 6, eps = 2^-10: every RK4 stage is (0,0,eps), h/6 = 1 and
    6*eps is exact, so x and y never change and each step adds 6*eps to z up to
    IEEE rounding of the one addition (|dz - 6 eps| <= ulp(z')/2)."""
    R, n = 8, 400
    w, g = _seed_world(R, n, 16, "advect", 9)
    eps, h = 2.0**-10, 6.0
    prev = {}
    for r in range(R):
        for p in _parts(w.incoming(r)):
            prev[int(p["id"])] = (float(p["x"]), float(p["y"]), float(p["z"]))
    rounds = 0
    while True:
        for r in range(R):
            w.advect_step(r, rounds + 1, 10**6, 0.0, eps, h, g)
        G = w.forward()
        rounds += 1
        cur = {}
        for r in range(R):
            for p in _parts(w.incoming(r)):
                i = int(p["id"])
                x, y, z = float(p["x"]), float(p["y"]), float(p["z"])
                px, py, pz = prev[i]
                assert x == px and y == py
                ulp = float(np.spacing(np.float32(z)))
                assert abs((z - pz) - 6 * eps) <= ulp / 2 + 1e-12
                assert oracle.grid_owner(x, y, z, g) == r      # delivered to the owner
                cur[i] = (x, y, z)
        # a particle retires exactly when it would leave the domain (z >= 1)
        for i, (px, py, pz) in prev.items():
            if i not in cur:
                assert pz + 6 * eps >= 1.0 - 1e-6
        prev = cur
        if G == 0:
            break
    # the slowest particle starts at z >= 0 and needs at most ceil(1 / (6 eps)) steps to leave
    assert rounds <= math.ceil(1.0 / (6 * eps)) + 1


def test_advection_rigid_rotation_rk4_accuracy():
    """eps = 0: one RK4 step of the rotation v = w(-(y-1/2), x-1/2) is the exact
    rotation by angle w*h up to the RK4 local error O((w h)^5) (the radius is
    kept to O((w h)^6)); checked against the float64 exact rotation."""
    R, n = 8, 300
    w, g = _seed_world(R, n, 16, "advect", 21)
    omega, h = 2 * math.pi / 64, 1.0
    before = {}
    for r in range(R):
        for p in _parts(w.incoming(r)):
            before[int(p["id"])] = (float(p["x"]), float(p["y"]), float(p["z"]))
    for r in range(R):
        w.advect_step(r, 1, 64, omega, 0.0, h, g)
    w.forward()
    a = omega * h
    bound = a**5 / 120 * 0.71 + 4e-7      # local error * max radius + float32 rounding
    seen = 0
    for r in range(R):
        for p in _parts(w.incoming(r)):
            x0, y0, z0 = before[int(p["id"])]
            ex = 0.5 + math.cos(a) * (x0 - 0.5) - math.sin(a) * (y0 - 0.5)
            ey = 0.5 + math.sin(a) * (x0 - 0.5) + math.cos(a) * (y0 - 0.5)
            assert abs(float(p["x"]) - ex) <= bound and abs(float(p["y"]) - ey) <= bound
            assert float(p["z"]) == z0
            seen += 1
    assert seen > 0.8 * R * n


def test_ray_march_straight_line_exit():
    """p_scatter = 0: rays fly straight; direction and id never change, t grows
    by exactly 1/256 per step, the integral stays in [0, t], and each ray
    retires at the float64 slab exit distance of its line from [0,1)^3 within
    one march step."""
    R, n = 8, 300
    w, g = _seed_world(R, n, 48, "march", 5)
    start = {}
    for r in range(R):
        for y in _rays(w.incoming(r)):
            start[int(y["id"])] = (y["o"].astype(np.float64), y["d"].astype(np.float64))
            assert abs(np.linalg.norm(y["d"].astype(np.float64)) - 1.0) < 1e-6
    res = np.full(R * n, -1.0, np.float32)
    last_t = {}
    rounds = 0
    while True:
        for r in range(R):
            w.march_step(r, 5, 0, 8, 100000, g, res)
        G = w.forward()
        rounds += 1
        for r in range(R):
            for y in _rays(w.incoming(r)):
                i = int(y["id"])
                o, d = start[i]
                assert np.array_equal(y["d"].astype(np.float64), d)
                t = float(y["t"])
                assert t * 256 == round(t * 256)
                assert 0.0 <= float(y["integral"]) <= t
                assert oracle.grid_owner(*[float(v) for v in y["o"]], g) == r
                last_t[i] = t
        if G == 0:
            break
    assert np.all(res >= 0)
    for i, (o, d) in start.items():
        with np.errstate(divide="ignore"):
            t1 = np.where(d > 0, (1.0 - o) / d, np.where(d < 0, (0.0 - o) / d, np.inf))
        t_exit = float(np.min(t1))
        assert res[i] <= t_exit + 1e-3
    assert rounds <= 3 + 1   # a straight line crosses at most 3 brick faces of a 2x2x2 grid


def _march_once(w, R, g, seed, p_thr, max_bounces, max_steps, n):
    res = np.full(R * n, -1.0, np.float32)
    for r in range(R):
        w.march_step(r, seed, p_thr, max_bounces, max_steps, g, res)
    return res, w.forward()


def _dist_to_boundary(o):
    return float(min(min(o), min(1.0 - np.asarray(o, np.float64))))


def test_ray_march_always_scatter_bounce_count_and_time():
    """p_thr = 2^32 - 1 (a scatter event at every step, barring hash value
    2^32-1) and max_steps = max_bounces = k on one brick: a ray whose origin
    is farther than k/256 from the domain boundary cannot leave it, so it
    takes exactly k steps -- t == k/256 exactly (dyadic sums), bounces == k,
    a unit direction after every redirect, displacement <= k/256 -- and is
    re-emitted to its own rank.  One more step makes bounces = k+1 > k: each
    of them retires on that step with 0 < integral <= t + 1/256."""
    R, n, k, seed = 1, 4000, 6, 11
    w, g = _seed_world(R, n, 48, "march", seed)
    start = {int(y["id"]): y["o"].astype(np.float64) for y in _rays(w.incoming(0))}
    deep = {i for i, o in start.items() if _dist_to_boundary(o) > (k + 1) / 256.0}
    assert len(deep) > 0.8 * n
    res, G = _march_once(w, R, g, seed, 2**32 - 1, k, k, n)
    rays = {int(y["id"]): y for y in _rays(w.incoming(0))}
    assert deep <= set(rays)                       # every deep ray survives the k steps
    for i in deep:
        y = rays[i]
        assert float(y["t"]) == k / 256.0 and int(y["bounces"]) == k
        assert abs(np.linalg.norm(y["d"].astype(np.float64)) - 1.0) < 4e-7
        assert np.linalg.norm(y["o"].astype(np.float64) - start[i]) <= k / 256.0 + 1e-6
        assert 0.0 < float(y["integral"]) <= k / 256.0
        assert res[i] == -1.0                      # not retired
    before = {i: float(rays[i]["integral"]) for i in deep}
    res, G = _march_once(w, R, g, seed, 2**32 - 1, k, 10**6, n)
    assert G == 0                                  # everything retired (bounce limit or domain exit)
    for i in deep:
        assert before[i] < res[i] <= before[i] + 1.0 / 256.0


@pytest.mark.parametrize("p_log2", [1, 2, 3])
def test_ray_march_scatter_probability(p_log2):
    """p_thr = 2^(32-p) scatters with probability 2^-p per step: over m steps
    deep inside one brick the mean bounce count is m * 2^-p (binomial; a
    reversed comparison would give m * (1 - 2^-p)), and redirected
    directions are isotropic (mean direction ~ 0)."""
    R, n, m, seed = 1, 20000, 8, 7
    w, g = _seed_world(R, n, 48, "march", seed)
    deep = {int(y["id"]) for y in _rays(w.incoming(0)) if _dist_to_boundary(y["o"]) > (m + 1) / 256.0}
    res, G = _march_once(w, R, g, seed, 2 ** (32 - p_log2), 10**6, m, n)
    rays = [y for y in _rays(w.incoming(0)) if int(y["id"]) in deep]
    b = np.array([int(y["bounces"]) for y in rays], np.float64)
    p = 2.0 ** -p_log2
    sd = np.sqrt(m * p * (1 - p) / len(b))
    assert abs(b.mean() - m * p) < 6 * sd
    moved = np.array([y["d"] for y in rays if int(y["bounces"]) > 0], np.float64)
    assert len(moved) > 1000 and np.all(np.abs(moved.mean(axis=0)) < 0.05)
    assert np.all(np.abs(np.linalg.norm(moved, axis=1) - 1.0) < 4e-7)


# ------------------------------------------------------------------ GPU parity

def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2605_30294_b200 import rafi
    return torch, rafi


def _canon(items, key_off):
    if len(items) == 0:
        return items
    ids = items[:, key_off:key_off + 4].copy().view(np.uint32).ravel()
    return items[np.argsort(ids, kind="stable")]


@pytest.mark.gpu
@pytest.mark.parametrize("R,n", [(8, 20000), (2, 30000), (1, 10000)])
def test_gpu_advection_matches_cpu_twin(R, n):
    torch, rafi = _gpu()
    g = oracle.grid_dims(R)
    omega, eps, h, max_rounds = 2 * math.pi / 64, 1.0 / 128, 1.0, 64
    w = oracle.World(R, 2 * n, 16)
    with rafi.Context(16, 2 * n, local_ranks=R) as ctx:
        for r in range(R):
            ctx.drv_advect_seed(n, 11, g, local=r)
            w.advect_seed(r, n, 11, g)
        k = 0
        while True:
            G = ctx.forward()
            assert G == w.forward()
            assert np.array_equal(ctx.matrix(), w.C())
            for r in range(R):
                assert np.array_equal(_canon(ctx.read_incoming(r), 0), _canon(w.incoming(r), 0)), (k, r)
            if G == 0:
                break
            k += 1
            ctx.drv_advect_step(k, max_rounds, omega, eps, h, g)
            for r in range(R):
                w.advect_step(r, k, max_rounds, omega, eps, h, g)
        assert k == max_rounds


@pytest.mark.gpu
@pytest.mark.parametrize("R,n,p", [(8, 20000, 0.01), (4, 20000, 0.02), (1, 5000, 0.05)])
def test_gpu_ray_march_matches_cpu_twin(R, n, p):
    torch, rafi = _gpu()
    g = oracle.grid_dims(R)
    thr, max_b, max_s = int(p * 2**32), 4, 256
    w = oracle.World(R, 2 * n, 48)
    res_c = np.full(R * n, -1.0, np.float32)
    res_g = torch.full((R * n,), -1.0, dtype=torch.float32, device="cuda")
    with rafi.Context(48, 2 * n, local_ranks=R) as ctx:
        for r in range(R):
            ctx.drv_march_seed(n, 13, g, local=r)
            w.march_seed(r, n, 13, g)
        rounds = 0
        while True:
            G = ctx.forward()
            assert G == w.forward()
            for r in range(R):
                assert np.array_equal(_canon(ctx.read_incoming(r), 28), _canon(w.incoming(r), 28)), (rounds, r)
            if G == 0:
                break
            rounds += 1
            ctx.drv_march_step(rounds, 13, thr, max_b, max_s, g, res_g)
            for r in range(R):
                w.march_step(r, 13, thr, max_b, max_s, g, res_c)
        torch.cuda.synchronize()
        assert np.array_equal(res_g.cpu().numpy(), res_c)
        assert np.all(res_c >= 0)
