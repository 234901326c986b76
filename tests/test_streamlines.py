"""NEXT-4: streamlines on a sampled vector field (§5.4).

CPU: the twin (oracle/streamlines.c) pinned by RK4's exactness for constant
fields (dyadic values make every float operation exact), trilinear
interpolation of linear fields, and rotation-invariant radii.  GPU: the driver
(per-rank blocks + one-vertex halo) against the twin (global field) round by
round, and partition independence: 1, 2 and 8 ranks give bit-identical
streamline end points."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle

PART = np.dtype([("id", "<u4"), ("p", "<f4", 3)])


def lattice(n, fn):
    """(n, n, n, 3) float32 field with v[k, j, i] = fn(x_i, y_j, z_k) on [0,1]^3."""
    c = np.linspace(0.0, 1.0, n)
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    v = np.stack(fn(x, y, z), axis=-1)
    return np.ascontiguousarray(v, dtype=np.float32)


def abc_field(n):
    A, B, C = 1.0, 0.7, 0.43
    tp = 2 * np.pi
    return lattice(n, lambda x, y, z: (A * np.sin(tp * z) + C * np.cos(tp * y),
                                       B * np.sin(tp * x) + A * np.cos(tp * z),
                                       C * np.sin(tp * y) + B * np.cos(tp * x)))


def run_twin(field, grid, seeds, h, eps, max_steps):
    R = grid[0] * grid[1] * grid[2]
    n = len(seeds)
    sl = oracle.Streamlines(R, 2 * n + 16, field, grid)
    sl.seed(0, seeds, 0)
    rpos = np.full((n, 3), np.nan, np.float32)
    rst = np.full(n, 0xFFFFFFFF, np.uint32)
    rounds, history = 0, []
    G = sl.w.forward()
    history.append(G)
    while G:
        rounds += 1
        sl.step(rounds, h, eps, max_steps, rpos, rst)
        G = sl.w.forward()
        history.append(G)
    return rpos, rst, history, sl


# ------------------------------------------------------------------ CPU pins

def test_constant_field_rk4_is_exact():
    c = (2.0**-4, -(2.0**-5), 2.0**-6)
    field = lattice(17, lambda x, y, z: (np.full_like(x, c[0]), np.full_like(x, c[1]), np.full_like(x, c[2])))
    h = 6 * 2.0**-6                       # h/6 = 2^-6: every operation below is exact
    seeds = np.array([[k / 64, 0.5 + k / 1024, 0.25 + k / 512] for k in range(1, 40)], np.float32)
    rpos, rst, hist, _ = run_twin(field, (2, 2, 2), seeds, h, 1e-9, 7)
    for i, s in enumerate(seeds):
        steps = int(rst[i])
        exp = [Fraction(float(s[a])) + steps * Fraction(h) * Fraction(c[a]) for a in range(3)]
        assert [Fraction(float(v)) for v in rpos[i]] == exp          # p + steps*h*c exactly
        assert steps == 7 or not (0 <= float(exp[0] + Fraction(h) * Fraction(c[0])) < 1)


def test_owner_face_rule_and_empty_streamline():
    field = lattice(17, lambda x, y, z: (x * 0, x * 0, x * 0 + 1.0))
    sl = oracle.Streamlines(8, 64, field, (2, 2, 2))
    assert sl.owner([0.49, 0.1, 0.1]) == 0
    assert sl.owner([0.5, 0.1, 0.1]) == 1                # a shared face belongs to the upper cell's block
    assert sl.owner([1.0, 1.0, 1.0]) == 7                # clamped to the last cell
    rpos, rst, hist, _ = run_twin(field, (2, 2, 2), np.array([[1.5, 0.2, 0.2]], np.float32), 0.01, 1e-9, 5)
    assert hist == [0] and rst[0] == 0xFFFFFFFF          # a seed outside the domain: empty streamline


def test_rigid_rotation_keeps_radius():
    """v = w(-(y-1/2), x-1/2, 0) is linear, so trilinear interpolation is exact
    up to rounding; RK4 then keeps the radius to O((w h)^5) per step."""
    w = 2 * math.pi
    field = lattice(33, lambda x, y, z: (-w * (y - 0.5), w * (x - 0.5), 0 * z))
    rng = np.random.default_rng(3)
    seeds = np.c_[0.5 + 0.3 * (rng.random((50, 2)) - 0.5), rng.random(50)].astype(np.float32)
    h = 1.0 / 256
    rpos, rst, hist, _ = run_twin(field, (2, 2, 1), seeds, h, 1e-9, 64)
    r0 = np.hypot(seeds[:, 0] - 0.5, seeds[:, 1] - 0.5)
    r1 = np.hypot(rpos[:, 0] - 0.5, rpos[:, 1] - 0.5)
    assert np.all(rst == 64)
    assert np.max(np.abs(r1 - r0)) < 64 * ((w * h) ** 5 + 1e-6)
    ang = np.arctan2(rpos[:, 1] - 0.5, rpos[:, 0] - 0.5) - np.arctan2(seeds[:, 1] - 0.5, seeds[:, 0] - 0.5)
    assert np.allclose(np.mod(ang, 2 * np.pi), 64 * w * h, atol=1e-4)


# ------------------------------------------------------------------ GPU

def _gpu_run(field, grid, seeds, h, eps, max_steps, compare_twin=None):
    torch = pytest.importorskip("torch")
    from paper_2605_30294_b200 import rafi
    R = grid[0] * grid[1] * grid[2]
    n = len(seeds)
    rpos = torch.full((n, 3), float("nan"), dtype=torch.float32, device="cuda")
    rst = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    hist = []
    with rafi.Context(16, 2 * n + 16, local_ranks=R) as ctx:
        f = rafi.StreamField(ctx, field, grid)
        try:
            f.seed(seeds, 0, local=0)
            G = ctx.forward()
            hist.append(G)
            k = 0
            twin = compare_twin
            while G:
                k += 1
                f.step(k, h, eps, max_steps, rpos, rst)
                G = ctx.forward()
                hist.append(G)
                if twin is not None and k <= 3:
                    for r in range(R):
                        got = np.sort(np.frombuffer(ctx.read_incoming(r).tobytes(), PART), order="id")
                        assert got.tobytes() == twin[k][r], (k, r)
            assert f.halo_misses() == 0
        finally:
            f.close()
    return rpos.cpu().numpy(), rst.cpu().numpy().astype(np.uint32), hist


def _twin_rounds(field, grid, seeds, h, eps, max_steps, upto=3):
    """Per-round incoming queues (sorted by id) of the CPU twin."""
    R = grid[0] * grid[1] * grid[2]
    n = len(seeds)
    sl = oracle.Streamlines(R, 2 * n + 16, field, grid)
    sl.seed(0, seeds, 0)
    sl.w.forward()
    rpos = np.full((n, 3), np.nan, np.float32)
    rst = np.full(n, 0xFFFFFFFF, np.uint32)
    out = {}
    for k in range(1, upto + 1):
        sl.step(k, h, eps, max_steps, rpos, rst)
        sl.w.forward()
        out[k] = [np.sort(np.frombuffer(sl.w.incoming(r).tobytes(), PART), order="id").tobytes() for r in range(R)]
    return out


@pytest.mark.gpu
def test_gpu_streamlines_match_twin_and_are_partition_independent():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    field = abc_field(33)
    vmax = float(np.abs(field).max())
    h = 0.4 * (1.0 / 32) / (vmax * 2)          # stages stay within half a cell: halo suffices
    rng = np.random.default_rng(11)
    seeds = rng.random((20000, 3)).astype(np.float32)
    eps, max_steps = 1e-7, 40
    twin_pos, twin_st, twin_hist, _ = run_twin(field, (2, 2, 2), seeds, h, eps, max_steps)
    rounds = _twin_rounds(field, (2, 2, 2), seeds, h, eps, max_steps)
    p8, s8, h8 = _gpu_run(field, (2, 2, 2), seeds, h, eps, max_steps, compare_twin=rounds)
    assert h8 == twin_hist
    assert np.array_equal(s8, twin_st)
    assert np.array_equal(p8.view(np.uint32), twin_pos.view(np.uint32))   # bitwise
    for grid in ((1, 1, 1), (2, 1, 1), (2, 2, 1)):
        p, s, _ = _gpu_run(field, grid, seeds, h, eps, max_steps)
        assert np.array_equal(s, s8) and np.array_equal(p.view(np.uint32), p8.view(np.uint32)), grid
