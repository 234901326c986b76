"""CPU oracle for RaFI forwarding -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product (``paper_2605_30294_b200``) never imports it, and the two share no
code: see ``oracle/rafi_oracle.c`` for the implementation and its citations.

This module is a ctypes wrapper (argument marshalling only) around
``oracle/liborafi.so``, which it compiles with gcc on first use if missing or
stale.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rafi_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "digest.c"), os.path.join(_HERE, "proxies.c"), os.path.join(_HERE, "nbody.c"),
         os.path.join(_HERE, "streamlines.c")]
_LIB = os.path.join(_HERE, "liborafi.so")

OK = 0
ERR_ARG = -1
ERR_NOMEM = -2
ERR_RECV_OVERFLOW = -3


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, -O2, no fast-math, no FMA contraction,
    single-threaded)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", tmp] + _SRCS + ["-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, u64, i64, i32, vp = C.c_void_p, C.c_uint64, C.c_int64, C.c_int, C.c_void_p
        sig = {
            "orc_create": (P, [i32, u64, u64]),
            "orc_destroy": (None, [P]),
            "orc_num_incoming": (u64, [P, i32]),
            "orc_get_incoming": (i32, [P, i32, u64, vp]),
            "orc_emit": (i32, [P, i32, vp, i64]),
            "orc_load_snapshot": (i32, [P, i32, vp, vp, u64, u64]),
            "orc_emit_many": (u64, [P, i32, vp, vp, u64]),
            "orc_set_incoming": (i32, [P, i32, vp, u64]),
            "orc_forward_plain": (i64, [P]),
            "orc_forward_literal": (i64, [P]),
            "orc_pack_keys": (None, [vp, u64, vp]),
            "orc_radix_sort_keys": (i32, [vp, u64]),
            "orc_gather": (None, [vp, vp, u64, u64, vp, vp]),
            "orc_compute_segments": (None, [vp, u64, i32, vp, vp]),
            "orc_alltoall_u64": (None, [i32, vp, vp]),
            "orc_alltoallv_bytes": (None, [i32, vp, vp, vp, vp, vp]),
            "orc_R": (i32, [P]),
            "orc_cap": (u64, [P]),
            "orc_B": (u64, [P]),
            "orc_out_ptr": (P, [P, i32]),
            "orc_dest_ptr": (P, [P, i32]),
            "orc_in_ptr": (P, [P, i32]),
            "orc_binned_ptr": (P, [P, i32]),
            "orc_emitted": (u64, [P, i32]),
            "orc_invalid": (u64, [P, i32]),
            "orc_dropped_last": (u64, [P, i32]),
            "orc_invalid_last": (u64, [P, i32]),
            "orc_C_ptr": (P, [P]),
            "orc_send_off_ptr": (P, [P]),
            "orc_recv_off_ptr": (P, [P]),
            "orc_G": (u64, [P]),
            # digest.c (streaming-digest mode of the plain forward)
            "orc_digest_items": (u64, [vp, u64, u64]),
            "orc_digest_create": (P, [i32, u64, u64]),
            "orc_digest_destroy": (None, [P]),
            "orc_digest_feed": (i32, [P, i32, vp, vp, u64]),
            "orc_digest_finish": (i64, [P]),
            "orc_digest_value": (u64, [P, i32]),
            "orc_digest_C_ptr": (P, [P]),
            # proxies.c (CPU twins of the proxy applications)
            "orc_grid_owner": (i32, [C.c_float, C.c_float, C.c_float, i32, i32, i32]),
            "orc_advect_seed": (None, [P, i32, u64, u64, i32, i32, i32]),
            "orc_advect_step": (None, [P, i32, C.c_uint32, C.c_uint32, C.c_float, C.c_float, C.c_float,
                                       i32, i32, i32]),
            "orc_march_seed": (None, [P, i32, u64, u64, i32, i32, i32]),
            "orc_march_step": (None, [P, i32, u64, C.c_uint32, C.c_uint32, C.c_uint32, i32, i32, i32, vp]),
            # nbody.c (CPU twin of the multi-context N-body exchange pattern)
            "orc_morton_owner": (i32, [C.c_float, C.c_float, C.c_float, i32]),
            "orc_nbody_seed": (None, [P, i32, u64, u64]),
            "orc_nbody_migrate": (None, [P, i32, C.c_float]),
            "orc_nbody_stats": (None, [P, i32, vp]),
            "orc_nbody_root": (None, [P, i32, vp]),
            "orc_nbody_refine": (None, [P, P, i32, vp, C.c_float]),
            "orc_nbody_respond": (None, [P, P, i32, vp]),
            # streamlines.c (CPU twin of the streamline driver, global-field sampling)
            "orc_sl_owner": (i32, [vp, i32, i32, i32, i32, i32, i32]),
            "orc_sl_seed": (None, [P, i32, vp, i32, i32, i32, i32, i32, i32, vp, u64, C.c_uint32]),
            "orc_sl_step": (None, [P, i32, vp, i32, i32, i32, i32, i32, i32, C.c_uint32, C.c_float, C.c_float,
                                   C.c_uint32, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _view(ptr, n, dtype):
    n = int(n)
    dtype = np.dtype(dtype)
    if n == 0:
        return np.zeros(0, dtype)
    buf = (C.c_uint8 * (n * dtype.itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=n)


class World:
    """R simulated ranks, each with a RaFI context of ``cap`` items of ``B`` bytes."""

    def __init__(self, R: int, cap: int, B: int):
        self.R, self.cap, self.B = int(R), int(cap), int(B)
        self._w = lib().orc_create(self.R, self.cap, self.B)
        if not self._w:
            raise MemoryError("orc_create failed")

    def close(self):
        if self._w:
            lib().orc_destroy(self._w)
            self._w = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device interface ------------------------------------------------
    def emit(self, r: int, item: bytes, d: int) -> bool:
        assert len(item) == self.B
        buf = np.frombuffer(bytes(item), np.uint8)
        return bool(lib().orc_emit(self._w, r, _ptr(buf), int(d)))

    def emit_many(self, r: int, items: np.ndarray, dests) -> int:
        """Sequential emits in array order (orc_emit_many); returns the number accepted."""
        items = np.ascontiguousarray(items, dtype=np.uint8).reshape(-1, self.B)
        d = np.ascontiguousarray(dests, dtype=np.int32)
        assert d.size == items.shape[0]
        if d.size == 0:
            return 0
        return int(lib().orc_emit_many(self._w, r, _ptr(items), _ptr(d), d.size))

    def load_snapshot(self, r: int, items: np.ndarray, dests: np.ndarray, ctr: int, invalid: int = 0):
        items = np.ascontiguousarray(items, dtype=np.uint8)
        dests = np.ascontiguousarray(dests, dtype=np.int32)
        rc = lib().orc_load_snapshot(self._w, r, _ptr(items), _ptr(dests), int(ctr), int(invalid))
        if rc != OK:
            raise ValueError("orc_load_snapshot rc=%d" % rc)

    def set_incoming(self, r: int, items: np.ndarray):
        items = np.ascontiguousarray(items, dtype=np.uint8).reshape(-1)
        n = items.size // self.B
        rc = lib().orc_set_incoming(self._w, r, _ptr(items), n)
        if rc != OK:
            raise ValueError("orc_set_incoming rc=%d" % rc)

    def num_incoming(self, r: int) -> int:
        return int(lib().orc_num_incoming(self._w, r))

    def incoming(self, r: int) -> np.ndarray:
        n = self.num_incoming(r)
        return _view(lib().orc_in_ptr(self._w, r), n * self.B, np.uint8).reshape(n, self.B).copy()

    # -- forward ------------------------------------------------------------
    def forward(self, literal: bool = False) -> int:
        f = lib().orc_forward_literal if literal else lib().orc_forward_plain
        return int(f(self._w))

    # -- state / results of the last forward ---------------------------------
    def emitted(self, r):
        return int(lib().orc_emitted(self._w, r))

    def invalid(self, r):
        return int(lib().orc_invalid(self._w, r))

    def dropped_last(self, r):
        return int(lib().orc_dropped_last(self._w, r))

    def invalid_last(self, r):
        return int(lib().orc_invalid_last(self._w, r))

    def out_items(self, r, n=None) -> np.ndarray:
        if n is None:
            n = min(self.emitted(r), self.cap)
        return _view(lib().orc_out_ptr(self._w, r), n * self.B, np.uint8).reshape(n, self.B).copy()

    def out_dests(self, r, n=None) -> np.ndarray:
        if n is None:
            n = min(self.emitted(r), self.cap)
        return _view(lib().orc_dest_ptr(self._w, r), n, np.int32).copy()

    def binned(self, r, n) -> np.ndarray:
        return _view(lib().orc_binned_ptr(self._w, r), n * self.B, np.uint8).reshape(n, self.B).copy()

    def C(self) -> np.ndarray:
        return _view(lib().orc_C_ptr(self._w), self.R * self.R, np.uint64).reshape(self.R, self.R).copy()

    def send_off(self) -> np.ndarray:
        return _view(lib().orc_send_off_ptr(self._w), self.R * self.R, np.uint64).reshape(self.R, self.R).copy()

    def recv_off(self) -> np.ndarray:
        return _view(lib().orc_recv_off_ptr(self._w), self.R * self.R, np.uint64).reshape(self.R, self.R).copy()

    def G(self) -> int:
        return int(lib().orc_G(self._w))

    # -- proxy applications (oracle/proxies.c), CPU twins of the GPU drivers --
    def advect_seed(self, r, n, seed, grid):
        lib().orc_advect_seed(self._w, r, n, seed, *grid)

    def advect_step(self, r, rnd, max_rounds, omega, eps, h, grid):
        lib().orc_advect_step(self._w, r, rnd, max_rounds, omega, eps, h, *grid)

    def march_seed(self, r, n, seed, grid):
        lib().orc_march_seed(self._w, r, n, seed, *grid)

    def march_step(self, r, seed, p_thr, max_bounces, max_steps, grid, result: np.ndarray):
        assert result.dtype == np.float32 and result.flags["C_CONTIGUOUS"]
        lib().orc_march_step(self._w, r, seed, p_thr, max_bounces, max_steps, *grid, result.ctypes.data)


class Digest:
    """Streaming-digest mode (oracle/digest.c): the plain forward's count
    matrix, G and a digest of every incoming queue, from the sources' queues
    fed once in (source, slot) order -- nothing materialised."""

    def __init__(self, R: int, cap: int, B: int):
        self.R, self.cap, self.B = int(R), int(cap), int(B)
        self._g = lib().orc_digest_create(self.R, self.cap, self.B)
        if not self._g:
            raise MemoryError("orc_digest_create failed")

    def close(self):
        if self._g:
            lib().orc_digest_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def feed(self, s: int, items: np.ndarray, dests: np.ndarray):
        items = np.ascontiguousarray(items, dtype=np.uint8)
        dests = np.ascontiguousarray(dests, dtype=np.int32)
        n = dests.size
        assert items.size == n * self.B
        if n == 0:
            return
        rc = lib().orc_digest_feed(self._g, s, _ptr(items), _ptr(dests), n)
        if rc != OK:
            raise ValueError("orc_digest_feed rc=%d" % rc)

    def finish(self) -> int:
        return int(lib().orc_digest_finish(self._g))

    def value(self, d: int) -> int:
        return int(lib().orc_digest_value(self._g, d))

    def C(self) -> np.ndarray:
        return _view(lib().orc_digest_C_ptr(self._g), self.R * self.R, np.uint64).reshape(self.R, self.R).copy()


def digest_items(items: np.ndarray, B: int) -> int:
    """The digest fold of oracle/digest.c applied to a materialised queue."""
    items = np.ascontiguousarray(items, dtype=np.uint8)
    n = items.size // B
    if n == 0:
        return int(lib().orc_digest_items(None, 0, B))
    return int(lib().orc_digest_items(_ptr(items), n, B))


NB_STATS = 42


class NBody:
    """The three-context N-body exchange pattern on R simulated ranks
    (oracle/nbody.c): P (40-B particles), V (24-B virtual particles),
    Q (4-B refinement requests)."""

    def __init__(self, R, cap_p, cap_v, cap_q):
        self.R = R
        self.P, self.V, self.Q = World(R, cap_p, 40), World(R, cap_v, 24), World(R, cap_q, 4)
        self.stats = np.zeros((R, NB_STATS), np.uint64)

    def seed(self, r, n, seed):
        lib().orc_nbody_seed(self.P._w, r, n, seed)

    def migrate(self, dt):
        for r in range(self.R):
            lib().orc_nbody_migrate(self.P._w, r, dt)

    def compute_stats(self):
        for r in range(self.R):
            lib().orc_nbody_stats(self.P._w, r, self.stats[r].ctypes.data)

    def root(self):
        for r in range(self.R):
            lib().orc_nbody_root(self.V._w, r, self.stats[r].ctypes.data)

    def refine(self, theta2):
        for r in range(self.R):
            lib().orc_nbody_refine(self.V._w, self.Q._w, r, self.stats[r].ctypes.data, theta2)

    def respond(self):
        for r in range(self.R):
            lib().orc_nbody_respond(self.Q._w, self.V._w, r, self.stats[r].ctypes.data)


class Streamlines:
    """R simulated ranks advecting particles on a sampled field (oracle/streamlines.c)."""

    def __init__(self, R, cap, field: np.ndarray, grid):
        self.R, self.grid = R, tuple(grid)
        self.field = np.ascontiguousarray(field, dtype=np.float32)
        self.nz, self.ny, self.nx = self.field.shape[:3]
        self.w = World(R, cap, 16)

    def _dims(self):
        return (self.nx, self.ny, self.nz) + self.grid

    def seed(self, r, seeds, id0):
        seeds = np.ascontiguousarray(seeds, dtype=np.float32)
        lib().orc_sl_seed(self.w._w, r, self.field.ctypes.data, *self._dims(), seeds.ctypes.data, seeds.shape[0], id0)

    def step(self, rnd, h, eps, max_steps, rpos, rsteps):
        assert rpos.dtype == np.float32 and rsteps.dtype == np.uint32
        for r in range(self.R):
            lib().orc_sl_step(self.w._w, r, self.field.ctypes.data, *self._dims(), rnd, h, eps, max_steps,
                              rpos.ctypes.data, rsteps.ctypes.data)

    def owner(self, p):
        q = np.ascontiguousarray(p, dtype=np.float32)
        return int(lib().orc_sl_owner(q.ctypes.data, *self._dims()))


def morton_owner(x, y, z, R) -> int:
    return int(lib().orc_morton_owner(x, y, z, R))


def grid_owner(x, y, z, grid) -> int:
    return int(lib().orc_grid_owner(x, y, z, *grid))


def grid_dims(R: int):
    """Brick / macrocell decomposition of [0,1)^3 for R ranks (gx*gy*gz = R)."""
    dims = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2), 16: (4, 2, 2), 32: (4, 4, 2), 64: (4, 4, 4)}
    if R in dims:
        return dims[R]
    return (R, 1, 1)


# -- pipeline pieces of the paper-literal forward, exposed for pinning ------

def pack_keys(dests) -> np.ndarray:
    d = np.ascontiguousarray(dests, dtype=np.int32)
    k = np.zeros(max(d.size, 1), np.uint64)
    lib().orc_pack_keys(_ptr(d), d.size, _ptr(k))
    return k[: d.size]


def radix_sort_keys(keys) -> np.ndarray:
    k = np.array(keys, dtype=np.uint64)
    k = np.ascontiguousarray(k) if k.size else np.zeros(1, np.uint64)
    n = len(keys)
    rc = lib().orc_radix_sort_keys(_ptr(k), n)
    assert rc == OK
    return k[:n]


def sort_and_gather(items: np.ndarray, dests, B: int):
    """pack_keys -> radix sort -> gather: returns (sorted items, sorted dests)."""
    items = np.ascontiguousarray(items, dtype=np.uint8).reshape(-1)
    n = len(dests)
    keys = radix_sort_keys(pack_keys(dests))
    keys = np.ascontiguousarray(keys) if n else np.zeros(1, np.uint64)
    out = np.zeros(max(n * B, 1), np.uint8)
    sd = np.zeros(max(n, 1), np.int32)
    src = items if items.size else np.zeros(1, np.uint8)
    lib().orc_gather(_ptr(src), _ptr(keys), n, B, _ptr(out), _ptr(sd))
    return out[: n * B].reshape(n, B), sd[:n]


def compute_segments(sorted_dests, R: int):
    d = np.ascontiguousarray(sorted_dests, dtype=np.int32)
    d = d if d.size else np.zeros(1, np.int32)
    cnt = np.zeros(R, np.uint64)
    off = np.zeros(R, np.uint64)
    lib().orc_compute_segments(_ptr(d), len(sorted_dests), R, _ptr(cnt), _ptr(off))
    return cnt, off


def alltoall_u64(send: np.ndarray) -> np.ndarray:
    send = np.ascontiguousarray(send, dtype=np.uint64)
    R = send.shape[0]
    recv = np.zeros((R, R), np.uint64)
    lib().orc_alltoall_u64(R, _ptr(send), _ptr(recv))
    return recv


def alltoallv_bytes(sendbufs, scount, sdispl, recvbufs, rdispl):
    """Simulated MPI_Alltoallv over lists of per-rank numpy uint8 buffers."""
    R = len(sendbufs)
    sp = (C.c_void_p * R)(*[b.ctypes.data for b in sendbufs])
    rp = (C.c_void_p * R)(*[b.ctypes.data for b in recvbufs])
    sc = np.ascontiguousarray(scount, dtype=np.uint64)
    sd = np.ascontiguousarray(sdispl, dtype=np.uint64)
    rd = np.ascontiguousarray(rdispl, dtype=np.uint64)
    lib().orc_alltoallv_bytes(R, C.cast(sp, C.c_void_p), _ptr(sc), _ptr(sd), C.cast(rp, C.c_void_p), _ptr(rd))
