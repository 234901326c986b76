"""Seeded synthetic work-item streams -- the ONE module both the CPU oracle
side and the CUDA side take inputs from.

It holds no forwarding arithmetic (no counting, binning, sorting or exchange):
only a counter-based generator (SplitMix64's finaliser applied to a counter,
Steele, Lea & Flood 2014) and the item/destination recipes of DESIGN.md
"Input recipe".  The same recipes are also implemented, separately, in the GPU
driver kernels (paper_2605_30294_b200/csrc/drivers.cu); tests check the two
agree byte for byte.

Item layout (B >= 16; shorter items are the prefix of this layout):
  bytes 0..3   u32 src rank
  bytes 4..7   u32 round
  bytes 8..15  u64 logical id = (src << 40) | seq
  bytes 16..   u32 words w_k = low32(splitmix64(id ^ (k * GOLDEN))), k = 0,1,..
               (truncated at B)
Destinations (for rank ``src`` of ``R``), h = splitmix64(seed ^ (src<<48) ^
(round<<40) ^ seq):
  uniform      ((h >> 32) * R) >> 32          (multiply-shift)
  self         src
  ring         (src + 1) % R
  all_to_one   target
  round_robin  seq % R
  skewed       self with probability 0.9, else a grid neighbour (cfg4 shape)
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

CONFIG_SEEDS = {i: 0x5EED0000 + i for i in range(1, 6)}


def splitmix64(x) -> np.ndarray:
    """SplitMix64 output for state ``x`` (i.e. mix(x + GOLDEN)); vectorised, wraps mod 2^64."""
    z = np.asarray(x, dtype=np.uint64) + GOLDEN
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def item_ids(src: int, seq0: int, n: int) -> np.ndarray:
    seq = np.arange(seq0, seq0 + n, dtype=np.uint64)
    return (np.uint64(src) << np.uint64(40)) | seq


def make_items(src: int, rnd: int, n: int, B: int, seq0: int = 0, ids: np.ndarray | None = None) -> np.ndarray:
    """(n, B) uint8 array of synthetic items for rank ``src`` in round ``rnd``."""
    if ids is None:
        ids = item_ids(src, seq0, n)
    ids = np.asarray(ids, dtype=np.uint64)
    n = ids.size
    nwords = max(0, (B - 16 + 3) // 4)
    full = np.zeros((n, 16 + 4 * nwords), np.uint8)
    full[:, 0:4] = np.full(n, src, np.uint32).view(np.uint8).reshape(n, 4)
    full[:, 4:8] = np.full(n, rnd, np.uint32).view(np.uint8).reshape(n, 4)
    full[:, 8:16] = ids.view(np.uint8).reshape(n, 8)
    if nwords:
        k = np.arange(nwords, dtype=np.uint64)
        with np.errstate(over="ignore"):
            salt = k * GOLDEN
        w = splitmix64(ids[:, None] ^ salt[None, :]).astype(np.uint32)  # low 32 bits
        full[:, 16:] = np.ascontiguousarray(w).view(np.uint8).reshape(n, 4 * nwords)
    return np.ascontiguousarray(full[:, :B])


def dest_hash(seed: int, src: int, rnd: int, seq: np.ndarray) -> np.ndarray:
    seq = np.asarray(seq, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(src) << np.uint64(48)) ^ (np.uint64(rnd) << np.uint64(40))
    return splitmix64(key ^ seq)


def make_dests(pattern: str, seed: int, src: int, rnd: int, n: int, R: int, seq0: int = 0,
               target: int = 0, invalid_frac: float = 0.0) -> np.ndarray:
    """int32 destination ranks for ``n`` items of rank ``src``."""
    seq = np.arange(seq0, seq0 + n, dtype=np.uint64)
    h = dest_hash(seed, src, rnd, seq)
    if pattern == "uniform":
        with np.errstate(over="ignore"):
            d = (((h >> np.uint64(32)) * np.uint64(R)) >> np.uint64(32)).astype(np.int64)
    elif pattern == "self":
        d = np.full(n, src, np.int64)
    elif pattern == "ring":
        d = np.full(n, (src + 1) % R, np.int64)
    elif pattern == "all_to_one":
        d = np.full(n, target, np.int64)
    elif pattern == "round_robin":
        d = (seq % np.uint64(R)).astype(np.int64)
    elif pattern == "skewed":
        u = (h >> np.uint64(32)).astype(np.uint64)
        stay = u < np.uint64(SKEW_STAY)
        if R == 1:
            nb = np.zeros(n, np.int64)
        else:
            pick = (h & np.uint64(0xFFFF)).astype(np.int64) % (R - 1)
            nb = (src + 1 + pick) % R
        d = np.where(stay, src, nb).astype(np.int64)
    else:
        raise ValueError("unknown pattern %r" % pattern)
    if invalid_frac > 0.0:
        bad = (h & np.uint64(0xFFFFFFFF)) < np.uint64(invalid_threshold(invalid_frac))
        d = np.where(bad, np.where((seq & np.uint64(1)) == 0, -1, R), d)
    return d.astype(np.int32)


def invalid_threshold(frac: float) -> int:
    """Integer threshold on the low 32 bits of h for an invalid-dest fraction."""
    return int(frac * 2**32)


SKEW_STAY = int(0.9 * 2**32)  # 3865470566: P(stay on own rank) in the skewed pattern

PATTERNS = {"uniform": 0, "self": 1, "ring": 2, "all_to_one": 3, "round_robin": 4, "skewed": 5}


def walk_dests(seed: int, rnd: int, ids: np.ndarray, R: int) -> np.ndarray:
    """Random-walk destination of each item id in round ``rnd`` (cfg1 driver):
    multiply-shift of splitmix64(seed ^ (rnd << 40) ^ id)."""
    ids = np.asarray(ids, dtype=np.uint64)
    h = splitmix64(np.uint64(seed) ^ (np.uint64(rnd) << np.uint64(40)) ^ ids)
    with np.errstate(over="ignore"):
        return (((h >> np.uint64(32)) * np.uint64(R)) >> np.uint64(32)).astype(np.int32)


def item_id_of(items: np.ndarray) -> np.ndarray:
    """Logical id (bytes 8..15) of each row of an (n, B>=16) item array."""
    items = np.ascontiguousarray(items, dtype=np.uint8)
    return items[:, 8:16].copy().view(np.uint64).reshape(-1)


def item_src_of(items: np.ndarray) -> np.ndarray:
    items = np.ascontiguousarray(items, dtype=np.uint8)
    return items[:, 0:4].copy().view(np.uint32).reshape(-1)
