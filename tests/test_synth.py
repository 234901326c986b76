"""The shared input generator (synth/) -- pinned to SplitMix64's published
reference stream and to the layout DESIGN.md "Input recipe" states."""
import numpy as np

import synth


def test_splitmix64_reference_stream():
    # SplitMix64 seeded with 0: state advances by GOLDEN before each output
    # (Steele, Lea & Flood 2014 / Vigna's splitmix64.c reference outputs).
    exp = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    with np.errstate(over="ignore"):
        states = np.arange(4, dtype=np.uint64) * synth.GOLDEN
    assert [int(v) for v in synth.splitmix64(states)] == exp


def test_item_layout():
    it = synth.make_items(3, 5, 4, 48, seq0=10)
    assert it.shape == (4, 48)
    assert list(it[:, 0:4].copy().view(np.uint32).ravel()) == [3] * 4
    assert list(it[:, 4:8].copy().view(np.uint32).ravel()) == [5] * 4
    ids = synth.item_id_of(it)
    assert [int(i) for i in ids] == [(3 << 40) | s for s in range(10, 14)]
    # short items are the prefix of the long layout
    assert np.array_equal(synth.make_items(3, 5, 4, 44, seq0=10), it[:, :44])
    assert np.array_equal(synth.make_items(3, 5, 4, 8, seq0=10), it[:, :8])


def test_dest_patterns_in_range():
    for R in (1, 2, 3, 8):
        for p in ("uniform", "self", "ring", "round_robin", "skewed", "all_to_one"):
            d = synth.make_dests(p, 1, min(1, R - 1), 0, 5000, R)
            assert d.dtype == np.int32 and d.min() >= 0 and d.max() < R
    d = synth.make_dests("uniform", 1, 0, 0, 80000, 8)
    c = np.bincount(d, minlength=8)
    assert c.min() > 9000 and c.max() < 11000          # roughly uniform
    d = synth.make_dests("uniform", 1, 0, 0, 10000, 4, invalid_frac=0.1)
    bad = (d < 0) | (d >= 4)
    assert 800 < bad.sum() < 1200
