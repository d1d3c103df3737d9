"""Pins for oracle/hashmask.py (dropout mask, reading R5)."""
import numpy as np

from oracle.hashmask import keep_mask, keep_threshold, splitmix64

GAMMA = 0x9E3779B97F4A7C15


def test_splitmix64_published_vectors():
    # SplitMix64 reference outputs (Vigna's splitmix64.c): first output from state 0, and the
    # sequence from seed 1234567 -- each call advances the state by the golden gamma.
    assert int(splitmix64(0)) == 0xE220A8397B1DCDAF
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423,
              4593380528125082431, 16408922859458223821]
    s = 1234567
    for e in expect:
        assert int(splitmix64(s)) == e
        s = (s + GAMMA) & (2 ** 64 - 1)


def test_threshold_and_p0():
    assert keep_threshold(0.0) == 0
    assert keep_threshold(0.5) == 1 << 23
    assert keep_threshold(1.0) == 1 << 24
    m = keep_mask(3, 1, 2, 1000, np.arange(100), 17, seed=4, p=0.0)
    assert m.all()


def test_keep_rate_within_4_sigma():
    for p in (0.1, 0.3, 0.5):
        m = keep_mask(2, 2, 4, 50000, np.arange(20000), 64, seed=4, p=p)
        k = m.size
        rate = m.mean()
        sigma = np.sqrt(p * (1 - p) / k)
        assert abs(rate - (1 - p)) < 4 * sigma


def test_mask_keyed_by_gid_not_position():
    # A halo copy of node g (any local position) shares its owner's mask (App. F consistency).
    gids = np.array([5, 17, 99, 3])
    a = keep_mask(7, 2, 3, 200, gids, 9, seed=11, p=0.5)
    b = keep_mask(7, 2, 3, 200, gids[::-1], 9, seed=11, p=0.5)
    assert (a == b[::-1]).all()
    # and differs between iterations and layers
    c = keep_mask(8, 2, 3, 200, gids, 9, seed=11, p=0.5)
    d = keep_mask(7, 3, 3, 200, gids, 9, seed=11, p=0.5)
    assert (a != c).any() and (a != d).any()


def test_mask_key_formula_by_hand():
    # key = ((t*(L+1)+l)*N + gid)*F + col ; keep iff (SplitMix64(key ^ seed) >> 40) >= thr
    t, l, L, N, F, seed, p = 3, 2, 4, 1000, 7, 123, 0.5
    gid, col = 42, 5
    key = ((t * (L + 1) + l) * N + gid) * F + col
    h = int(splitmix64(key ^ seed))
    assert bool(keep_mask(t, l, L, N, [gid], F, seed, p)[0, col]) == ((h >> 40) >= (1 << 23))
