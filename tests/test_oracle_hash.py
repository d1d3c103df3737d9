"""Pins for oracle/hashmask.py (dropout mask, reading R5)."""
import numpy as np

from oracle.hashmask import dropout, keep_mask, keep_threshold, splitmix64

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


def test_masks_of_different_iterations_and_layers_are_independent():
    # R5 keys every (t, l, gid, col) to its own counter; masks of two different (t, l) on the same rows
    # must agree as often as two independent Bernoulli(1-p) draws: p^2 + (1-p)^2, within 4 sigma (a key
    # collision between layers or iterations -- e.g. a dropped (L+1) or N factor -- shows up as ~100%)
    p, n, F = 0.3, 20000, 50
    base = keep_mask(5, 2, 3, 40000, np.arange(n), F, seed=9, p=p)
    q = p * p + (1 - p) * (1 - p)
    sigma = np.sqrt(q * (1 - q) / base.size)
    for t, l in ((6, 2), (5, 3), (5, 1), (4, 2)):
        other = keep_mask(t, l, 3, 40000, np.arange(n), F, seed=9, p=p)
        assert abs((base == other).mean() - q) < 4 * sigma, (t, l)
    # neighbouring rows and columns of one mask are independent too (no shared key between (g, F-1)
    # and (g+1, 0) beyond the formula's contiguity): agreement of column c with column c+1
    agree = (base[:, :-1] == base[:, 1:]).mean()
    sigma2 = np.sqrt(q * (1 - q) / base[:, 1:].size)
    assert abs(agree - q) < 4 * sigma2


def test_dropout_preserves_the_mean():
    # PAPER.md:983 applies standard (inverted) dropout: E[D] = H, i.e. the kept entries are scaled by
    # 1/(1-p).  With H = 1 the sample mean of D must be 1 within 4 sigma (sigma^2 = p/((1-p) n)); a
    # missing scale (mean 1-p) or a 1/p scale (mean (1-p)/p) fails.
    for p in (0.1, 0.3, 0.5):
        n, F = 20000, 40
        H = np.ones((n, F))
        D, keep = dropout(H, 3, 2, 3, 50000, np.arange(n), seed=4, p=p)
        sigma = np.sqrt(p / ((1 - p) * H.size))
        assert abs(D.mean() - 1.0) < 4 * sigma, p
        assert np.all(D[keep] == 1.0 / (1.0 - p)) and np.all(D[~keep] == 0.0)
