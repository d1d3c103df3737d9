"""Dropout mask of the oracle -- test infrastructure only (see oracle/__init__.py).

PAPER.md:983 (App. F) requires dropout to be applied *after* communication, with
the same mask for the input tensor and its gradient.  The paper does not define
the random stream, so DESIGN.md reading R5 fixes a counter-based one that both
the oracle and the CUDA path implement independently:

    key  = ((t * (L + 1) + l) * N + gid) * F + col            (uint64, wrapping)
    h    = SplitMix64(key XOR seed)
    keep = (h >> 40) >= floor(p * 2^24 + 0.5)
    D    = H * keep / (1 - p)

with t the iteration, l the layer whose *input* is dropped, N the global node
count, gid the global node id, F = F_{l-1} the true (unpadded) width.  Keying by
global id makes an owner row and every halo copy of it share one mask.

SplitMix64 (Steele, Lea, Flood 2014; public-domain reference by S. Vigna) is the
mixing step; its published outputs are pinned in tests/test_oracle_hash.py.
"""
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """SplitMix64 output for state x (one step: x += golden gamma; mix)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def keep_threshold(p: float) -> int:
    return int(np.floor(p * 16777216.0 + 0.5))


def keep_mask(t: int, layer: int, n_layers: int, n_global: int, gids, width: int, seed: int,
              p: float) -> np.ndarray:
    """Boolean keep mask [len(gids), width] for the input of `layer` at iteration t."""
    gids = np.asarray(gids, dtype=np.uint64)
    if p <= 0.0:
        return np.ones((gids.size, width), dtype=bool)
    with np.errstate(over="ignore"):
        base = (np.uint64(t) * np.uint64(n_layers + 1) + np.uint64(layer)) * np.uint64(n_global)
        key = (base + gids)[:, None] * np.uint64(width) + np.arange(width, dtype=np.uint64)[None, :]
    h = splitmix64(key ^ np.uint64(seed))
    return (h >> np.uint64(40)) >= np.uint64(keep_threshold(p))


def dropout(H: np.ndarray, t: int, layer: int, n_layers: int, n_global: int, gids, seed: int,
            p: float):
    """(D, keep) with D = H * keep / (1 - p) in float64."""
    keep = keep_mask(t, layer, n_layers, n_global, gids, H.shape[1], seed, p)
    scale = 1.0 / (1.0 - p) if p > 0 else 1.0
    return H * keep * scale, keep
