"""Synthetic workload generators (bench/test tooling): determinism and the
statistics SURVEY.md §8(d) quotes for the BASELINE configurations."""

import numpy as np

from oracle import voxsplat_oracle as O
from workloads import scenes


def _solvable_counts(pos, size=0.5, tau=10):
    k = O.keys_of(pos, size)
    _, cnt = np.unique(k, axis=0, return_counts=True)
    return cnt[cnt >= tau]


def test_config1_scan_deterministic_and_shaped():
    a = scenes.config1_scan(seed=0, frame=0)
    b = scenes.config1_scan(seed=0, frame=0)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert 40000 < len(a[0]) <= 60000                   # ~51k hits of 60k rays
    s = _solvable_counts(a[0])
    assert 1000 < len(s) < 2500 and 15 < s.mean() < 35  # SURVEY: 1283 solvable, mean 24


def test_config3_rosette_has_heavy_tail():
    pos, _ = scenes.config3_scan(seed=0, frame=0)
    s = _solvable_counts(pos)
    assert s.max() > 500                                # SURVEY: p99 646, max 742


def test_planar_map_histogram_and_keys():
    pos, col, counts, keys, owner = scenes.planar_map(20000, seed=3)
    assert len(pos) == counts.sum() == len(owner)
    assert counts.min() >= 10 and counts.max() < 160
    frac = np.array([(counts < 16).mean(), ((counts >= 16) & (counts < 32)).mean()])
    assert np.all(np.abs(frac - [0.56, 0.29]) < 0.03)
    k = O.keys_of(pos, 0.5)
    np.testing.assert_array_equal(k, keys[owner])       # every point lies in its voxel
    assert col.min() >= 0 and col.max() <= 1
