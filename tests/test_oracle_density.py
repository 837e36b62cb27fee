"""Pins of the oracle's T1 density statistics (NEXT-1; §III-C1-C2 l.181-206).

SPEC.md l.224-235 examples, a library pin (scipy's KD-tree ball / kNN queries), and the
closed-form statistics example of S:233.
"""
import numpy as np
import pytest
from scipy.spatial import cKDTree

import oracle


def test_spec_examples_local_density():
    # 2 points at distance 0.5, r=1 -> [1, 1]; at distance 2 -> [0, 0]
    assert list(oracle.local_density([[0, 0, 0], [0.5, 0, 0]], 1.0)) == [1, 1]
    assert list(oracle.local_density([[0, 0, 0], [2.0, 0, 0]], 1.0)) == [0, 0]


@pytest.mark.parametrize("seed", [0, 1])
def test_local_density_matches_kdtree(seed):
    # 1000 random points, exact counts (library pin: scipy cKDTree.query_ball_point)
    r = np.random.default_rng(seed)
    pts = np.concatenate([r.normal(0, 0.2, (600, 3)), r.uniform(-2, 2, (400, 3))]).astype(np.float32)
    rad = 0.15
    got = oracle.local_density(pts, rad)
    tree = cKDTree(pts.astype(np.float64))
    ref = np.array([len(tree.query_ball_point(p, rad * (1 - 1e-6))) - 1 for p in pts.astype(np.float64)])
    ref_hi = np.array([len(tree.query_ball_point(p, rad * (1 + 1e-6))) - 1 for p in pts.astype(np.float64)])
    assert ((got >= ref) & (got <= ref_hi)).all()  # equal up to float ties at |q - p| == r
    assert (got == ref).mean() > 0.999


def test_knn_mean_matches_kdtree():
    r = np.random.default_rng(2)
    pts = r.normal(0, 1, (500, 3)).astype(np.float32)
    got = oracle.knn_mean_distance(pts, 8)
    d, _ = cKDTree(pts.astype(np.float64)).query(pts.astype(np.float64), k=9)
    np.testing.assert_allclose(got, d[:, 1:].mean(1), rtol=1e-12)


def test_threshold_statistics_closed_form():
    # densities [1,2,3,4,5], alpha = beta = 1 -> mu 3, sigma sqrt(2)
    s = oracle.density_thresholds([1, 2, 3, 4, 5])
    assert s["mu"] == 3.0 and abs(s["sigma"] - np.sqrt(2)) < 1e-15
    assert abs(s["rho_low"] - (3 - np.sqrt(2))) < 1e-15 and abs(s["rho_high"] - (3 + np.sqrt(2))) < 1e-15
    # all equal -> low == high == d
    s = oracle.density_thresholds([4, 4, 4])
    assert s["rho_low"] == s["rho_high"] == 4.0


def test_contrast_fixture_has_100x_density_contrast():
    # the paper's skew: dense vs sparse regions differ ~100x in local density
    r = np.random.default_rng(3)
    dense = r.uniform(-0.1, 0.1, (1000, 3))
    sparse = r.uniform(-1, 1, (1000, 3)) + np.array([3.0, 0, 0])
    pts = np.concatenate([dense, sparse]).astype(np.float32)
    rho = oracle.local_density(pts, 0.1)
    ratio = rho[:1000].mean() / max(rho[1000:].mean(), 1e-9)
    assert ratio > 100
    s = oracle.density_thresholds(rho)
    assert s["above"] > 0 and s["sigma"] / s["mu"] > 1.0
