"""Pins of the NEXT-1 density-control oracle (oracle/density.py; §III-C l.181-228)
against SPEC.md's worked examples, a library (scipy cKDTree) and invariants.  The paper's
deviation outcome (Fig. 5(a)) is measured, not reproduced: see the last test."""
import math

import numpy as np
import pytest
from scipy.spatial import cKDTree

import gen
import oracle
from oracle import density as D


def _theta(means, logit=0.0, seed=0):
    """theta[59n] with the given means, unit-ish scales, random quats/SH, a fixed opacity logit."""
    r = np.random.default_rng(seed)
    m = np.asarray(means, np.float32).reshape(-1, 3)
    n = m.shape[0]
    ls = np.full((n, 3), np.log(0.01), np.float32) + r.normal(0, 0.1, (n, 3)).astype(np.float32)
    q = r.normal(0, 1, (n, 4)).astype(np.float32)
    op = np.broadcast_to(np.asarray(logit, np.float32), (n,)).astype(np.float32)
    sh = r.normal(0, 0.2, (n, 48)).astype(np.float32)
    return np.concatenate([m.ravel(), ls.ravel(), q.ravel(), op, sh.ravel()]).astype(np.float32), n


def test_stats_spec_example():
    # densities [1..5], alpha = beta = 1 -> mu 3, sigma sqrt(2)
    th = oracle.density_thresholds([1, 2, 3, 4, 5])
    assert th["mu"] == 3.0 and abs(th["sigma"] - math.sqrt(2.0)) < 1e-15
    assert abs(th["rho_low"] - (3 - math.sqrt(2))) < 1e-15 and abs(th["rho_high"] - (3 + math.sqrt(2))) < 1e-15


def test_knn_matches_kdtree():
    r = np.random.default_rng(1)
    pts = r.normal(0, 1, (400, 3)).astype(np.float32)
    dist, idx = D.knn(pts, 8)
    d, i = cKDTree(pts.astype(np.float64)).query(pts.astype(np.float64), k=9)
    np.testing.assert_allclose(dist, d[:, 1:], rtol=1e-12)
    assert (idx == i[:, 1:]).mean() > 0.999  # identical up to exact distance ties
    th, n = _theta(pts)
    st = D.stats(th, n, r=1.2)  # 3 r = 3.6 exceeds every 8-NN distance of this cloud
    assert d[:, 1:].max() < 3.6
    assert abs(st["mu_d"] - d[:, 1:].mean()) < 1e-12
    assert abs(st["d_merge"] - (st["mu_d"] + st["sigma_d"])) < 1e-15  # gamma = 1
    np.testing.assert_allclose(st["d_bar"], oracle.knn_mean_distance(pts, 8), rtol=1e-12)
    # R32's truncation at 3 r (r = 0.2: many 8-NN distances exceed 0.6)
    st2 = D.stats(th, n, r=0.2)
    cap = 3 * float(np.float32(0.2))
    dt = np.minimum(d[:, 1:], cap)
    assert (d[:, 1:] > cap).any()
    np.testing.assert_allclose(st2["d_bar"], dt.mean(1), rtol=1e-12)
    assert abs(st2["mu_d"] - dt.mean()) < 1e-12


def test_merged_gaussian_spec_example():
    # p1 = (0,0,0) w = 1, p2 = (2,0,0) w = 3 -> merged at (1.5, 0, 0)
    th, n = _theta([[0, 0, 0], [2, 0, 0]])
    th[10 * n + 0] = math.log(0.2 / 0.8)  # opacity 0.2
    th[10 * n + 1] = math.log(0.6 / 0.4)  # opacity 0.6 (3x)
    row = D.merged_gaussian(th, n, 0, 1).astype(np.float64)
    np.testing.assert_allclose(row[0:3], [1.5, 0, 0], atol=1e-6)
    s = np.exp(th[3 * n:6 * n].reshape(n, 3).astype(np.float64))
    np.testing.assert_allclose(np.exp(row[3:6]), 0.5 * (s[0] + s[1]), rtol=1e-6)
    np.testing.assert_array_equal(row[6:10], th[6 * n + 4:6 * n + 8])  # higher opacity's quaternion
    assert abs(1 / (1 + math.exp(-row[10])) - 0.8) < 1e-6  # clamped sum 0.2 + 0.6
    sh = th[11 * n:].reshape(n, 48).astype(np.float64)
    np.testing.assert_allclose(row[11:], (0.2 * sh[0] + 0.6 * sh[1]) / 0.8, atol=1e-6)


def _clustered(seed, n_dense=600, n_sparse=60):
    r = np.random.default_rng(seed)
    dense = r.normal(0, 0.05, (n_dense, 3))
    sparse = r.uniform(-1.5, 1.5, (n_sparse, 3))
    return np.concatenate([dense, sparse]).astype(np.float32)


def test_merge_pairs_are_mutual_nearest_dense_neighbours():
    pts = _clustered(3)
    th, n = _theta(pts)
    st = D.stats(th, n, r=0.05)
    pairs = D.merge_pairs(th, n, st)
    assert pairs, "the fixture has dense pairs"
    used = [i for pq in pairs for i in pq]
    assert len(used) == len(set(used))  # disjoint
    dense = np.nonzero(st["rho"] > st["rho_high"])[0]
    tree = cKDTree(pts[dense].astype(np.float64))
    d, j = tree.query(pts[dense].astype(np.float64), k=2)  # library pin of the nearest dense neighbour
    nn = {int(dense[a]): (int(dense[j[a, 1]]), d[a, 1]) for a in range(len(dense))}
    want = sorted((p, q) for p, (q, dd) in nn.items()
                  if p < q and dd <= st["d_merge"] and nn[q][0] == p)
    assert sorted(pairs) == want


def test_no_op_cases():
    r = np.random.default_rng(4)
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3), -1).reshape(-1, 3) * 0.1  # a uniform lattice
    th, n = _theta(g + r.normal(0, 1e-4, g.shape))
    st = D.stats(th, n, r=0.1001)
    interior = st["rho"] == st["rho"].max()
    assert interior.any()
    c = D.child_counts(st, n)
    # on a lattice only boundary points are below mu - sigma; nothing in the interior spawns
    assert (c[interior] == 0).all()
    th2, n2 = _theta([[0, 0, 0], [5, 5, 5]])  # two far points: rho = 0 everywhere
    st2 = D.stats(th2, n2, r=0.1)
    assert D.merge_pairs(th2, n2, st2) == [] and (D.child_counts(st2, n2) == 0).all()


def test_apply_counts_positions_and_moments():
    pts = _clustered(5)
    th, n = _theta(pts, seed=5)
    m = np.random.default_rng(6).normal(0, 1, 59 * n).astype(np.float32)
    st = D.stats(th, n, r=0.05)
    pairs = D.merge_pairs(th, n, st)
    c = D.child_counts(st, n)
    z = gen.rng(7).standard_normal((int(c.sum()), 3))
    u = gen.rng(8).uniform(-1, 1, (int(c.sum()), 3))
    th2, m2, v2, n2 = D.apply(th, m, m, n, st, pairs, c, z, u, alpha_sigma=1.5, delta=0.005)
    assert n2 == n - len(pairs) + int(c.sum())
    s2 = D._seg(th2, n2)
    removed = {q for _, q in pairs}
    surv = [i for i in range(n) if i not in removed]
    for k, i in enumerate(surv):  # merged means lie on the segment between the members
        if i in dict(pairs):
            q = dict(pairs)[i]
            a, b, x = pts[i].astype(np.float64), pts[q].astype(np.float64), s2["means"][k].astype(np.float64)
            t = np.dot(x - a, b - a) / np.dot(b - a, b - a)
            assert -1e-5 <= t <= 1 + 1e-5 and np.linalg.norm(a + t * (b - a) - x) < 1e-5
            assert not D._seg(m2, n2)["means"][k].any()
        else:
            np.testing.assert_array_equal(s2["means"][k], pts[i])
            np.testing.assert_array_equal(D._seg(m2, n2)["sh"][k], D._seg(m, n)["sh"][i])
    # children: parent + alpha_sigma d_bar z + delta u, in (parent, j) order
    kk = len(surv)
    for i in np.nonzero(c)[0]:
        for _ in range(c[i]):
            want = pts[i].astype(np.float64) + 1.5 * st["d_bar"][i] * z[kk - len(surv)] + 0.005 * u[kk - len(surv)]
            np.testing.assert_allclose(s2["means"][kk], want, rtol=1e-6, atol=1e-7)
            kk += 1
    th3, _, _, n3 = D.apply(th, m, m, n, st, pairs, c, z, u, alpha_sigma=1.5, delta=0.005)
    assert n3 == n2 and np.array_equal(th3, th2)  # deterministic


def test_merging_thins_the_dense_region_on_a_100x_contrast_fixture():
    # 100x density contrast (SPEC.md l.268's fixture shape, scaled to the brute-force
    # oracle): one merge pass (no densification) lowers the number of points above rho_high
    # and never touches the sparse region.  The paper's Fig. 5(a) outcome (normalized
    # deviation down to 51 %) is NOT reproduced by readings R31-R36 on this fixture:
    # the alpha_sigma > 1 spread scatters children beyond r (measured: 0.42 -> 0.51 after
    # one full step) -- recorded as parity unpinned in DESIGN.md.
    r = np.random.default_rng(9)
    dense = r.uniform(0, 1, (2500, 3))
    sparse = r.uniform(0, 1, (25, 3)) + np.array([1.5, 0, 0])
    pts = np.concatenate([dense, sparse]).astype(np.float32)
    th, n = _theta(pts, seed=9)
    r_d = float(np.median(D.knn(pts, 8)[0][:, -1]))  # r = median 8-NN distance
    st = D.stats(th, n, r=r_d)
    pairs = D.merge_pairs(th, n, st)
    assert pairs and all(q < 2500 for _, q in pairs)
    c0 = np.zeros(n, np.int64)
    th2, _, _, n2 = D.apply(th, np.zeros_like(th), np.zeros_like(th), n, st, pairs, c0, [], [])
    rho2 = oracle.local_density(D._seg(th2, n2)["means"], r_d)
    assert n2 == n - len(pairs)
    assert (rho2 > st["rho_high"]).sum() < (st["rho"] > st["rho_high"]).sum()
    c = D.child_counts(st, n)
    assert (c[2500:] > 0).all()  # every sparse point is below rho_low and spawns


def test_densify_rounds_reach_the_desired_density_spec_example():
    """SPEC.md l.250's example for the iterated densification (R35'): a single isolated point
    with rho_low = 2 and enough rounds ends with >= 2 neighbours within r; with one child per
    round and children within r that takes exactly two rounds, and a third round spawns
    nothing (the desired density is achieved)."""
    pts = np.zeros((1, 3), np.float32)
    th, n = _theta(pts, seed=3)
    m = np.zeros_like(th)
    r = 1.0
    z = np.array([[0.1, 0.0, 0.0]])
    counts = []
    for t in range(3):
        th, m, m2, n, kc = D.densify_round(th, m, m, n, r, np.array([0]), np.array([1.0]), 2.0,
                                           z * (t + 1), np.zeros((1, 3)), max_new=1, delta=0.0)
        counts.append(kc)
    assert counts == [1, 1, 0] and n == 3
    mu = D._seg(th, n)["means"]
    assert np.allclose(mu[1], [0.1, 0, 0]) and np.allclose(mu[2], [0.2, 0, 0])  # p + sigma z, exact
    assert oracle.local_density(mu, r)[0] >= 2
    assert not m.any()  # children have zero Adam moments


def test_densify_round_appends_in_parent_order_and_keeps_the_scene():
    """R35': the n points are unchanged (moments kept), children follow in (parent, j) order
    with the parent's attributes; parents at or above rho_low spawn nothing."""
    r = np.random.default_rng(5)
    pts = np.concatenate([r.uniform(0, 0.2, (40, 3)), [[5.0, 5.0, 5.0], [-5.0, 0.0, 0.0]]]).astype(np.float32)
    th, n = _theta(pts, seed=5)
    m = r.normal(0, 1, th.shape).astype(np.float32)
    parents = np.array([40, 41, 0])  # two isolated points and one inside the cluster
    rho = oracle.local_density(pts, 0.05)
    lo = 0.5 * (rho[0] + 1) if rho[0] > 0 else 0.5  # parent 0 is at or above it
    lo = min(lo, float(rho[0]))
    z = r.normal(0, 1, (8, 3))
    th2, m2, _, n2, kc = D.densify_round(th, m, m, n, 0.05, parents, np.array([0.01, 0.02, 0.03]), max(lo, 1.0),
                                         z, np.zeros((8, 3)), max_new=3, delta=0.0)
    c40 = min(3, math.ceil(max(lo, 1.0) - rho[40]))
    c41 = min(3, math.ceil(max(lo, 1.0) - rho[41]))
    c0 = min(3, math.ceil(max(lo, 1.0) - rho[0])) if rho[0] < max(lo, 1.0) else 0
    assert kc == c40 + c41 + c0 and n2 == n + kc
    s1, s2 = D._seg(th, n), D._seg(th2, n2)
    for key in ("means", "log_scales", "quats", "opacity", "sh"):
        assert np.array_equal(s2[key][:n], s1[key][:n])
    assert np.array_equal(D._seg(m2, n2)["sh"][:n], D._seg(m, n)["sh"])
    assert np.allclose(s2["means"][n], pts[40] + 0.01 * z[0]) and np.array_equal(s2["sh"][n], s1["sh"][40])
    assert np.allclose(s2["means"][n + c40], pts[41] + 0.02 * z[c40])
