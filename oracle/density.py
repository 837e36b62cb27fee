"""Oracle for NEXT-1's density-control step (§III-C l.181-228):
statistics, merging of dense pairs, densification of sparse points -- plain float64 numpy,
brute force (O(n^2)), for the small fixtures the tests use.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and never by the
product package.  Shares no code with paper_2510_14564_b200/csrc/density.cu; random draws
of the method (the densification's N(0, 1) and U(-1, 1) variates) are inputs.

Readings (R31-R36):
  R31  rho(p) = #{q != p : |q - p| <= r} (the C++ oracle's float decision, orc_local_density);
       rho_low / rho_high = mu -/+ alpha / beta sigma over all rho (population sigma).
  R32  neighbour distances: each point's k = 8 nearest other points (double, ties by index),
       each truncated at 3 r (a neighbour farther than 3 r, or a missing one, counts as 3 r:
       the search stays inside a fixed neighbourhood of the density grid, and an isolated
       point's densification spread stays bounded); d_bar_p = their mean; mu_d,
       sigma_d over all n k truncated distances pooled; d_merge = mu_d + gamma
       sigma_d.
  R33  merge pairing: a point p with rho > rho_high pairs with its nearest other dense point q
       within d_merge (squared distance in double, ties by lower index) when p is also q's
       nearest -- a mutual-nearest-neighbour matching (deterministic and parallel; SPEC's
       greedy ascending-distance order, is sequential).  Pairs are disjoint.
  R34  merged Gaussian (kept at the lower index, the other removed): mean = opacity-weighted
       centroid, scale = component-wise mean of the two scales (in linear
       units), rotation = the higher-opacity member's quaternion (ties: lower index), opacity =
       min(0.999, o_p + o_q) (S:262's clamped sum, capped so the logit stays finite), SH =
       opacity-weighted mean.  Computed in double, rounded once to float.
  R35  densification, round 1: each point with rho < max(rho_low, 0) spawns c = min(max_new,
       ceil(rho_low - rho)) children, child j at p + sigma_p z + delta u with sigma_p =
       alpha_sigma d_bar_p, z ~ N(0, I3), u ~ U(-1, 1)^3, scale,
       rotation, opacity and SH copied from the parent.  Children are numbered in
       (parent index, j) order; z and u are indexed by that number.
  R35' rounds 2 .. max_rounds ("This process is repeated iteratively until the desired
       density is achieved"; until the point's recomputed local density
       >= rho_low or max_rounds): the parents are round 1's sparse points (at their indices
       in the round-1 output, sigma_p and rho_low of the step's statistics kept); each round
       re-counts rho over the whole current scene (children included) and a parent still
       below rho_low spawns min(max_new, ceil(rho_low - rho)) more children, appended in
       (parent, j) order; the loop ends early when no parent is below rho_low.
  R36  output order: survivors in index order (a merged pair's result at the lower index),
       then the children; Adam moments are kept for unmerged survivors and zero for merged
       Gaussians and children.
"""
from __future__ import annotations

import math

import numpy as np

import oracle


def _seg(theta, n):
    t = np.asarray(theta, np.float32)
    return dict(means=t[0:3 * n].reshape(n, 3), log_scales=t[3 * n:6 * n].reshape(n, 3),
                quats=t[6 * n:10 * n].reshape(n, 4), opacity=t[10 * n:11 * n], sh=t[11 * n:59 * n].reshape(n, 48))


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


def sqdist(means):
    """Squared distances in double: ((dx^2 + dy^2) + dz^2) with dx = (double)q - (double)p."""
    m = np.asarray(means, np.float32).astype(np.float64)
    d = m[None, :, :] - m[:, None, :]
    return (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]


def knn(means, k=8):
    """R32: each point's k nearest other points: (dist [n][k] ascending, idx [n][k]); ties by index."""
    d2 = sqdist(means)
    n = d2.shape[0]
    np.fill_diagonal(d2, np.inf)
    kk = min(k, n - 1)
    order = np.lexsort((np.broadcast_to(np.arange(n), d2.shape), d2), axis=1)[:, :kk]
    return np.sqrt(np.take_along_axis(d2, order, 1)), order


def stats(theta, n, r, alpha=1.0, beta=1.0, gamma=1.0, k=8):
    """R31-R32: local densities, thresholds, neighbour-distance statistics and d_merge."""
    s = _seg(theta, n)
    rho = oracle.local_density(s["means"], r).astype(np.int64)
    th = oracle.density_thresholds(rho, alpha, beta)
    dist, _ = knn(s["means"], k)
    cap = 3.0 * float(np.float32(r))
    dist = np.minimum(dist, cap)
    if dist.shape[1] < k:  # fewer than k other points: the missing ones count as 3 r
        dist = np.concatenate([dist, np.full((dist.shape[0], k - dist.shape[1]), cap)], 1)
    mu_d = float(dist.mean())
    sd_d = float(np.sqrt(((dist - mu_d) ** 2).mean()))
    return {"rho": rho, "mu_rho": th["mu"], "sigma_rho": th["sigma"], "rho_low": th["rho_low"],
            "rho_high": th["rho_high"], "d_bar": dist.mean(1), "mu_d": mu_d, "sigma_d": sd_d,
            "d_merge": mu_d + gamma * sd_d}


def merge_pairs(theta, n, st):
    """R33: mutual nearest dense neighbours within d_merge -> sorted list of (p, q), p < q."""
    s = _seg(theta, n)
    dense = st["rho"] > st["rho_high"]
    d2 = sqdist(s["means"])
    lim = st["d_merge"] ** 2
    nn = np.full(n, -1)
    for p in np.nonzero(dense)[0]:
        best, bq = np.inf, -1
        for q in np.nonzero(dense)[0]:
            if q == p or d2[p, q] > lim:
                continue
            if d2[p, q] < best:  # strict: ties keep the lower index (ascending q)
                best, bq = d2[p, q], q
        nn[p] = bq
    return [(p, int(nn[p])) for p in range(n) if nn[p] > p and nn[nn[p]] == p]


def child_counts(st, n, max_new=4):
    """R35: children per point (the densification deficit, capped)."""
    lo = st["rho_low"]
    c = np.zeros(n, np.int64)
    if lo > 0:
        for i in range(n):
            if st["rho"][i] < lo:
                c[i] = min(max_new, math.ceil(lo - st["rho"][i]))
    return c


def merged_gaussian(theta, n, p, q):
    """R34: the merged attributes of pair (p, q) as a float32 [59] row in the
    (mean 3, log_scale 3, quat 4, opacity logit 1, sh 48) order."""
    s = _seg(theta, n)
    op, oq = _sigmoid(s["opacity"][p]), _sigmoid(s["opacity"][q])
    w = op + oq
    mean = (op * s["means"][p].astype(np.float64) + oq * s["means"][q].astype(np.float64)) / w
    scale = 0.5 * (np.exp(s["log_scales"][p].astype(np.float64)) + np.exp(s["log_scales"][q].astype(np.float64)))
    quat = s["quats"][p] if op >= oq else s["quats"][q]
    o = min(0.999, w)
    sh = (op * s["sh"][p].astype(np.float64) + oq * s["sh"][q].astype(np.float64)) / w
    return np.concatenate([mean, np.log(scale), quat.astype(np.float64), [math.log(o / (1.0 - o))], sh]).astype(np.float32)


def apply(theta, m, v, n, st, pairs, counts, normals, uniforms, alpha_sigma=1.5, delta=0.0):
    """R35-R36: the new (theta, m, v, n') in theta's segment layout."""
    s = _seg(theta, n)
    sm, sv = _seg(m, n), _seg(v, n)
    removed = np.zeros(n, bool)
    merged = {}
    for p, q in pairs:
        removed[q] = True
        merged[p] = merged_gaussian(theta, n, p, q)
    rows, mrows, vrows = [], [], []

    def row(seg, i):
        return np.concatenate([seg["means"][i], seg["log_scales"][i], seg["quats"][i], [seg["opacity"][i]], seg["sh"][i]])

    for i in range(n):
        if removed[i]:
            continue
        if i in merged:
            rows.append(merged[i])
            mrows.append(np.zeros(59, np.float32))
            vrows.append(np.zeros(59, np.float32))
        else:
            rows.append(row(s, i))
            mrows.append(row(sm, i))
            vrows.append(row(sv, i))
    c = 0
    for i in range(n):
        sig = alpha_sigma * st["d_bar"][i]
        for _ in range(int(counts[i])):
            base = row(s, i).astype(np.float64)
            pos = s["means"][i].astype(np.float64) + sig * np.asarray(normals[c], np.float64) + \
                delta * np.asarray(uniforms[c], np.float64)
            base[0:3] = pos
            rows.append(base.astype(np.float32))
            mrows.append(np.zeros(59, np.float32))
            vrows.append(np.zeros(59, np.float32))
            c += 1
    nn = len(rows)

    def pack(rs):
        a = np.asarray(rs, np.float32).reshape(nn, 59)
        return np.concatenate([a[:, 0:3].ravel(), a[:, 3:6].ravel(), a[:, 6:10].ravel(), a[:, 10], a[:, 11:59].ravel()])

    return pack(rows), pack(mrows), pack(vrows), nn


def sparse_parents(theta, n, st, pairs, alpha_sigma=1.5):
    """R35': round 1's sparse points (rho < rho_low, rho_low > 0) as (index in apply's
    output, sigma_p) -- sparse points are never merged, so their output index is their rank
    among the survivors."""
    removed = np.zeros(n, bool)
    for _, q in pairs:
        removed[q] = True
    out_idx = np.cumsum(~removed) - 1
    lo = st["rho_low"]
    sel = [i for i in range(n) if lo > 0 and st["rho"][i] < lo]
    return np.asarray([out_idx[i] for i in sel], np.int64), \
        np.asarray([alpha_sigma * st["d_bar"][i] for i in sel], np.float64)


def densify_round(theta, m, v, n, r, parents, sigma, rho_low, normals, uniforms, max_new=4, delta=0.0):
    """R35' one further round on the current scene (theta, m, v of n points): rho of every
    point re-counted at radius r; parent p (index into the scene) below rho_low spawns
    min(max_new, ceil(rho_low - rho_p)) children at p + sigma_p z + delta u, appended after
    the n points in (parent, j) order (zero moments).  Returns (theta', m', v', n', children)."""
    s = _seg(theta, n)
    rho = oracle.local_density(s["means"], r).astype(np.int64)
    counts = [min(max_new, math.ceil(rho_low - rho[p])) if rho[p] < rho_low else 0 for p in parents]
    nc = int(sum(counts))
    if nc == 0:
        return theta, m, v, n, 0
    sm, sv = _seg(m, n), _seg(v, n)

    def rows(seg):
        return [np.concatenate([seg["means"][i], seg["log_scales"][i], seg["quats"][i], [seg["opacity"][i]],
                                seg["sh"][i]]) for i in range(n)]

    R, Mr, Vr = rows(s), rows(sm), rows(sv)
    c = 0
    for p, sg, cnt in zip(parents, sigma, counts):
        for _ in range(cnt):
            base = R[p].astype(np.float64)
            base[0:3] = s["means"][p].astype(np.float64) + sg * np.asarray(normals[c], np.float64) + \
                delta * np.asarray(uniforms[c], np.float64)
            R.append(base.astype(np.float32))
            Mr.append(np.zeros(59, np.float32))
            Vr.append(np.zeros(59, np.float32))
            c += 1
    nn = n + nc

    def pack(rs):
        a = np.asarray(rs, np.float32).reshape(nn, 59)
        return np.concatenate([a[:, 0:3].ravel(), a[:, 3:6].ravel(), a[:, 6:10].ravel(), a[:, 10], a[:, 11:59].ravel()])

    return pack(R), pack(Mr), pack(Vr), nn, nc


def normalized_deviation(means, r):
    """Fig. 5(a) of the paper: sigma_rho / mu_rho."""
    rho = oracle.local_density(means, r).astype(np.float64)
    return float(rho.std() / rho.mean())
