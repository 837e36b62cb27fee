"""Pins of the NEXT-3 oracle (oracle/importance.py; §IV-C1/C3) against SPEC.md's
worked examples, exhaustive bijection, a brute-force grouping, closed forms and
a per-pixel loop re-evaluation."""
import math

import numpy as np

import gen
import oracle
from oracle import importance as I


def test_quantize_spec_examples():
    assert I.quantize([1.0, 1.0, 1.0]).tolist() == [15, 15, 15]
    assert I.quantize([0.0, 0.0, 0.0]).tolist() == [0, 0, 0]
    assert I.quantize([200 / 256, 0, 0]).tolist()[0] == 12  # c8 = 200 -> level 12
    assert I.quantize([1.7, -0.2, 0.5]).tolist() == [15, 0, 8]  # clamped to the unit range


def test_hash_is_the_paper_formula_and_a_bijection():
    assert I.hash_key([0, 0, 0]) == 0 and I.hash_key([15, 15, 15]) == 4095 and I.hash_key([1, 2, 3]) == 291
    q = np.stack(np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij"), -1).reshape(-1, 3)
    k = I.hash_key(q)
    assert sorted(k.tolist()) == list(range(4096))
    assert (np.stack([k // 256, (k // 16) % 16, k % 16], -1) == q).all()  # decode(hash(q)) = q


def test_tile_buckets_equal_a_grouping_by_key():
    r = np.random.default_rng(0)
    img = r.random((3, 40, 37)).astype(np.float32) * 1.1
    fT = r.random((40, 37)).astype(np.float32)
    b = I.tile_buckets(img, fT)
    assert sum(v[0] for v in b.values()) == 40 * 37
    # independent grouping: np.unique over (tile, key) and np.add.at sums
    c = np.clip(img.astype(np.float64), 0, 1)
    q = np.minimum(255, np.floor(c * 256)).astype(int) // 16
    key = q[0] * 256 + q[1] * 16 + q[2]
    ys, xs = np.mgrid[0:40, 0:37]
    tid = (ys // 16) * 3 + xs // 16
    pairs = np.stack([tid.ravel(), key.ravel()], 1)
    uniq, inv = np.unique(pairs, axis=0, return_inverse=True)
    cnt = np.zeros(len(uniq), int)
    np.add.at(cnt, inv.ravel(), 1)
    osum = np.zeros(len(uniq))
    np.add.at(osum, inv.ravel(), 1.0 - fT.ravel().astype(np.float64))
    assert len(uniq) == len(b)
    for u, k_, o in zip(uniq, cnt, osum):
        got = b[(int(u[0]), int(u[1]))]
        assert got[0] == k_ and abs(got[2] - o) < 1e-9


def _pre_one(rgb, opacity, conic, xy, rect):
    return dict(radius=np.array([10], np.int32), xy=np.array([xy], np.float32),
                conic=np.array([conic], np.float32), opacity=np.array([opacity], np.float32),
                rgb=np.array([rgb], np.float32), rect=np.array([rect], np.int32))


def test_importance_closed_forms():
    # a Gaussian whose colour equals every covered pixel colour with alpha at its
    # 0.99 clamp everywhere -> I = 0.99 (sim = 1); covering no pixel -> 0
    c = [0.3, 0.6, 0.2]
    img = np.broadcast_to(np.asarray(c, np.float32)[:, None, None], (3, 32, 32)).copy()
    pre = _pre_one(c, 1.0, [1e-9, 0.0, 1e-9], [16.0, 16.0], [0, 0, 2, 2])
    imp, cnt = I.importance(pre, img, 32, 32)
    assert cnt[0] == 32 * 32 and abs(imp[0] - 0.99) < 1e-12
    pre["radius"][0] = 0
    imp, cnt = I.importance(pre, img, 32, 32)
    assert imp[0] == 0.0 and cnt[0] == 0
    # complementary colours: sim = 1 - |c - (1 - c)| / sqrt(3)
    pre["radius"][0] = 10
    imp, _ = I.importance(pre, 1.0 - img, 32, 32)
    d = np.linalg.norm(np.asarray(c) - (1 - np.asarray(c)))
    assert abs(imp[0] - 0.99 * (1 - d / math.sqrt(3))) < 1e-6


def test_importance_equals_a_per_pixel_loop():
    s = gen.small_scene(3, 60, 40, 36)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, s.sh_degree, cam)
    pre = f["pre"]
    imp, cnt = I.importance(pre, f["image"], cam.width, cam.height)
    img = np.clip(f["image"].astype(np.float64), 0, 1)
    for g in np.nonzero(pre["radius"] > 0)[0][:12]:
        x0, y0, x1, y1 = pre["rect"][g]
        tot, k = 0.0, 0
        for y in range(y0 * 16, min(cam.height, y1 * 16)):
            for x in range(x0 * 16, min(cam.width, x1 * 16)):
                dx, dy = float(pre["xy"][g, 0]) - x, float(pre["xy"][g, 1]) - y
                a, b, c = [float(v) for v in pre["conic"][g]]
                power = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
                al = min(0.99, float(pre["opacity"][g]) * math.exp(power))
                if power > 0 or al < 1 / 255:
                    continue
                cg = np.clip(pre["rgb"][g].astype(np.float64), 0, 1)
                tot += (1 - np.linalg.norm(cg - img[:, y, x]) / math.sqrt(3)) * al
                k += 1
        assert cnt[g] == k and abs(imp[g] - (tot / k if k else 0.0)) < 1e-12


def test_keep_mask_rule():
    assert I.keep_mask(np.array([0.5, 0.2, 0.9]), 1.0).all()
    assert I.keep_mask(np.array([0.1, 0.9]), 0.5).tolist() == [True, False]
    assert I.keep_mask(np.array([0.1, 0.9]), 0.5, invert=True).tolist() == [False, True]
    assert I.keep_mask(np.array([0.3, 0.3, 0.3]), 0.5).tolist() == [True, True, False]  # ties by index
    r = np.random.default_rng(1)
    x = r.random(100)
    assert (I.keep_mask(x, 0.37) == I.keep_mask(3.0 * x + 7.0, 0.37)).all()  # rank-based
