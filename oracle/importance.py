"""Oracle for NEXT-3: T2's similarity-based sampling -- colour
quantisation, hash-based grouping into 4096 buckets per 16x16 tile, bucket aggregation and
the per-Gaussian importance score -- and the keep rule NEXT-4's serving uses.  Plain float64
numpy over the C++ oracle's preprocess outputs and rendered image.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/).  Shares no code with
paper_2510_14564_b200/csrc/importance.cu.

Paper: PAPER.md §IV-C1 (l.253-268): c_quant = floor(c / 256 * 16) per 8-bit channel,
hash = R_q * 256 + G_q * 16 + B_q, buckets aggregate colour (average) and opacity (sum) with
a count; §IV-C3 (l.279-284): I_g = (1/N) sum_i similarity(c_g, c_i) alpha_i, "retained for use
during rendering".  Readings (R37-R40):
  R37  a unit-range colour c (clamped to [0, 1]) maps to c8 = min(255, floor(256 c)),
       then c_quant = floor(c8 / 16); key = R_q 256 + G_q 16 + B_q.
  R38  buckets per 16x16 tile over its pixels: key of the pixel's rendered colour; count,
       colour sum (clamped colours), opacity sum (the pixel's accumulated alpha 1 - T_final).
  R39  I_g = (1/N_g) sum over the pixels i of g's tile rect (inside the image) where g's
       blend alpha_g(i) >= 1/255 (R14: power <= 0, alpha = min(0.99, o G)) of
       sim(c_g, c_i) alpha_g(i), sim = 1 - |c_g - c_i|_2 / sqrt(3) with c_g the Gaussian's
       view-dependent colour and c_i the rendered pixel colour (both clamped to [0, 1]);
       N_g = that pixel count; I_g = 0 when N_g = 0.
  R40  keep rule: rank by ascending I_g (ties by index), keep the first
       ceil(f n); `invert` ranks by descending I_g instead (the formula/prose conflict).
"""
from __future__ import annotations

import math

import numpy as np

SQRT3 = math.sqrt(3.0)


def quantize(rgb) -> np.ndarray:
    """R37: [..., 3] unit-range colours -> [..., 3] levels in [0, 15]."""
    c = np.clip(np.asarray(rgb, np.float64), 0.0, 1.0)
    c8 = np.minimum(255, np.floor(c * 256.0)).astype(np.int64)
    return c8 // 16


def hash_key(q) -> np.ndarray:
    q = np.asarray(q, np.int64)
    return q[..., 0] * 256 + q[..., 1] * 16 + q[..., 2]


def tile_buckets(image, final_T, tile=16) -> dict:
    """R38: {(tile_id, key): (count, colour_sum[3], opacity_sum)} over all tiles."""
    img = np.clip(np.asarray(image, np.float64), 0.0, 1.0)
    _, H, W = img.shape
    tx = (W + tile - 1) // tile
    keys = hash_key(quantize(np.moveaxis(img, 0, -1)))
    out = {}
    for y in range(H):
        for x in range(W):
            t = (y // tile) * tx + x // tile
            k = (t, int(keys[y, x]))
            cnt, cs, os_ = out.get(k, (0, np.zeros(3), 0.0))
            out[k] = (cnt + 1, cs + img[:, y, x], os_ + (1.0 - float(final_T[y, x])))
    return out


def importance(pre, image, W, H, tile=16) -> tuple[np.ndarray, np.ndarray]:
    """R39: (I [n], N [n]) from the oracle's preprocess outputs and rendered image."""
    img = np.clip(np.asarray(image, np.float64), 0.0, 1.0)
    n = pre["radius"].shape[0]
    imp = np.zeros(n)
    cnt = np.zeros(n, np.int64)
    ys, xs = np.mgrid[0:H, 0:W]
    for g in np.nonzero(pre["radius"] > 0)[0]:
        x0, y0, x1, y1 = [int(v) for v in pre["rect"][g]]  # tile rect [x0, x1) x [y0, y1)
        px0, px1 = x0 * tile, min(W, x1 * tile)
        py0, py1 = y0 * tile, min(H, y1 * tile)
        if px0 >= px1 or py0 >= py1:
            continue
        X = xs[py0:py1, px0:px1].astype(np.float64)
        Y = ys[py0:py1, px0:px1].astype(np.float64)
        gx, gy = float(pre["xy"][g, 0]), float(pre["xy"][g, 1])
        a, b, c = [float(v) for v in pre["conic"][g]]
        dx, dy = gx - X, gy - Y
        power = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
        alpha = np.minimum(0.99, float(pre["opacity"][g]) * np.exp(power))
        ok = (power <= 0.0) & (alpha >= 1.0 / 255.0)
        if not ok.any():
            continue
        cg = np.clip(pre["rgb"][g].astype(np.float64), 0.0, 1.0)
        ci = img[:, py0:py1, px0:px1]
        dist = np.sqrt(((ci - cg[:, None, None]) ** 2).sum(0))
        sim = 1.0 - dist / SQRT3
        cnt[g] = int(ok.sum())
        imp[g] = float((sim * alpha)[ok].sum()) / cnt[g]
    return imp, cnt


def keep_mask(imp, fraction, invert=False) -> np.ndarray:
    """R40: the first ceil(f n) Gaussians by ascending I_g (ties by index), or descending."""
    n = len(imp)
    order = np.lexsort((np.arange(n), -np.asarray(imp) if invert else np.asarray(imp)))
    keep = np.zeros(n, bool)
    keep[order[:math.ceil(fraction * n)]] = True
    return keep
