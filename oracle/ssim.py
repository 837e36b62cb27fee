"""Oracle for NEXT-2: the 3DGS training loss
    Loss = (1 - lam) * mean|x - y| + lam * (1 - mean SSIM(x, y)),   lam = 0.2,
and its gradient dLoss/dx, in plain float64 numpy.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): imported by tests/ and never by the
product package.  It shares no code with paper_2510_14564_b200/csrc/loss.cu.

Paper basis: SSIM is the paper's quality metric ("PSNR, SSIM [Wang et al. 2004]",
PAPER.md §VI-A l.394); the training loop is inherited from 3DGS (SPEC.md
l.13), whose loss is 0.8 L1 + 0.2 D-SSIM.  SPEC.md l.168-176 states SSIM with an 11x11
Gaussian window.  Readings (R28-R30):
  R28  per-channel SSIM on RGB, averaged over channels and pixels (the 3DGS training loss;
       SPEC's luma SSIM is its CPU program's evaluation metric, not the training loss);
  R29  window: 11x11, separable Gaussian, sigma = 1.5, normalised to sum 1; statistics at
       every pixel with ZERO padding outside the image (3DGS's conv2d(padding=5));
       C1 = 0.01^2, C2 = 0.03^2 (unit data range) [Wang et al. 2004];
  R30  the target is an 8-bit image read as t/255; lam = 0.2; sign(0) = 0 for the L1 term.

Definitions (Wang et al. 2004, eq. 13, with sample statistics taken under the window w):
  mu_x = w * x,  sigma_x^2 = w * x^2 - mu_x^2,  sigma_xy = w * (x y) - mu_x mu_y
  SSIM = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2))
where `*` is the zero-padded 2-D correlation with the 11x11 window, written out below as a
plain sum over the 121 window offsets (no separable shortcut).
"""
from __future__ import annotations

import numpy as np

WIN = 11
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2
LAMBDA = 0.2


def window() -> np.ndarray:
    """R29: the normalised 11x11 Gaussian window, w[i, j] = g_i g_j, g_k ~ exp(-(k-5)^2 / (2 sigma^2))."""
    k = np.arange(WIN, dtype=np.float64) - WIN // 2
    g = np.exp(-(k * k) / (2.0 * SIGMA * SIGMA))
    g /= g.sum()
    return np.outer(g, g)


def correlate(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Zero-padded 'same' 2-D correlation of img[h][w] with the window, as the plain sum
    over window offsets: out[p] = sum_{(i, j)} w[i, j] img[p + (i - 5, j - 5)], img = 0 outside."""
    h, wd = img.shape
    r = WIN // 2
    pad = np.zeros((h + 2 * r, wd + 2 * r))
    pad[r:r + h, r:r + wd] = img
    out = np.zeros((h, wd))
    for i in range(WIN):
        for j in range(WIN):
            out += w[i, j] * pad[i:i + h, j:j + wd]
    return out


def ssim_map(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Per-channel SSIM map (R28): x, y [3][h][w] float64 -> [3][h][w]."""
    w = window()
    out = np.empty_like(x, dtype=np.float64)
    for c in range(x.shape[0]):
        xc, yc = x[c].astype(np.float64), y[c].astype(np.float64)
        mx, my = correlate(xc, w), correlate(yc, w)
        sxx = correlate(xc * xc, w) - mx * mx
        syy = correlate(yc * yc, w) - my * my
        sxy = correlate(xc * yc, w) - mx * my
        out[c] = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sxx + syy + C2))
    return out


def target_float(target_u8: np.ndarray) -> np.ndarray:
    """R30: the 8-bit target as t / 255 (float64)."""
    return target_u8.astype(np.float64) / 255.0


def loss(x: np.ndarray, target_u8: np.ndarray, lam: float = LAMBDA) -> float:
    """Loss = (1 - lam) mean|x - y| + lam (1 - mean SSIM)  (means over all 3 h w values)."""
    y = target_float(target_u8)
    x = x.astype(np.float64)
    return float((1.0 - lam) * np.abs(x - y).mean() + lam * (1.0 - ssim_map(x, y).mean()))


def loss_grad(x: np.ndarray, target_u8: np.ndarray, lam: float = LAMBDA) -> np.ndarray:
    """dLoss/dx [3][h][w] by the chain rule through the window statistics.

    With A1 = 2 mx my + C1, A2 = 2 sxy + C2, B1 = mx^2 + my^2 + C1, B2 = sxx + syy + C2 and
    S = A1 A2 / (B1 B2) at map position p, the partials w.r.t. the raw window moments
    m = w*x, E = w*x^2, P = w*(x y) are
      dS/dE = -S / B2,   dS/dP = 2 A1 / (B1 B2),
      dS/dm = 2 my A2 / (B1 B2) - 2 mx S / B1 + 2 mx S / B2 - 2 my A1 / (B1 B2)
    (the last three terms through B1, sxx and sxy).  Each raw moment at p is sum_q w[q - p]
    f(x_q), so dS_p/dx_q = w[q - p] (dS/dm + 2 x_q dS/dE + y_q dS/dP), and summing over p is
    the correlation with the flipped window (= the window: it is symmetric).
    """
    y = target_float(target_u8)
    x = x.astype(np.float64)
    n = x.size
    w = window()
    g = (1.0 - lam) * np.sign(x - y) / n
    for c in range(x.shape[0]):
        xc, yc = x[c], y[c]
        mx, my = correlate(xc, w), correlate(yc, w)
        sxx = correlate(xc * xc, w) - mx * mx
        syy = correlate(yc * yc, w) - my * my
        sxy = correlate(xc * yc, w) - mx * my
        a1, a2 = 2 * mx * my + C1, 2 * sxy + C2
        b1, b2 = mx * mx + my * my + C1, sxx + syy + C2
        s = a1 * a2 / (b1 * b2)
        d_e = -s / b2
        d_p = 2 * a1 / (b1 * b2)
        d_m = 2 * my * a2 / (b1 * b2) - 2 * mx * s / b1 + 2 * mx * s / b2 - 2 * my * a1 / (b1 * b2)
        wf = w[::-1, ::-1]
        ds_dx = correlate(d_m, wf) + 2 * xc * correlate(d_e, wf) + yc * correlate(d_p, wf)
        g[c] += -lam * ds_dx / n
    return g
