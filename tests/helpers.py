"""Small input builders for tests (inputs only: no method arithmetic)."""
import math

import numpy as np

import gen

INV_SQRT_4PI = 1.0 / math.sqrt(4.0 * math.pi)  # value of the l=0 orthonormal SH (math fact)


def gaussians(means, log_scales=None, quats=None, ologits=None, sh=None):
    means = np.asarray(means, np.float32).reshape(-1, 3)
    n = means.shape[0]
    ls = np.full((n, 3), math.log(0.05), np.float32) if log_scales is None else np.asarray(log_scales, np.float32).reshape(n, 3)
    q = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)) if quats is None else np.asarray(quats, np.float32).reshape(n, 4)
    ol = np.zeros(n, np.float32) if ologits is None else np.asarray(ologits, np.float32).reshape(n)
    s = np.zeros((n, 16, 3), np.float32) if sh is None else np.asarray(sh, np.float32).reshape(n, 16, 3)
    return gen.pack(means, ls, q, ol, s), n


def sh_for_rgb(rgb):
    """DC coefficient giving colour rgb at SH degree 0 (rgb = Y_0 * dc + 0.5, R12)."""
    sh = np.zeros((16, 3), np.float32)
    sh[0] = (np.asarray(rgb, np.float64) - 0.5) / INV_SQRT_4PI
    return sh


def axis_camera(W, H, f=None, bg=(0.2, 0.4, 0.6), campos=(0.0, 0.0, 0.0)):
    f = W if f is None else f
    cam = gen.make_camera(np.eye(3), [0, 0, 0], W, H, f, f, bg=bg)
    cam.campos = np.asarray(campos, np.float32)
    return cam


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)
