"""Pins of the NEXT-2 loss oracle (oracle/ssim.py) against closed forms, a library
routine, symmetry and finite differences (no GPU)."""
import numpy as np
import pytest
import scipy.signal

from oracle import ssim as S


def test_window_is_the_normalised_gaussian():
    w = S.window()
    assert w.shape == (11, 11)
    assert abs(w.sum() - 1.0) < 1e-15
    assert np.allclose(w, w.T) and np.allclose(w, w[::-1, ::-1])
    # separable, sigma = 1.5: neighbouring taps differ by exp(-(2k+1) / (2 sigma^2))
    g = w[5] / w[5].sum()
    assert np.allclose(np.outer(g, g), w, rtol=1e-12)
    assert abs(g[6] / g[5] - np.exp(-1.0 / (2 * 1.5 ** 2))) < 1e-14
    assert abs(g[8] / g[5] - np.exp(-9.0 / (2 * 1.5 ** 2))) < 1e-14


def test_correlate_matches_scipy():
    r = np.random.default_rng(0)
    img = r.random((23, 31))
    w = r.random((11, 11))  # a non-symmetric kernel pins the orientation
    ref = scipy.signal.correlate2d(img, w, mode="same", boundary="fill", fillvalue=0.0)
    assert np.allclose(S.correlate(img, w), ref, rtol=1e-12, atol=1e-12)


def test_identical_images_give_one():
    r = np.random.default_rng(1)
    x = r.random((3, 20, 25))
    assert np.allclose(S.ssim_map(x, x), 1.0, atol=1e-12)


def test_constant_images_closed_form_in_the_interior():
    a, b = 0.3, 0.7
    x = np.full((3, 30, 30), a)
    y = np.full((3, 30, 30), b)
    m = S.ssim_map(x, y)
    expect = (2 * a * b + S.C1) / (a * a + b * b + S.C1)  # sigma terms vanish: (C2 / C2)
    assert np.allclose(m[:, 5:-5, 5:-5], expect, rtol=1e-12)
    # zero padding: at the corner the window sees 36 % zeros, so the means shrink
    assert not np.isclose(m[0, 0, 0], expect)


def test_symmetric_and_inverted_structure():
    r = np.random.default_rng(2)
    x, y = r.random((3, 24, 24)), r.random((3, 24, 24))
    assert np.allclose(S.ssim_map(x, y), S.ssim_map(y, x), rtol=1e-13)
    assert S.ssim_map(x, 1.0 - x).mean() < 0.0  # the negative scores below 0


def test_loss_at_the_target_is_zero():
    r = np.random.default_rng(3)
    t = r.integers(0, 256, (3, 16, 18)).astype(np.uint8)
    assert abs(S.loss(t / 255.0, t)) < 1e-12


@pytest.mark.parametrize("lam", [0.2, 0.0, 1.0])
def test_loss_grad_finite_differences(lam):
    r = np.random.default_rng(4)
    t = r.integers(0, 256, (3, 13, 17)).astype(np.uint8)
    y = t / 255.0
    # keep |x - y| away from the L1 kink
    x = np.clip(y + np.where(r.random(y.shape) < 0.5, -1, 1) * r.uniform(0.05, 0.2, y.shape), -0.5, 1.5)
    g = S.loss_grad(x, t, lam)
    h = 1e-6
    idx = [(c, i, j) for c in range(3) for i in (0, 1, 6, 12) for j in (0, 4, 9, 16)]
    for p in idx:
        xp, xm = x.copy(), x.copy()
        xp[p] += h
        xm[p] -= h
        fd = (S.loss(xp, t, lam) - S.loss(xm, t, lam)) / (2 * h)
        assert abs(fd - g[p]) <= 1e-7 * max(1.0, abs(fd)) + 1e-9, (p, fd, g[p])
