"""Pins of the oracle's preprocess (O1-O9) against closed forms and invariants.

Each test names the passage it pins: PAPER.md l.128-142 (§II-A: G(x), Sigma' =
J W Sigma W^T J^T), SPEC.md l.138-140 / l.182 examples and properties, and the
readings R1-R12 of DESIGN.md §3.
"""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import INV_SQRT_4PI, axis_camera, gaussians


def conic_to_cov(conic):
    cx, cy, cz = (float(v) for v in conic)
    m = np.array([[cx, cy], [cy, cz]], np.float64)
    return np.linalg.inv(m)


def test_on_axis_projects_to_principal_point():
    # W = I, mu = (0,0,2) -> centre at the principal point; R1: ((W-1)/2, (H-1)/2)
    for W, H in [(128, 128), (97, 64), (1237, 822)]:
        th, n = gaussians([[0, 0, 2.0]])
        pre = oracle.preprocess(th, n, 0, axis_camera(W, H))
        assert pre["radius"][0] > 0
        assert pre["xy"][0, 0] == (W - 1) / 2 and pre["xy"][0, 1] == (H - 1) / 2


def test_off_axis_pixel_hand_computed():
    # pinhole: x_pix = ((x / (z tan_fovx) + 1) W - 1) / 2  (R1, R2)
    W, H, f = 160, 96, 140.0
    cam = axis_camera(W, H, f)
    pts = np.array([[0.3, -0.2, 2.5], [-0.7, 0.4, 3.1], [0.05, 0.01, 0.9]])
    th, n = gaussians(pts)
    pre = oracle.preprocess(th, n, 0, cam)
    for i, (x, y, z) in enumerate(pts):
        ex = ((x / (z * W / (2 * f)) + 1) * W - 1) / 2
        ey = ((y / (z * H / (2 * f)) + 1) * H - 1) / 2
        assert abs(pre["xy"][i, 0] - ex) < 2e-4 and abs(pre["xy"][i, 1] - ey) < 2e-4


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_isotropic_closed_form_any_rotation(seed):
    # S:138 (+R8 low-pass): on-axis isotropic s at depth z: Sigma' = ((f s / z)^2 + 0.3) I,
    # invariant under any rotation; R10: r = ceil(3 sqrt(a + sqrt(0.1)))
    r = np.random.default_rng(seed)
    W = H = 128
    f = 128.0
    z = float(r.uniform(1.5, 5.0))
    s = float(r.uniform(0.01, 0.2))
    q = r.standard_normal(4)
    th, n = gaussians([[0, 0, z]], log_scales=[[math.log(s)] * 3], quats=[q])
    pre = oracle.preprocess(th, n, 0, axis_camera(W, H, f))
    a = (f * s / z) ** 2 + 0.3
    cov = conic_to_cov(pre["conic"][0])
    assert abs(cov[0, 0] - a) / a < 1e-5 and abs(cov[1, 1] - a) / a < 1e-5
    assert abs(cov[0, 1]) / a < 1e-5
    np.testing.assert_allclose(pre["conic"][0], [1 / a, 0, 1 / a], rtol=2e-6, atol=2e-6 / a)
    rr = 3 * math.sqrt(a + math.sqrt(0.1))
    if abs(rr - round(rr)) > 1e-3:
        assert pre["radius"][0] == math.ceil(rr)


def test_axis_aligned_and_quarter_turn_swap():
    # R6: q = (1,0,0,0) -> Sigma = diag(s^2); a 90-degree turn about z swaps s_x and s_y
    W = H = 96
    f = 100.0
    z = 3.0
    s = np.array([0.05, 0.11, 0.02])
    c = math.cos(math.pi / 4)
    th, n = gaussians([[0, 0, z]] * 2, log_scales=[np.log(s)] * 2, quats=[[1, 0, 0, 0], [c, 0, 0, c]])
    pre = oracle.preprocess(th, n, 0, axis_camera(W, H, f))
    cov0 = conic_to_cov(pre["conic"][0])
    cov1 = conic_to_cov(pre["conic"][1])
    ex = [(f * s[0] / z) ** 2 + 0.3, (f * s[1] / z) ** 2 + 0.3]
    np.testing.assert_allclose([cov0[0, 0], cov0[1, 1]], ex, rtol=1e-5)
    np.testing.assert_allclose([cov1[0, 0], cov1[1, 1]], ex[::-1], rtol=1e-5)


def test_opacity_and_scale_activations():
    # R5: o = sigmoid(logit)
    lg = np.array([-6.0, -1.0, 0.0, 0.5, 3.0, 9.0], np.float32)
    th, n = gaussians([[0, 0, 2.0]] * 6, ologits=lg)
    # R10's square rect: o < 1/255 (logit -6) blends nowhere and R11' would cull it
    pre = oracle.preprocess(th, n, 0, axis_camera(64, 64), mode=oracle.SQUARE_RECT)
    np.testing.assert_allclose(pre["opacity"], 1 / (1 + np.exp(-lg.astype(np.float64))), rtol=1e-7)
    assert pre["opacity"][2] == 0.5


def test_near_cull():
    # R3 / S:139: cull iff t_z <= near (0.2); t_z = 0.2 exactly is culled
    th, n = gaussians([[0, 0, 0.2], [0, 0, 0.21], [0, 0, -1.0], [0, 0, 0.0]], log_scales=[[math.log(0.01)] * 3] * 4)
    pre = oracle.preprocess(th, n, 0, axis_camera(64, 64))
    assert list(pre["radius"] > 0) == [False, True, False, False]
    assert list(pre["tiles_touched"] > 0) == [False, True, False, False]


def test_focal_doubling():
    # doubling focal doubles centre offsets and quadruples cov2d (here Sigma' - 0.3 I, R8)
    W, H = 128, 96
    r = np.random.default_rng(7)
    pts = np.array([[0.1, -0.05, 2.0], [-0.2, 0.1, 3.0], [0.0, 0.0, 2.5]])
    ls = np.log(r.uniform(0.02, 0.06, size=(3, 3)))
    q = r.standard_normal((3, 4))
    th, n = gaussians(pts, log_scales=ls, quats=q)
    a = oracle.preprocess(th, n, 0, axis_camera(W, H, 60.0))
    b = oracle.preprocess(th, n, 0, axis_camera(W, H, 120.0))
    c = np.array([(W - 1) / 2, (H - 1) / 2])
    off_a, off_b = a["xy"] - c, b["xy"] - c
    mask = np.abs(off_a) > 1e-3
    np.testing.assert_allclose(off_b[mask], 2 * off_a[mask], rtol=1e-5)
    for i in range(3):
        ca = conic_to_cov(a["conic"][i]) - 0.3 * np.eye(2)
        cb = conic_to_cov(b["conic"][i]) - 0.3 * np.eye(2)
        np.testing.assert_allclose(cb, 4 * ca, rtol=1e-4, atol=1e-4 * np.abs(ca).max())


def test_jacobian_clamp_branch():
    # R7: t_x / t_z clamped to +-1.3 tan_fovx; hand-evaluated J at the clamp
    W = H = 64
    f = 64.0
    tan = W / (2 * f)
    mu = [3.0, 0.0, 2.0]
    s = 2.0
    th, n = gaussians([mu], log_scales=[[math.log(s)] * 3])
    pre = oracle.preprocess(th, n, 0, axis_camera(W, H, f))
    assert pre["radius"][0] > 0
    assert pre["cbits"][0] & oracle.CB_JX and not pre["cbits"][0] & oracle.CB_JX_NEG
    z = mu[2]
    tpx = 1.3 * tan * z
    j00, j02, j11 = f / z, -f * tpx / z ** 2, f / z
    a = s * s * (j00 ** 2 + j02 ** 2) + 0.3
    c = s * s * j11 ** 2 + 0.3
    cov = conic_to_cov(pre["conic"][0])
    np.testing.assert_allclose([cov[0, 0], cov[1, 1]], [a, c], rtol=2e-5)
    assert abs(cov[0, 1]) < 1e-4 * a
    # and without the clamp (mode bit) the unclamped Jacobian is used
    pre2 = oracle.preprocess(th, n, 0, axis_camera(W, H, f), mode=oracle.NO_JCLAMP)
    j02u = -f * mu[0] / z ** 2
    a2 = s * s * (j00 ** 2 + j02u ** 2) + 0.3
    np.testing.assert_allclose(conic_to_cov(pre2["conic"][0])[0, 0], a2, rtol=2e-5)


def test_sh_degree0_value_and_direction_independence():
    # O9 / R12: rgb = Y_0 dc + 0.5 with Y_0 = 1/sqrt(4 pi) (orthonormal l=0 harmonic)
    sh = np.zeros((3, 16, 3), np.float32)
    sh[:, 0, :] = [[0.3, -0.2, 1.0]] * 3
    th, n = gaussians([[0, 0, 2.0], [0.4, 0.3, 3.0], [-0.5, 0.1, 2.2]], sh=sh)
    for deg in (0, 3):
        pre = oracle.preprocess(th, n, deg, axis_camera(64, 64))
        np.testing.assert_allclose(pre["rgb"], np.tile(0.5 + INV_SQRT_4PI * np.array([0.3, -0.2, 1.0]), (3, 1)),
                                   rtol=1e-6)


def _basis_values(dirs):
    """Y_k(d) for k < 16 read through the oracle: one Gaussian per k with a one-hot 0.1 coefficient,
    the camera position placed so that the view direction is d (campos is an independent input)."""
    mu = np.array([0.0, 0.0, 2.0])
    out = np.zeros((len(dirs), 16))
    sh = np.zeros((16, 16, 3), np.float32)
    for k in range(16):
        sh[k, k, 0] = 0.1
    th, n = gaussians([mu] * 16, sh=sh)
    for j, d in enumerate(dirs):
        cam = axis_camera(64, 64, campos=mu - d)
        pre = oracle.preprocess(th, n, 3, cam)
        assert (pre["radius"] > 0).all()
        out[j] = (pre["rgb"][:, 0].astype(np.float64) - 0.5) / 0.1
    return out


def test_sh_orthonormality_quadrature():
    # R12 constants: integral of Y_k Y_l over the sphere = delta_kl
    # (product Gauss-Legendre in cos(theta) x trapezoid in phi, exact for these degrees)
    xg, wg = np.polynomial.legendre.leggauss(10)
    nphi = 20
    dirs, w = [], []
    for ct, wt in zip(xg, wg):
        st = math.sqrt(1 - ct * ct)
        for k in range(nphi):
            ph = 2 * math.pi * k / nphi
            dirs.append(np.array([st * math.cos(ph), st * math.sin(ph), ct]))
            w.append(wt * 2 * math.pi / nphi)
    Y = _basis_values(dirs)
    gram = (Y * np.asarray(w)[:, None]).T @ Y
    np.testing.assert_allclose(gram, np.eye(16), atol=2e-5)


def test_sh_degree1_signs():
    # R12 sign convention ([3DGS]): Y_1 = -C1 y, Y_2 = C1 z, Y_3 = -C1 x, C1 = sqrt(3 / (4 pi))
    c1 = math.sqrt(3 / (4 * math.pi))
    Y = _basis_values([np.array([1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([0, 0, 1.0])])
    np.testing.assert_allclose(Y[:, 1:4], [[0, 0, -c1], [-c1, 0, 0], [0, c1, 0]], atol=2e-6)


def _real_sh_scipy(d):
    """Real spherical harmonics Y_k(d), k = l^2 + l + m (l <= 3), built from scipy's complex
    Y_l^m (scipy.special.sph_harm_y, Condon-Shortley phase included) -- a library evaluation
    independent of the oracle's hand-expanded polynomials.  [3DGS] real form (R12, the
    convention of the SH coefficients PAPER.md l.59 names): m < 0 -> sqrt2 Im Y_l^|m|,
    m = 0 -> Y_l^0, m > 0 -> sqrt2 Re Y_l^m (the CS phase kept, which gives Y_1 = -C1 y,
    Y_3 = -C1 x)."""
    from scipy.special import sph_harm_y

    x, y, z = (float(v) for v in d)
    theta = math.acos(max(-1.0, min(1.0, z)))  # polar
    phi = math.atan2(y, x)                      # azimuth
    out = np.zeros(16)
    for l in range(4):
        for m in range(-l, l + 1):
            c = complex(sph_harm_y(l, abs(m), theta, phi))
            if m < 0:
                v = math.sqrt(2.0) * c.imag
            elif m == 0:
                v = c.real
            else:
                v = math.sqrt(2.0) * c.real
            out[l * l + l + m] = v
    return out


def test_sh_basis_every_coefficient_against_scipy():
    # R12 (§I: colour from SH coefficients): every Y_k, k < 16, value AND sign,
    # at 40 directions (random + the axes + diagonals) against scipy's complex SH turned into
    # the real form; a flipped sign or swapped polynomial in any Y_k fails here (the
    # orthonormality quadrature above is blind to a single sign flip).
    r = np.random.default_rng(11)
    dirs = list(r.standard_normal((30, 3)))
    dirs += [np.array(v, float) for v in ([1, 0, 0], [0, 1, 0], [0, 0, 1], [-1, 0, 0], [0, -1, 0], [0, 0, -1],
                                          [1, 1, 1], [-1, 2, 0.5], [0.3, -0.2, -1], [2, -1, 1])]
    dirs = [d / np.linalg.norm(d) for d in dirs]
    got = _basis_values(dirs)
    want = np.array([_real_sh_scipy(d) for d in dirs])
    np.testing.assert_allclose(got, want, atol=3e-6)
    # and the pin is not vacuous: every coefficient takes values of both signs over the set
    for k in range(1, 16):
        assert (want[:, k] > 1e-3).any() and (want[:, k] < -1e-3).any(), k


def test_sh_clamped_below_only():
    # R12: rgb clamped below at 0, never above (R17)
    sh = np.zeros((2, 16, 3), np.float32)
    sh[0, 0, :] = [-5.0, 5.0, 0.0]
    th, n = gaussians([[0, 0, 2.0], [0, 0, 2.0]], sh=sh)
    pre = oracle.preprocess(th, n, 0, axis_camera(64, 64))
    assert pre["rgb"][0, 0] == 0.0 and pre["cbits"][0] & oracle.CB_R
    assert pre["rgb"][0, 1] > 1.0 and not pre["cbits"][0] & oracle.CB_G


def test_rect_square_three_sigma():
    # R10/R11: square half-width r around the centre, floor-then-clamp to the tile grid
    W, H = 100, 70  # ragged edge tiles
    th, n = gaussians([[0.0, 0.0, 2.0], [0.9, 0.6, 2.0], [5.0, 5.0, 2.0]],
                      log_scales=[[math.log(0.02)] * 3, [math.log(0.05)] * 3, [math.log(0.01)] * 3])
    pre = oracle.preprocess(th, n, 0, axis_camera(W, H))
    tx, ty = 7, 5
    for i in range(2):
        x, y = pre["xy"][i]
        r = pre["radius"][i]
        ex = [max(0, min(tx, math.floor((x - r) / 16))), max(0, min(ty, math.floor((y - r) / 16))),
              max(0, min(tx, math.floor((x + r + 15) / 16))), max(0, min(ty, math.floor((y + r + 15) / 16)))]
        assert list(pre["rect"][i]) == ex
    assert pre["radius"][2] == 0 and pre["tiles_touched"][2] == 0  # entirely off-screen -> absent
