"""Pins of the blend's threshold EQUALITY cases (readings R14, R15 of DESIGN.md §3).

PAPER.md l.143-149 (§II-A) gives the composite C = sum c_i a_i prod_{j<i}(1 - a_j); the
cut-offs are [3DGS]'s, restated in SPEC.md l.153 / l.187 and fixed by R14 / R15:
  R14  skip the entry iff alpha < 1/255   -> alpha == 1/255 exactly is BLENDED
  R15  stop iff T (1 - alpha) < 1e-4      -> T (1 - alpha) == 1e-4 exactly CONTINUES
Both cases are built at a Gaussian's own projected centre (an on-axis mean projects to the
pixel ((W-1)/2, (H-1)/2) exactly, pinned in test_oracle_projection.py), where power = 0 and
G = exp(0) = 1 exactly, so alpha = o bit for bit.  The opacities below are float32 values
(numpy float32 arithmetic, IEEE single rounding) and the logits were found by a search over
float32 logits whose double sigmoid rounds to them (R5); the tests assert the oracle's
opacities equal them before relying on it.
"""
import math

import numpy as np

import oracle
from tests.helpers import axis_camera, gaussians, sh_for_rgb

F32 = np.float32
ONE = F32(1.0)
W = 65  # odd: the on-axis centre (W-1)/2 = 32 is a pixel
C = 32

# R15 fixture: three Gaussians on the axis, front to back alpha = 0.9, A2, A3 with
# fl(fl(1 - 0.9) * (1 - A2)) * (1 - A3) == 1e-4f exactly; A3_UP = the next float above A3.
A1, A2, A3 = F32(0.9), F32(0.97009975), F32(0.9665555)
A3_UP = np.nextafter(A3, F32(2.0))
LOGITS = {"a1": F32(2.1972244), "a2": F32(3.479532), "a3": F32(3.3638506), "a3_up": F32(3.3638525)}
T_STOP = F32(1e-4)


def r15_scene(a3_logit):
    """Four on-axis Gaussians at depths 2 < 2.5 < 3 < 3.5 (front to back), the last one opaque."""
    cam = axis_camera(W, W)
    means = [[0, 0, 2.0], [0, 0, 2.5], [0, 0, 3.0], [0, 0, 3.5]]
    ol = [LOGITS["a1"], LOGITS["a2"], a3_logit, F32(4.0)]
    sh = [sh_for_rgb(c) for c in ([0.9, 0.1, 0.1], [0.1, 0.9, 0.1], [0.1, 0.1, 0.9], [0.5, 0.5, 0.5])]
    th, n = gaussians(means, log_scales=[[math.log(0.05)] * 3] * 4, ologits=ol, sh=sh)
    return cam, th, n


def test_fixture_arithmetic():
    # the fixture's own premises, in IEEE float32 (numpy)
    T1 = ONE - A1
    T2 = F32(T1 * F32(ONE - A2))
    assert F32(T2 * F32(ONE - A3)) == T_STOP
    assert F32(T2 * F32(ONE - A3_UP)) < T_STOP
    assert A3_UP <= F32(0.99) and A2 <= F32(0.99)


def test_r15_equality_continues():
    # T (1 - alpha) == 1e-4 exactly: the pixel continues and the Gaussian is blended (R15);
    # the next entry (alpha >= 1/255) then crosses below 1e-4 and stops the walk unblended
    cam, th, n = r15_scene(LOGITS["a3"])
    f = oracle.forward(th, n, 0, cam)
    pre = f["pre"]
    assert pre["opacity"][0] == A1 and pre["opacity"][1] == A2 and pre["opacity"][2] == A3
    assert (pre["xy"][:, 0] == C).all() and (pre["xy"][:, 1] == C).all()
    assert f["n_contrib"][C, C] == 3
    assert f["final_T"][C, C] == T_STOP


def test_r15_just_below_stops():
    # one float more opacity: T (1 - alpha) < 1e-4 -> done, this Gaussian NOT blended (R15)
    cam, th, n = r15_scene(LOGITS["a3_up"])
    f = oracle.forward(th, n, 0, cam)
    assert f["pre"]["opacity"][2] == A3_UP
    T2 = F32(F32(ONE - A1) * F32(ONE - A2))
    assert f["n_contrib"][C, C] == 2
    assert f["final_T"][C, C] == T2


def _r14(opacity):
    cam = axis_camera(W, W)
    th, n = gaussians([[0, 0, 2.0]], log_scales=[[math.log(0.05)] * 3], ologits=[0.0],
                      sh=[sh_for_rgb([0.8, 0.3, 0.1])])
    pre = oracle.preprocess(th, n, 0, cam)
    # no float32 logit's sigmoid rounds to exactly 1/255 (searched): set the activated
    # opacity directly -- the blend (O14) reads only the preprocessed record
    pre["opacity"][0] = opacity
    srt = oracle.sort_keys(pre, cam)
    return cam, pre, oracle.render_fwd(pre, srt, cam)


def test_r14_equality_is_blended():
    thr = ONE / F32(255.0)  # the threshold 1/255 as a float32 (correctly rounded division)
    cam, pre, f = _r14(thr)
    assert f["n_contrib"][C, C] == 1
    assert f["final_T"][C, C] == F32(ONE - thr)
    rgb = pre["rgb"][0]
    want = [float(rgb[ch]) * float(thr) + float(ONE - thr) * float(cam.bg[ch]) for ch in range(3)]
    np.testing.assert_allclose(f["image"][:, C, C], want, rtol=2e-7)


def test_r14_just_below_is_skipped():
    below = np.nextafter(ONE / F32(255.0), F32(0.0))
    cam, _, f = _r14(below)
    assert f["n_contrib"][C, C] == 0
    assert f["final_T"][C, C] == ONE
    np.testing.assert_array_equal(f["image"][:, C, C], np.asarray(cam.bg, np.float32))
