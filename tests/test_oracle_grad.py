"""Pins of the oracle backward (O15-O16) and Adam (O17).

The paper has no backward (it inherits 3DGS training);
reading R18 defines the gradient as the derivative of the forward O1-O14 with
every discrete decision frozen.  Pins: central finite differences in double of
the frozen forward (BASELINE.json north_star: "central finite differences for
every gradient"), closed forms, culled => 0; Adam against torch.optim.Adam.
"""
import math

import numpy as np
import pytest
import torch

import gen
import oracle
from tests.helpers import axis_camera, gaussians, rel_l2, sh_for_rgb


def _fd_scene():
    # 40 Gaussians on 40x32 px plus three that exercise the frozen branches:
    # J clamp (off-screen right, large), rgb clamp (negative DC red), alpha clamp (o ~ 1 at centre)
    s = gen.small_scene(11, 40, 40, 32, scale_mu=0.12)
    seg = gen.segments(s.theta, s.n)
    extra_means = np.array([[3.0, 0.2, 2.0], [0.1, 0.05, 2.2], [-0.2, 0.1, 2.6]])
    extra_ls = np.log(np.array([[1.2, 0.8, 1.0], [0.08, 0.05, 0.06], [0.1, 0.1, 0.1]]))
    extra_q = np.random.default_rng(1).standard_normal((3, 4))
    extra_sh = np.zeros((3, 16, 3), np.float32)
    extra_sh[:, 1:, :] = 0.05 * np.random.default_rng(2).standard_normal((3, 15, 3))
    extra_sh[0, 0] = [0.5, 0.2, -0.3]
    extra_sh[1, 0] = [-4.0, 0.4, 0.1]
    extra_sh[2, 0] = [0.3, 0.3, 0.3]
    theta = gen.pack(np.concatenate([seg["means"], extra_means]), np.concatenate([seg["log_scales"], extra_ls]),
                     np.concatenate([seg["quats"], extra_q]),
                     np.concatenate([seg["opacity_logits"], [1.0, 2.0, 12.0]]),
                     np.concatenate([seg["sh"], extra_sh]))
    return theta, s.n + 3, s.cameras[0]


def test_frozen_double_forward_matches_float_forward():
    s = gen.tiny()
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam, want_lists=True)
    img = oracle.render_frozen(s.theta.astype(np.float64), s.n, 3, cam, f)
    assert np.abs(img - f["image"]).max() < 1e-5


@pytest.mark.parametrize("deg", [3, 1])
def test_gradients_match_central_differences(deg):
    theta, n, cam = _fd_scene()
    f = oracle.forward(theta, n, deg, cam, want_lists=True)
    pre = f["pre"]
    assert pre["cbits"][n - 3] & oracle.CB_JX and pre["radius"][n - 3] > 0
    assert pre["cbits"][n - 2] & oracle.CB_R
    assert f["list_aclamp"][: f["list_ptr"][-1]].any()
    w = gen.random_dl_dimage(3, cam.width, cam.height)
    g = oracle.backward(theta, n, deg, cam, f, w)["grad"]
    th = theta.astype(np.float64)
    fd = np.zeros_like(th)
    wd = w.astype(np.float64)
    for j in range(th.size):
        h = 1e-6 * max(1.0, abs(th[j]))
        tp = th.copy()
        tp[j] += h
        lp = float((wd * oracle.render_frozen(tp, n, deg, cam, f)).sum())
        tp[j] -= 2 * h
        lm = float((wd * oracle.render_frozen(tp, n, deg, cam, f)).sum())
        fd[j] = (lp - lm) / (2 * h)
    for name, idx in oracle.group_slices(n).items():
        if name == "sh_rest" and deg == 0:
            continue
        err = rel_l2(g[idx], fd[idx])
        assert err < 1e-6, (name, err)
    # coefficients above the active degree get no gradient (R12)
    sh_g = g[11 * n:].reshape(n, 16, 3)
    assert not sh_g[:, (deg + 1) ** 2:, :].any()


def test_opacity_gradient_closed_form():
    # single unclamped Gaussian at a pixel centre: dC/do = G T (c - bg) with G = 1, T = 1
    W = 33
    c = np.array([0.7, 0.2, 0.9])
    bg = np.array([0.2, 0.4, 0.6])
    cam = axis_camera(W, W, bg=bg)
    th, n = gaussians([[0, 0, 2.0]], log_scales=[[math.log(0.05)] * 3], ologits=[0.3], sh=[sh_for_rgb(c)])
    f = oracle.forward(th, n, 0, cam)
    for ch in range(3):
        w = np.zeros((3, W, W), np.float32)
        w[ch, 16, 16] = 1.0
        g = oracle.backward(th, n, 0, cam, f, w)
        assert abs(g["opacity"][0] - (c[ch] - bg[ch])) < 2e-6
        o = 1 / (1 + math.exp(-0.3))
        assert abs(g["rgb"][0, ch] - o) < 1e-6  # dC/dc = alpha T
        assert abs(g["grad"][10 * n] - (c[ch] - bg[ch]) * o * (1 - o)) < 2e-6


def test_culled_gaussian_has_zero_gradient():
    s = gen.small_scene(8, 60, 48, 32)
    seg = gen.segments(s.theta, s.n)
    seg["means"][5] = [0.0, 0.0, 0.1]  # behind the near plane
    seg["means"][6] = [50.0, 0.0, 2.0]  # off-screen
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    g = oracle.backward(s.theta, s.n, 3, cam, f, gen.random_dl_dimage(0, 48, 32))["grad"]
    gi = g.copy()
    for i in (5, 6):
        assert f["pre"]["radius"][i] == 0
        for off, w in ((0, 3), (3, 3), (6, 4), (10, 1)):
            assert not gi[off * s.n + w * i: off * s.n + w * (i + 1)].any()
        assert not gi[11 * s.n + 48 * i: 11 * s.n + 48 * (i + 1)].any()


# ---------------------------------------------------------------- Adam (O17)
LR6 = [1.6e-4, 5e-3, 1e-3, 0.05, 2.5e-3, 1.25e-4]


def test_adam_matches_torch():
    # R21: PyTorch Adam semantics; library pin = torch.optim.Adam(foreach=False), one param group per lr group
    n = 50
    r = np.random.default_rng(0)
    th0 = r.standard_normal(59 * n)
    groups = oracle.group_slices(n)
    params = {k: torch.tensor(th0[idx], dtype=torch.float64, requires_grad=True) for k, idx in groups.items()}
    opt = torch.optim.Adam([{"params": [params[k]], "lr": LR6[i]} for i, k in enumerate(oracle.GROUPS)],
                           betas=(0.9, 0.999), eps=1e-15, foreach=False)
    th, m, v = th0.copy(), np.zeros(59 * n), np.zeros(59 * n)
    for step in range(1, 4):
        g = r.standard_normal(59 * n) * (10.0 ** r.uniform(-6, 0, 59 * n))
        for k, idx in groups.items():
            params[k].grad = torch.tensor(g[idx], dtype=torch.float64)
        opt.step()
        th, m, v = oracle.adam(th, g, m, v, n, LR6, step=step)
        ref = np.zeros(59 * n)
        for k, idx in groups.items():
            ref[idx] = params[k].detach().numpy()
        np.testing.assert_allclose(th, ref, rtol=1e-12, atol=1e-14)


def test_adam_first_step_closed_form():
    # step 1: m^ = g, v^ = g^2 -> delta = -lr g / (|g| + eps)
    n = 10
    g = np.random.default_rng(1).standard_normal(59 * n)
    th, _, _ = oracle.adam(np.zeros(59 * n), g, np.zeros(59 * n), np.zeros(59 * n), n, LR6, step=1)
    lr = np.zeros(59 * n)
    for i, (k, idx) in enumerate(oracle.group_slices(n).items()):
        lr[idx] = LR6[i]
    np.testing.assert_allclose(th, -lr * g / (np.abs(g) + 1e-15), rtol=1e-12)


def test_threading_does_not_change_results():
    # bgs_oracle.cpp threads over independent units with fixed-order reductions: the serial
    # program (1 thread) and all host cores give bit-identical outputs
    s = gen.small_scene(21, 3000, 150, 90, scale_mu=0.05)
    cam = s.cameras[0]
    dl = gen.random_dl_dimage(5, cam.width, cam.height)
    outs = []
    for k in (1, 0):
        oracle.set_threads(k)
        f = oracle.forward(s.theta, s.n, s.sh_degree, cam)
        b = oracle.backward(s.theta, s.n, s.sh_degree, cam, f, dl)
        outs.append((f, b))
    oracle.set_threads(0)
    (f1, b1), (f2, b2) = outs
    for key in ("image", "final_T", "n_contrib", "flags"):
        assert np.array_equal(f1[key], f2[key]), key
    for key in ("sorted_keys", "sorted_values", "ranges"):
        assert np.array_equal(f1["srt"][key], f2["srt"][key]), key
    assert np.array_equal(b1["grad"], b2["grad"])
