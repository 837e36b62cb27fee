"""Pins of the oracle's keys/sort/ranges (O10-O13) and blend forward (O14).

PAPER.md l.143-149 (§II-A): C = sum_{i in N} c_i alpha_i prod_{j<i}(1 - alpha_j), N
sorted by depth.  SPEC.md l.147-158 examples and l.179-181 properties, adapted to
readings R13-R17.
"""
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle
from tests.helpers import axis_camera, gaussians, sh_for_rgb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "blend_examples.json")))


# ---------------------------------------------------------------- keys / sort / ranges
def test_keys_one_tile_two_tiles_none():
    # inside one tile -> 1 key; spanning a boundary -> 2 keys; 0 splats -> empty ranges
    W = H = 64
    f = 64.0
    cam = axis_camera(W, H, f)
    # pixel (8, 8) at depth 2: x = ((X/(z*0.5)+1)*64-1)/2 = 8  -> X = (17/64 - 1) * z * 0.5
    X = (17 / 64 - 1) * 2 * 0.5
    th, n = gaussians([[X, X, 2.0]], log_scales=[[math.log(0.001)] * 3])
    pre = oracle.preprocess(th, n, 0, cam)
    srt = oracle.sort_keys(pre, cam)
    assert srt["K"] == 1 and int(srt["sorted_keys"][0] >> 32) == 0
    # centre on the boundary between tile columns 0 and 1 (x = 15.5)
    X2 = (32 / 64 - 1) * 2 * 0.5
    th, n = gaussians([[X2, X, 2.0]], log_scales=[[math.log(0.001)] * 3])
    pre = oracle.preprocess(th, n, 0, cam)
    srt = oracle.sort_keys(pre, cam)
    assert srt["K"] == 2 and [int(k >> 32) for k in srt["sorted_keys"]] == [0, 1]
    th, n = gaussians(np.zeros((0, 3)))
    pre = oracle.preprocess(th, 0, 0, cam)
    srt = oracle.sort_keys(pre, cam)
    assert srt["K"] == 0 and not srt["ranges"].any()


@pytest.mark.parametrize("cfg", ["tiny", "small"])
def test_sort_invariants(cfg):
    s = gen.tiny() if cfg == "tiny" else gen.small_scene(3, 700, 100, 70)
    cam = s.cameras[0]
    pre = oracle.preprocess(s.theta, s.n, 3, cam)
    srt = oracle.sort_keys(pre, cam)
    K = srt["K"]
    assert K == int(pre["tiles_touched"].astype(np.int64).sum())
    # keys/values as a multiset are preserved and ascending after the sort
    assert np.array_equal(np.sort(srt["keys"]), srt["sorted_keys"])
    # stable: equal keys keep ascending Gaussian index; order = (tile, depth bits, index) (R13)
    tile = (srt["sorted_keys"] >> np.uint64(32)).astype(np.int64)
    dbits = (srt["sorted_keys"] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    order = np.lexsort((srt["sorted_values"], dbits, tile))
    assert np.array_equal(order, np.arange(K))
    # depth bits are the Gaussian's depth, tile inside its rect
    v = srt["sorted_values"]
    assert np.array_equal(dbits.astype(np.uint32), pre["depth"][v].view(np.uint32))
    tx, _ = cam.tiles()
    r = pre["rect"][v]
    assert ((tile % tx >= r[:, 0]) & (tile % tx < r[:, 2]) & (tile // tx >= r[:, 1]) & (tile // tx < r[:, 3])).all()
    # ranges: disjoint, ascending, cover [0, K)
    rg = srt["ranges"].astype(np.int64)
    ne = rg[rg[:, 1] > rg[:, 0]]
    assert (ne[:, 1] - ne[:, 0]).sum() == K
    assert (ne[1:, 0] == ne[:-1, 1]).all() and (ne[0, 0] == 0 if K else True)
    for t in range(rg.shape[0]):
        assert (tile[rg[t, 0]:rg[t, 1]] == t).all()
    # each Gaussian appears exactly tiles_touched times
    assert np.array_equal(np.bincount(v, minlength=s.n), pre["tiles_touched"])


# ---------------------------------------------------------------- blend closed forms
def _single(W, c, ologit, bg):
    cam = axis_camera(W, W, bg=bg)
    th, n = gaussians([[0, 0, 2.0]], log_scales=[[math.log(0.05)] * 3], ologits=[ologit], sh=[sh_for_rgb(c)])
    return cam, oracle.forward(th, n, 0, cam)


def test_golden_single_opaque_splat():
    g = GOLD["single_opaque"]
    W = 33  # odd: the projected centre (W-1)/2 = 16 is a pixel centre, so G = exp(0) = 1
    cam, f = _single(W, g["c"], 30.0, GOLD["bg"])
    np.testing.assert_allclose(f["image"][:, 16, 16], g["expected"], atol=2e-6)
    assert f["n_contrib"][16, 16] == 1


def test_golden_two_splats():
    g = GOLD["two_splats"]
    W = 33
    cam = axis_camera(W, W, bg=GOLD["bg"])
    th, n = gaussians([[0, 0, 3.0], [0, 0, 2.0]], log_scales=[[math.log(0.05)] * 3] * 2, ologits=[30.0, 0.0],
                      sh=[sh_for_rgb(g["c2"]), sh_for_rgb(g["c1"])])
    f = oracle.forward(th, n, 0, cam)
    np.testing.assert_allclose(f["image"][:, 16, 16], g["expected"], atol=2e-6)
    assert f["n_contrib"][16, 16] == 2


def test_golden_empty_scene_is_background():
    cam = axis_camera(40, 24, bg=GOLD["bg"])
    th, n = gaussians(np.zeros((0, 3)))
    f = oracle.forward(th, 0, 0, cam)
    assert (f["image"] == np.asarray(GOLD["empty"]["expected"], np.float32)[:, None, None]).all()
    assert (f["final_T"] == 1).all() and (f["n_contrib"] == 0).all()


def test_transparent_scene_is_background():
    # opacity logit -100 -> o ~ 0: image = bg exactly, T = 1, n_contrib = 0 (BASELINE.json north_star)
    s = gen.small_scene(1, 300, 64, 48)
    seg = gen.segments(s.theta, s.n)
    seg["opacity_logits"][:] = -100.0
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    assert (f["image"] == cam.bg[:, None, None]).all()
    assert (f["final_T"] == 1).all() and (f["n_contrib"] == 0).all()


@pytest.mark.parametrize("cfg", ["tiny", "small"])
def test_tiled_equals_bruteforce(cfg):
    # the per-tile sorted lists give exactly the per-pixel brute-force composite
    s = gen.tiny() if cfg == "tiny" else gen.small_scene(4, 512, 64, 64, scale_mu=0.08)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    b = oracle.bruteforce(f["pre"], cam)
    assert np.array_equal(f["image"], b["image"])
    assert np.array_equal(f["n_contrib"], b["n_contrib"])
    assert np.array_equal(f["final_T"], b["final_T"])


def test_transmittance_bounds_and_counts():
    s = gen.tiny()
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    assert (f["final_T"] >= 1e-4).all() and (f["final_T"] <= 1).all()
    assert (f["n_contrib"] <= f["walked"]).all() and (f["blended"] <= f["n_contrib"]).all()
    # T non-increasing along each walk: follows from alpha in [0, 0.99]; check on the frozen lists
    fl = oracle.forward(s.theta, s.n, 3, cam, want_lists=True)
    assert (fl["list_ptr"][1:] - fl["list_ptr"][:-1] == fl["blended"].reshape(-1)).all()


def test_energy_bound():
    # S:180 adapted (R17): image <= max_g rgb_g (1 - T) + T bg, and >= T bg
    s = gen.small_scene(2, 800, 96, 64)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    vis = f["pre"]["radius"] > 0
    cmax = f["pre"]["rgb"][vis].max(0)
    T = f["final_T"]
    for ch in range(3):
        assert (f["image"][ch] <= cmax[ch] * (1 - T) + T * cam.bg[ch] + 1e-5).all()
        assert (f["image"][ch] >= T * cam.bg[ch] - 1e-6).all()


def test_permutation_invariance():
    # permuting the input order leaves the render bit-identical (no exact depth ties here)
    s = gen.small_scene(5, 600, 80, 64)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    perm = np.random.default_rng(0).permutation(s.n)
    seg = gen.segments(s.theta, s.n)
    th2 = gen.pack(seg["means"][perm], seg["log_scales"][perm], seg["quats"][perm], seg["opacity_logits"][perm],
                   seg["sh"][perm])
    f2 = oracle.forward(th2, s.n, 3, cam)
    d = f["pre"]["depth"][f["pre"]["radius"] > 0]
    assert len(np.unique(d.view(np.uint32))) == len(d)
    assert np.array_equal(f["image"], f2["image"]) and np.array_equal(f["n_contrib"], f2["n_contrib"])


def test_depth_ties_broken_by_index():
    # R13 / S:188: equal depth bits -> lower Gaussian index in front
    W = 33
    cam = axis_camera(W, W, bg=(0, 0, 0))
    th, n = gaussians([[0, 0, 2.0], [0, 0, 2.0]], ologits=[0.0, 0.0],
                      sh=[sh_for_rgb([1, 0, 0]), sh_for_rgb([0, 1, 0])])
    f = oracle.forward(th, n, 0, cam)
    px = f["image"][:, 16, 16]
    assert px[0] > px[1]  # Gaussian 0 (red) composited first: 0.5 vs 0.25
    np.testing.assert_allclose(px[:2], [0.5, 0.25], atol=1e-6)


def test_early_stop_soundness():
    # S:181 adapted to R15: the stop drops the crossing Gaussian and everything behind it, so
    # disabling it moves a pixel by at most final_T * max(c, bg); final_T < 1e-4/(1-0.99) = 0.01
    s = gen.tiny()
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    g = oracle.forward(s.theta, s.n, 3, cam, mode=oracle.NO_EARLY_STOP)
    bound = max(float(f["pre"]["rgb"].max()), float(cam.bg.max()))
    d = np.abs(f["image"] - g["image"]).max(0)
    assert (d <= f["final_T"] * bound + 1e-6).all()
    stopped = f["final_T"] < 1e-2
    assert (d[~stopped] <= 1e-6).all()


def _p146_literal(theta, n, cam, rgb):
    """PAPER.md l.128-149 evaluated literally in double: alpha_i = o_i G_i(x) with
    G(x) = exp(-1/2 d^T Sigma'^-1 d), Sigma' = J W Sigma W^T J^T (standard first-order
    pinhole Jacobian), C = sum c_i alpha_i prod_{j<i}(1 - alpha_j), N sorted by
    depth; plus T bg (R16).  No clamp, cutoff, early stop, low-pass or tiles."""
    seg = gen.segments(theta.astype(np.float64), n)
    V = np.asarray(cam.view, np.float64).reshape(4, 4).T  # column-major -> row-major
    Pm = np.asarray(cam.proj, np.float64).reshape(4, 4).T
    W, H = cam.width, cam.height
    fx, fy = W / (2 * cam.tan_fovx), H / (2 * cam.tan_fovy)
    recs = []
    for i in range(n):
        mu = seg["means"][i]
        t = V[:3, :3] @ mu + V[:3, 3]
        if t[2] <= cam.near:
            continue
        clip = Pm @ np.append(mu, 1.0)
        px = ((clip[0] / clip[3] + 1) * W - 1) / 2
        py = ((clip[1] / clip[3] + 1) * H - 1) / 2
        q = seg["quats"][i] / np.linalg.norm(seg["quats"][i])
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        S = np.diag(np.exp(seg["log_scales"][i]))
        Sig = R @ S @ S.T @ R.T
        J = np.array([[fx / t[2], 0, -fx * t[0] / t[2] ** 2], [0, fy / t[2], -fy * t[1] / t[2] ** 2]])
        Sp = J @ V[:3, :3] @ Sig @ V[:3, :3].T @ J.T
        o = 1 / (1 + math.exp(-seg["opacity_logits"][i]))
        recs.append((t[2], i, np.array([px, py]), np.linalg.inv(Sp), o))
    recs.sort(key=lambda r: (r[0], r[1]))
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    C = np.zeros((3, H, W))
    T = np.ones((H, W))
    for _, i, m, Q, o in recs:
        dx, dy = xs - m[0], ys - m[1]
        a = o * np.exp(-0.5 * (Q[0, 0] * dx * dx + 2 * Q[0, 1] * dx * dy + Q[1, 1] * dy * dy))
        C += rgb[i][:, None, None] * (a * T)[None]
        T *= 1 - a
    return C + T[None] * np.asarray(cam.bg, np.float64)[:, None, None]


@pytest.mark.parametrize("seed", [0, 1])
def test_plain_mode_equals_paper_formula(seed):
    # every reading switched off == P:146 literally (pins the formula itself)
    s = gen.small_scene(seed, 24, 48, 32, scale_mu=0.08)
    seg = gen.segments(s.theta, s.n)
    seg["opacity_logits"][:] = np.random.default_rng(seed).normal(-1.0, 1.0, s.n)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam, mode=oracle.PLAIN)
    assert (f["pre"]["radius"] > 0).sum() == s.n
    ref = _p146_literal(s.theta, s.n, cam, f["pre"]["rgb"].astype(np.float64))
    assert np.abs(f["image"] - ref).max() < 2e-5


def test_canon_exp_is_exp_to_float_accuracy():
    # R23 parity mode: the canonical exponential is exp within a few float ulps on the blend's
    # range (power <= 0 down to the alpha cutoff: power >= ln(1/255) - margin > -12)
    x = np.linspace(-12.0, 0.0, 200001).astype(np.float32)
    got = oracle.canon_exp(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    # the float rounding of x = power * log2(e) (|x| <= 17.3: <= 2^-20 absolute) dominates;
    # the polynomial adds < 2^-22 (the same budget as MUFU.EX2 on that x)
    assert (np.abs(got - ref) <= 1.5e-6 * ref).all()
    mid = x > -4.0
    assert (np.abs(got - ref)[mid] <= 4e-7 * ref[mid]).all()
    assert oracle.canon_exp(np.float32([0.0]))[0] == 1.0  # 2^0 * p(0) = 1 exactly


def test_parity_mode_forward_close_to_default():
    s = gen.small_scene(5, 700, 48, 40)
    cam = s.cameras[0]
    a = oracle.forward(s.theta, s.n, s.sh_degree, cam)
    b = oracle.forward(s.theta, s.n, s.sh_degree, cam, mode=oracle.CANON_EXP)
    ok = (a["flags"] == 0) & (b["flags"] == 0)
    assert np.array_equal(a["n_contrib"][ok], b["n_contrib"][ok])
    assert np.abs(a["image"] - b["image"])[:, ok].max() <= 1e-5


@pytest.mark.parametrize("cfg", ["tiny", "small", "opaque"])
def test_alpha_box_rect_loses_no_contribution(cfg):
    """R11': the tile lists built from each Gaussian's alpha >= 1/255 box give exactly the
    image and transmittance of lists holding EVERY visible Gaussian in EVERY tile (the alpha
    cutoff R14 and early stop R15 on): no tile outside a Gaussian's box has a pixel that
    blends it.  R10's square rect (3 sqrt(lambda_1)) truncates high-opacity Gaussians, whose
    alpha >= 1/255 set reaches sqrt(2 ln 255) = 3.33 sigma, so it is pinned only as a superset
    of keys it is not.  'opaque': logits ~ N(6, 1), the case where the two rects differ."""
    if cfg == "opaque":
        s = gen.small_scene(5, 400, 64, 48, scale_mu=0.08)
        seg = gen.segments(s.theta, s.n)
        seg["opacity_logits"][:] = 6.0 + gen.rng(6).standard_normal(s.n).astype(np.float32)
    else:
        s = gen.tiny() if cfg == "tiny" else gen.small_scene(4, 512, 64, 64, scale_mu=0.08)
    cam = s.cameras[0]
    f = oracle.forward(s.theta, s.n, 3, cam)
    full = oracle.forward(s.theta, s.n, 3, cam, mode=oracle.FULL_RECT)
    assert np.array_equal(f["image"], full["image"])
    assert np.array_equal(f["final_T"], full["final_T"])
    # the blended entries are the same, so n_contrib counts positions in shorter lists
    assert f["srt"]["K"] < full["srt"]["K"]
    sq = oracle.forward(s.theta, s.n, 3, cam, mode=oracle.SQUARE_RECT)
    print(cfg, "K alpha box", f["srt"]["K"], "K square", sq["srt"]["K"],
          "max |image - square image|", float(np.abs(f["image"] - sq["image"]).max()))
