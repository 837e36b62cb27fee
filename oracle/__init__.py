"""ctypes wrapper of the CPU oracle (oracle/bgs_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs, never by the product package
paper_2510_14564_b200/ (which fails loudly without its CUDA library instead).

Each function cites the step of SURVEY.md §8(c) (O1-O17) it wraps; the C++
file cites the paper passages.  Parity status per function is in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bgs_oracle.cpp")
LIB = os.path.join(HERE, "liborc.so")

# mode bits (switch readings off; plain mode = all of them), see bgs_oracle.cpp
NO_LOWPASS, NO_JCLAMP, FULL_RECT = 1, 2, 4
NO_ALPHA_CLAMP, NO_ALPHA_CUTOFF, NO_EARLY_STOP, NO_POWER_GUARD = 8, 16, 32, 64
PLAIN = 127
CANON_EXP = 128  # R23 parity mode: the canonical exponential the GPU's parity mode also uses
SQUARE_RECT = 256  # R10/R11: 3DGS's square rect of half-width radius instead of R11' (the alpha box)
# clamp bits
CB_R, CB_G, CB_B, CB_JX, CB_JX_NEG, CB_JY, CB_JY_NEG = 1, 2, 4, 8, 16, 32, 64

# R23 near-tie margins: relative distance of a decision input
# to its threshold under which a pixel is flagged.  The GPU's G = ex2.approx(power*log2e)
# differs from exp(power) by <= 2^-20.5 relative for |power| <= 5.6 (log2e product rounding
# 8*2^-24 plus ex2.approx's ~2^-22); DELTA_ALPHA leaves a 4x margin over that.  T is a
# product of (1 - alpha) factors, each relative error <= 99 * 2^-20.5 (alpha < 0.99
# unclamped), so DELTA_T = 2^-11 covers several such factors.
DELTA_ALPHA = 2.0 ** -18
DELTA_T = 2.0 ** -11

CFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liborc.so with g++ (no -ffast-math, no FP contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, "-o", tmp, SRC])
        os.replace(tmp, LIB)
    return LIB


class Camera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("proj", C.c_float * 16), ("campos", C.c_float * 3),
                ("tan_fovx", C.c_float), ("tan_fovy", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32), ("bg", C.c_float * 3), ("near_plane", C.c_float)]


def camera(cam) -> Camera:
    c = Camera()
    c.view[:] = [float(x) for x in np.asarray(cam.view, np.float32)]
    c.proj[:] = [float(x) for x in np.asarray(cam.proj, np.float32)]
    c.campos[:] = [float(x) for x in np.asarray(cam.campos, np.float32)]
    c.tan_fovx, c.tan_fovy = float(cam.tan_fovx), float(cam.tan_fovy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.bg[:] = [float(x) for x in np.asarray(cam.bg, np.float32)]
    c.near_plane = float(cam.near)
    return c


P = C.c_void_p


def lib():
    global _lib
    with _lock:
        if _lib is None:
            l = C.CDLL(build())
            sig = {
                "orc_preprocess": [C.c_int64, C.c_int32, P, P, C.c_uint32] + [P] * 9,
                "orc_scan": [C.c_int64, P, P],
                "orc_duplicate": [C.c_int64, P, P, P, P, C.c_int32, P, P],
                "orc_sort": [C.c_int64, P, P],
                "orc_ranges": [C.c_int64, P, C.c_int32, P],
                "orc_render_fwd": [P, C.c_uint32, P, P, P, P, P, P, P, P, P, P, P, P, C.c_double, C.c_double, P, P, P],
                "orc_render_bruteforce": [P, C.c_uint32, C.c_int64, P, P, P, P, P, P, P, P, P, P],
                "orc_render_frozen": [C.c_int64, C.c_int32, P, P, C.c_uint32, P, P, P, P, P, P],
                "orc_render_bwd": [C.c_int64, C.c_int32, P, P, C.c_uint32, P, P, P, P, P, P, P, P, P, P, P, P, P],
                "orc_preprocess_bwd": [C.c_int64, C.c_int32, P, P, C.c_uint32, P, P, P, P, P, P, P],
                "orc_adam": [C.c_int64, P, P, P, P, P, C.c_double, C.c_double, C.c_double, C.c_int64],
                "orc_local_density": [C.c_int64, P, C.c_float, P],
                "orc_knn_mean": [C.c_int64, P, C.c_int32, P],
                "orc_canon_exp": [C.c_int64, P, P],
            }
            for name, args in sig.items():
                fn = getattr(l, name)
                fn.argtypes = args
                fn.restype = None
            l.orc_scan.restype = C.c_int64
            l.orc_set_threads.argtypes = [C.c_int32]
            l.orc_set_threads.restype = C.c_int32
            _lib = l
    return _lib


def set_threads(k: int = 0) -> int:
    """Host threads for the oracle's parallel loops (0 = all cores, 1 = serial); results do
    not depend on it (bgs_oracle.cpp: fixed-order reductions).  Returns the count in effect."""
    return int(lib().orc_set_threads(int(k)))


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be contiguous"
    return a.ctypes.data_as(C.c_void_p)


def tiles_of(cam):
    return (cam.width + 15) // 16, (cam.height + 15) // 16


# ---------------------------------------------------------------------------
def preprocess(theta, n, deg, cam, mode=0) -> dict:
    """O1-O9 (+ tiles_touched): SURVEY §8(c); PAPER.md l.128-142 (§II-A)."""
    theta = np.ascontiguousarray(theta, np.float32)
    out = dict(radius=np.zeros(n, np.int32), depth=np.zeros(n, np.float32), xy=np.zeros((n, 2), np.float32),
               conic=np.zeros((n, 3), np.float32), opacity=np.zeros(n, np.float32), rgb=np.zeros((n, 3), np.float32),
               cbits=np.zeros(n, np.uint8), rect=np.zeros((n, 4), np.int32), tiles_touched=np.zeros(n, np.uint32))
    c = camera(cam)
    lib().orc_preprocess(n, deg, _p(theta), C.byref(c), mode, *[_p(out[k]) for k in
                         ("radius", "depth", "xy", "conic", "opacity", "rgb", "cbits", "rect", "tiles_touched")])
    return out


def sort_keys(pre: dict, cam) -> dict:
    """O10-O13: scan, (tile|depth) keys in index order, std::stable_sort, ranges."""
    n = pre["radius"].shape[0]
    tx, ty = tiles_of(cam)
    offsets = np.zeros(n, np.uint64)
    K = lib().orc_scan(n, _p(pre["tiles_touched"]), _p(offsets))
    keys = np.zeros(K, np.uint64)
    values = np.zeros(K, np.uint32)
    lib().orc_duplicate(n, _p(pre["tiles_touched"]), _p(pre["depth"]), _p(pre["rect"]), _p(offsets), tx,
                        _p(keys), _p(values))
    skeys, svalues = keys.copy(), values.copy()
    lib().orc_sort(K, _p(skeys), _p(svalues))
    ranges = np.zeros((tx * ty, 2), np.uint32)
    lib().orc_ranges(K, _p(skeys), tx * ty, _p(ranges))
    return dict(offsets=offsets, K=int(K), keys=keys, values=values, sorted_keys=skeys, sorted_values=svalues,
                ranges=ranges)


def render_fwd(pre, srt, cam, mode=0, want_lists=False, delta_alpha=DELTA_ALPHA, delta_T=DELTA_T) -> dict:
    """O14: front-to-back alpha blend per pixel (Eq. for C)."""
    W, H = cam.width, cam.height
    out = dict(image=np.zeros((3, H, W), np.float32), final_T=np.zeros((H, W), np.float32),
               n_contrib=np.zeros((H, W), np.uint32), walked=np.zeros((H, W), np.uint32),
               blended=np.zeros((H, W), np.uint32), flags=np.zeros((H, W), np.uint8))
    c = camera(cam)
    lp = lg = la = None
    if want_lists:
        tx, _ = tiles_of(cam)
        r = srt["ranges"].astype(np.int64)
        ys, xs = np.mgrid[0:H, 0:W]
        t = (ys // 16) * tx + xs // 16
        cap = int((r[t, 1] - r[t, 0]).sum())
        out["list_ptr"] = np.zeros(W * H + 1, np.int64)
        out["list_gid"] = np.zeros(max(cap, 1), np.int32)
        out["list_aclamp"] = np.zeros(max(cap, 1), np.uint8)
        lp, lg, la = (_p(out[k]) for k in ("list_ptr", "list_gid", "list_aclamp"))
    lib().orc_render_fwd(C.byref(c), mode, _p(srt["ranges"]), _p(srt["sorted_values"]), _p(pre["xy"]),
                         _p(pre["conic"]), _p(pre["opacity"]), _p(pre["rgb"]), _p(out["image"]), _p(out["final_T"]),
                         _p(out["n_contrib"]), _p(out["walked"]), _p(out["blended"]), _p(out["flags"]),
                         float(delta_alpha), float(delta_T), lp, lg, la)
    return out


def forward(theta, n, deg, cam, mode=0, want_lists=False) -> dict:
    """O1-O14 for one view; returns every intermediate."""
    pre = preprocess(theta, n, deg, cam, mode)
    srt = sort_keys(pre, cam)
    fw = render_fwd(pre, srt, cam, mode, want_lists)
    return dict(pre=pre, srt=srt, **fw)


def bruteforce(pre, cam, mode=0) -> dict:
    """per-pixel list built over all N, std::sort by (depth bits, index)."""
    n = pre["radius"].shape[0]
    W, H = cam.width, cam.height
    out = dict(image=np.zeros((3, H, W), np.float32), final_T=np.zeros((H, W), np.float32),
               n_contrib=np.zeros((H, W), np.uint32))
    c = camera(cam)
    lib().orc_render_bruteforce(C.byref(c), mode, n, _p(pre["tiles_touched"]), _p(pre["rect"]), _p(pre["depth"]),
                                _p(pre["xy"]), _p(pre["conic"]), _p(pre["opacity"]), _p(pre["rgb"]),
                                _p(out["image"]), _p(out["final_T"]), _p(out["n_contrib"]))
    return out


def render_frozen(theta_d, n, deg, cam, fwd, mode=0) -> np.ndarray:
    """Double-precision forward with the float run's decisions frozen (R18)."""
    theta_d = np.ascontiguousarray(theta_d, np.float64)
    img = np.zeros((3, cam.height, cam.width), np.float64)
    c = camera(cam)
    lib().orc_render_frozen(n, deg, _p(theta_d), C.byref(c), mode, _p(fwd["pre"]["radius"]), _p(fwd["pre"]["cbits"]),
                            _p(fwd["list_ptr"]), _p(fwd["list_gid"]), _p(fwd["list_aclamp"]), _p(img))
    return img


def backward(theta, n, deg, cam, fwd, dl_dimage, mode=0) -> dict:
    """O15 + O16: blend backward then preprocess backward (double, decisions frozen)."""
    theta = np.ascontiguousarray(theta, np.float32)
    dl = np.ascontiguousarray(dl_dimage, np.float32)
    pre, srt = fwd["pre"], fwd["srt"]
    g = dict(xy=np.zeros((n, 2)), conic=np.zeros((n, 3)), opacity=np.zeros(n), rgb=np.zeros((n, 3)))
    c = camera(cam)
    lib().orc_render_bwd(n, deg, _p(theta), C.byref(c), mode, _p(pre["radius"]), _p(pre["cbits"]),
                         _p(srt["ranges"]), _p(srt["sorted_values"]), _p(pre["xy"]), _p(pre["conic"]),
                         _p(pre["opacity"]), _p(pre["rgb"]), _p(dl), _p(g["xy"]), _p(g["conic"]), _p(g["opacity"]),
                         _p(g["rgb"]))
    grad = np.zeros(59 * n)
    lib().orc_preprocess_bwd(n, deg, _p(theta), C.byref(c), mode, _p(pre["radius"]), _p(pre["cbits"]), _p(g["xy"]),
                             _p(g["conic"]), _p(g["opacity"]), _p(g["rgb"]), _p(grad))
    g["grad"] = grad
    return g


def adam(theta, grad, m, v, n, lr6, b1=0.9, b2=0.999, eps=1e-15, step=1):
    """O17: Adam, PyTorch semantics (R21), double; returns new (theta, m, v)."""
    th = np.array(theta, np.float64)
    gr = np.array(grad, np.float64)
    mm = np.array(m, np.float64)
    vv = np.array(v, np.float64)
    lr = np.asarray(lr6, np.float64)
    lib().orc_adam(n, _p(th), _p(gr), _p(mm), _p(vv), _p(lr), b1, b2, eps, step)
    return th, mm, vv


def canon_exp(x) -> np.ndarray:
    """R23 parity mode: the canonical float exponential (bgs_oracle.cpp canon_exp)."""
    a = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(a)
    lib().orc_canon_exp(a.size, _p(a), _p(out))
    return out


def local_density(means, r) -> np.ndarray:
    """T1 (§III-C1 l.181-183): rho(p) = number of other points within radius r."""
    m = np.ascontiguousarray(means, np.float32).reshape(-1, 3)
    out = np.zeros(m.shape[0], np.uint32)
    lib().orc_local_density(m.shape[0], _p(m), float(np.float32(r)), _p(out))
    return out


def knn_mean_distance(means, k=8) -> np.ndarray:
    """T1 (§III-C2 l.188-191): d_p = mean distance to the k nearest neighbours."""
    m = np.ascontiguousarray(means, np.float32).reshape(-1, 3)
    out = np.zeros(m.shape[0], np.float64)
    lib().orc_knn_mean(m.shape[0], _p(m), int(k), _p(out))
    return out


def density_thresholds(rho, alpha=1.0, beta=1.0) -> dict:
    """T1 (§III-C1 l.184-186): rho_low = mu - alpha sigma, rho_high = mu + beta sigma,
    mu / sigma the mean and (population) standard deviation of all local densities."""
    r = np.asarray(rho, np.float64)
    mu = float(r.mean())
    sd = float(np.sqrt(((r - mu) ** 2).mean()))
    return {"mu": mu, "sigma": sd, "rho_low": mu - alpha * sd, "rho_high": mu + beta * sd,
            "below": int((r < mu - alpha * sd).sum()), "above": int((r > mu + beta * sd).sum())}


GROUPS = ("means", "log_scales", "quats", "opacity", "sh_dc", "sh_rest")


def group_slices(n):
    """Index arrays of the six Adam/gradient groups inside theta[59n]."""
    sh = np.arange(11 * n, 59 * n)
    dc = sh[((sh - 11 * n) % 48) < 3]
    rest = sh[((sh - 11 * n) % 48) >= 3]
    return dict(means=np.arange(0, 3 * n), log_scales=np.arange(3 * n, 6 * n), quats=np.arange(6 * n, 10 * n),
                opacity=np.arange(10 * n, 11 * n), sh_dc=dc, sh_rest=rest)
