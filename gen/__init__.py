"""Seeded synthetic scenes and cameras for the BalanceGS hot path (inputs only).

This module is shared by the oracle tests, the CUDA parity tests and bench.py.
It holds NONE of the method's arithmetic: no projection, no SH constants, no
blending.  It only draws random numbers (numpy Philox, counter-based, seeded
per config) and builds camera matrices in the convention the boundary takes
(column-major 4x4 world->camera `view`, world->clip `proj`
= P.V with the 3DGS pinhole P, plus tan_fov, W, H, campos, bg).

Parameter layout (BASELINE.json "~59 floats per Gaussian"):
    theta = [means 3N | log_scales 3N | quats 4N (w,x,y,z) | opacity_logits N | sh 48N]
with sh stored [N][16][3], coefficient 0 = DC.

Scene shapes follow the recipe in DESIGN.md §"Input recipe",
which targets the paper's measured workload skew: >=100x local density contrast
(Challenge-1) and a >=40x per-pixel workload gap
(Challenge-2).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FLOATS_PER_GAUSSIAN = 59
SEG = {  # (offset multiplier, width) of each segment in units of N
    "means": (0, 3),
    "log_scales": (3, 3),
    "quats": (6, 4),
    "opacity_logits": (10, 1),
    "sh": (11, 48),
}


def rng(seed: int) -> np.random.Generator:
    """Counter-based generator (Philox-4x32) keyed by the config seed."""
    return np.random.Generator(np.random.Philox(key=int(seed)))


def segments(theta: np.ndarray, n: int) -> dict:
    """Views of the flat theta[59n] buffer, shaped per segment."""
    out = {}
    for name, (off, w) in SEG.items():
        v = theta[off * n:(off + w) * n]
        out[name] = v.reshape(n, 16, 3) if name == "sh" else (v.reshape(n, w) if w > 1 else v)
    return out


def pack(means, log_scales, quats, opacity_logits, sh) -> np.ndarray:
    n = means.shape[0]
    theta = np.empty(FLOATS_PER_GAUSSIAN * n, dtype=np.float32)
    s = segments(theta, n)
    s["means"][:] = means
    s["log_scales"][:] = log_scales
    s["quats"][:] = quats
    s["opacity_logits"][:] = opacity_logits
    s["sh"][:] = sh
    return theta


@dataclasses.dataclass
class Camera:
    view: np.ndarray      # float32[16], column-major world->camera
    proj: np.ndarray      # float32[16], column-major world->clip (P . view)
    campos: np.ndarray    # float32[3]
    tan_fovx: float
    tan_fovy: float
    width: int
    height: int
    bg: np.ndarray        # float32[3]
    near: float = 0.2

    def tiles(self):
        return (self.width + 15) // 16, (self.height + 15) // 16


def _colmajor(m4: np.ndarray) -> np.ndarray:
    # element (r, k) of the row-major matrix goes to index r + 4k
    return np.ascontiguousarray(m4.T).reshape(16).astype(np.float32)


def pinhole_proj(tan_fovx: float, tan_fovy: float, znear: float = 0.01, zfar: float = 100.0) -> np.ndarray:
    """The 3DGS pinhole clip matrix (row-major), z_sign = +1 (camera looks along +z)."""
    p = np.zeros((4, 4), dtype=np.float64)
    p[0, 0] = 1.0 / tan_fovx
    p[1, 1] = 1.0 / tan_fovy
    p[2, 2] = zfar / (zfar - znear)
    p[2, 3] = -(zfar * znear) / (zfar - znear)
    p[3, 2] = 1.0
    return p


def make_camera(R_wc: np.ndarray, campos, width: int, height: int, fx: float, fy: float,
                bg=(0.0, 0.0, 0.0), near: float = 0.2) -> Camera:
    """R_wc rows = camera x (right), y (down), z (forward) axes in world coordinates."""
    campos = np.asarray(campos, dtype=np.float64)
    m = np.eye(4)
    m[:3, :3] = R_wc
    m[:3, 3] = -R_wc @ campos
    tanx = width / (2.0 * fx)
    tany = height / (2.0 * fy)
    full = pinhole_proj(tanx, tany) @ m
    return Camera(view=_colmajor(m), proj=_colmajor(full), campos=campos.astype(np.float32),
                  tan_fovx=float(np.float32(tanx)), tan_fovy=float(np.float32(tany)),
                  width=int(width), height=int(height), bg=np.asarray(bg, np.float32), near=near)


def look_at(campos, target, width, height, fx, fy, up=(0.0, 1.0, 0.0), bg=(0.0, 0.0, 0.0)) -> Camera:
    campos = np.asarray(campos, np.float64)
    f = np.asarray(target, np.float64) - campos
    f /= np.linalg.norm(f)
    down = -np.asarray(up, np.float64)
    x = np.cross(down, f)
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    return make_camera(np.stack([x, y, f]), campos, width, height, fx, fy, bg=bg)


# ---------------------------------------------------------------------------
# Gaussian attribute draws (shared by every config)
# ---------------------------------------------------------------------------

def _sh_rest(r: np.random.Generator, n: int) -> np.ndarray:
    """SH coefficients 1..15, sigma 0.10 / 0.05 / 0.025 for degrees 1 / 2 / 3."""
    sig = np.array([0.10] * 3 + [0.05] * 5 + [0.025] * 7, dtype=np.float32)
    return (r.standard_normal((n, 15, 3), dtype=np.float32) * sig[None, :, None])


def _sh_dc(r: np.random.Generator, means: np.ndarray) -> np.ndarray:
    """A smooth per-position DC field plus noise (values of the raw DC coefficient)."""
    k = r.uniform(1.0, 4.0, size=(3, 3)).astype(np.float32)
    phi = r.uniform(0.0, 2 * np.pi, size=3).astype(np.float32)
    field = np.sin(means @ k.T + phi[None, :]) * np.float32(1.25)
    return (field + 0.18 * r.standard_normal((means.shape[0], 3), dtype=np.float32)).astype(np.float32)


def _opacity_bimodal(r: np.random.Generator, n: int) -> np.ndarray:
    hi = r.random(n) < 0.4
    return np.where(hi, r.normal(4.0, 1.0, n), r.normal(-3.0, 1.5, n)).astype(np.float32)


def _log_scales(r, n, mu, sigma, flat_factor=None):
    ls = (np.log(mu) + sigma * r.standard_normal((n, 3))).astype(np.float32)
    if flat_factor is not None:  # one (randomly oriented) axis flattened: surface splats
        ls[:, 2] += np.float32(np.log(flat_factor))
    return ls


def _assemble(r, means, log_scales, opac):
    n = means.shape[0]
    quats = r.standard_normal((n, 4), dtype=np.float32)
    sh = np.empty((n, 16, 3), dtype=np.float32)
    sh[:, 0, :] = _sh_dc(r, means)
    sh[:, 1:, :] = _sh_rest(r, n)
    return pack(means.astype(np.float32), log_scales, quats, opac, sh)


def _unit(r, n):
    v = r.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _on_ellipsoid(r, n, c, radii):
    return np.asarray(c) + _unit(r, n) * np.asarray(radii)


def _on_box(r, n, c, half):
    half = np.asarray(half, np.float64)
    p = r.uniform(-1, 1, size=(n, 3)) * half
    face = r.integers(0, 6, size=n)
    ax = face // 2
    sgn = np.where(face % 2 == 0, -1.0, 1.0)
    p[np.arange(n), ax] = sgn * half[ax]
    return np.asarray(c) + p


def _ground(r, n, y, rmax, scale=2.0):
    rad = r.exponential(scale, size=n * 2)
    rad = rad[rad < rmax][:n]
    while rad.shape[0] < n:
        extra = r.exponential(scale, size=n)
        rad = np.concatenate([rad, extra[extra < rmax]])[:n]
    th = r.uniform(0, 2 * np.pi, n)
    return np.stack([rad * np.cos(th), np.full(n, y) + 0.003 * r.standard_normal(n), rad * np.sin(th)], 1)


def _shell(r, n, r0, r1, upper_bias=0.0):
    d = _unit(r, n)
    if upper_bias:
        d[:, 1] = np.abs(d[:, 1]) * (1 - upper_bias) + upper_bias * np.abs(d[:, 1])
    rad = r.uniform(r0, r1, n)
    return d * rad[:, None]


# ---------------------------------------------------------------------------
# Configs (BASELINE.json `configs`; recipe in DESIGN.md)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class Scene:
    name: str
    n: int
    theta: np.ndarray          # float32[59n]
    cameras: list              # list[Camera]
    sh_degree: int = 3
    extent: float = 1.0        # 1.1 x radius of the camera centres' bounding sphere (R21)


def _extent(cams):
    c = np.stack([cam.campos for cam in cams]).astype(np.float64)
    ctr = c.mean(0)
    return float(1.1 * max(np.linalg.norm(c - ctr, axis=1).max(), 1e-3))


def tiny(seed: int = 0, n: int = 4096, width: int = 128, height: int = 128) -> Scene:
    """BASELINE.json configs[0]: 4,096 Gaussians, one 128x128 camera, SH degree 3."""
    r = rng(seed)
    means = np.stack([r.uniform(-1, 1, n), r.uniform(-1, 1, n), r.uniform(2, 4, n)], 1)
    ls = _log_scales(r, n, 0.03, 0.5)
    opac = (2.0 * r.standard_normal(n)).astype(np.float32)
    theta = _assemble(r, means, ls, opac)
    f = width / (2 * 0.5)
    cam = make_camera(np.eye(3), [0, 0, 0], width, height, f, f, bg=(0.2, 0.4, 0.6))
    return Scene("tiny", n, theta, [cam], 3, _extent([cam]))


def ring_cameras(n_cams, radius, height, target, width, fx, img_h, bg=(0, 0, 0)):
    cams = []
    for i in range(n_cams):
        a = 2 * np.pi * i / n_cams
        pos = [radius * np.cos(a), height, radius * np.sin(a)]
        cams.append(look_at(pos, target, width, img_h, fx, fx, bg=bg))
    return cams


def garden(seed: int = 1, n: int = 5_800_000, n_cams: int = 64) -> Scene:
    """Mip-NeRF360 'garden'-shaped: 1237x822, fx = fy = 1150, ring of cameras."""
    r = rng(seed)
    n_obj, n_gnd = int(0.5 * n), int(0.3 * n)
    n_bg = n - n_obj - n_gnd
    k = n_obj // 3
    obj = np.concatenate([
        _on_ellipsoid(r, k, (-0.30, -0.40, 0.10), (0.35, 0.40, 0.35)),
        _on_box(r, k, (0.35, -0.50, -0.20), (0.25, 0.30, 0.25)),
        _on_ellipsoid(r, n_obj - 2 * k, (0.05, -0.10, 0.35), (0.20, 0.25, 0.20)),
    ])
    obj += 0.004 * r.standard_normal(obj.shape)
    gnd = _ground(r, n_gnd, -0.8, 8.0)
    bgp = _shell(r, n_bg, 10.0, 30.0)
    means = np.concatenate([obj, gnd, bgp]).astype(np.float32)
    ls = np.concatenate([
        _log_scales(r, n_obj, 0.004, 0.5, 0.25),
        _log_scales(r, n_gnd, 0.02, 0.6, 0.25),
        _log_scales(r, n_bg, 0.25, 0.7),
    ])
    theta = _assemble(r, means, ls, _opacity_bimodal(r, n))
    cams = ring_cameras(n_cams, 3.0, 1.2, (0, -0.3, 0), 1237, 1150.0, 822)
    return Scene("garden", n, theta, cams, 3, _extent(cams))


def tandt_train(seed: int = 1, n: int = 1_100_000, n_cams: int = 64) -> Scene:
    """Tanks&Temples 'train'-shaped: 980x545, fx = fy = 0.9 W."""
    r = rng(seed)
    n_obj, n_gnd = int(0.55 * n), int(0.30 * n)
    n_bg = n - n_obj - n_gnd
    obj = _on_box(r, n_obj, (0, 0, 0), (2.0, 0.4, 0.4)) + 0.005 * r.standard_normal((n_obj, 3))
    gnd = _ground(r, n_gnd, -0.4, 10.0)
    bgp = _shell(r, n_bg, 12.0, 40.0)
    means = np.concatenate([obj, gnd, bgp]).astype(np.float32)
    ls = np.concatenate([
        _log_scales(r, n_obj, 0.006, 0.5, 0.25),
        _log_scales(r, n_gnd, 0.02, 0.6, 0.25),
        _log_scales(r, n_bg, 0.3, 0.7),
    ])
    theta = _assemble(r, means, ls, _opacity_bimodal(r, n))
    cams = ring_cameras(n_cams, 5.0, 1.2, (0, 0, 0), 980, 0.9 * 980, 545)
    return Scene("tandt_train", n, theta, cams, 3, _extent(cams))


def db_playroom(seed: int = 1, n: int = 2_300_000, n_cams: int = 64) -> Scene:
    """Deep Blending 'playroom'-shaped: 1264x832, fx = fy = 0.75 W, cameras inside a room."""
    r = rng(seed)
    n_room = int(0.55 * n)
    n_furn = n - n_room
    room = _on_box(r, n_room, (0, 1.5, 0), (4.0, 1.5, 3.0))
    per = n_furn // 10
    furn = []
    for i in range(10):
        m = per if i < 9 else n_furn - 9 * per
        c = (r.uniform(-3.2, 3.2), r.uniform(0.3, 1.0), r.uniform(-2.4, 2.4))
        h = (r.uniform(0.2, 0.6), r.uniform(0.2, 0.6), r.uniform(0.2, 0.6))
        furn.append(_on_box(r, m, c, h))
    means = np.concatenate([room] + furn).astype(np.float32)
    ls = np.concatenate([_log_scales(r, n_room, 0.01, 0.6, 0.25), _log_scales(r, n_furn, 0.008, 0.5, 0.25)])
    theta = _assemble(r, means, ls, _opacity_bimodal(r, n))
    cams = []
    for i in range(n_cams):
        pos = np.array([r.uniform(-1, 1), 1.5, r.uniform(-1, 1)])
        yaw = r.uniform(0, 2 * np.pi)
        tgt = pos + np.array([np.cos(yaw), 0.0, np.sin(yaw)])
        cams.append(look_at(pos, tgt, 1264, 832, 0.75 * 1264, 0.75 * 1264))
    return Scene("db_playroom", n, theta, cams, 3, _extent(cams))


CONFIGS = {"tiny": tiny, "tandt_train": tandt_train, "db_playroom": db_playroom, "garden": garden}


def make(name: str, seed: int | None = None, **kw) -> Scene:
    fn = CONFIGS[name]
    return fn(**kw) if seed is None else fn(seed=seed, **kw)


def small_scene(seed: int, n: int, width: int, height: int, sh_degree: int = 3,
                depth=(2.0, 4.0), scale_mu=0.05, bg=(0.2, 0.4, 0.6), spread=1.0) -> Scene:
    """Parametric small scene for the parity tests (several tiles and a ragged tail)."""
    r = rng(seed)
    tanx = 0.5
    f = width / (2 * tanx)
    ext_x = spread * tanx * depth[0]
    ext_y = spread * (height / (2 * f)) * depth[0]
    means = np.stack([r.uniform(-ext_x, ext_x, n), r.uniform(-ext_y, ext_y, n),
                      r.uniform(depth[0], depth[1], n)], 1)
    ls = _log_scales(r, n, scale_mu, 0.6)
    theta = _assemble(r, means, ls, _opacity_bimodal(r, n))
    cam = make_camera(np.eye(3), [0, 0, 0], width, height, f, f, bg=bg)
    return Scene(f"small{n}_{width}x{height}", n, theta, [cam], sh_degree, 1.0)


def random_dl_dimage(seed: int, width: int, height: int, scale: float = 1.0) -> np.ndarray:
    """A seeded upstream gradient dL/dimage [3][H][W] for parity tests."""
    return (scale * rng(seed).standard_normal((3, height, width))).astype(np.float32)
