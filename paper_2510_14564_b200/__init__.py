"""Thin Python binding of libbgs (include/bgs.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libbgs.so (sm_100a); PyTorch only
provides device memory, streams and (in bench.py) the NCCL process group.  There is no
CPU or PyTorch fallback: importing this package without the built library raises.

Names follow the C ABI: bgs_preprocess / bgs_sort / bgs_render_fwd / bgs_render_bwd /
bgs_adam_step (BASELINE.json north_star), plus the l1 helper, status and debug calls.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BGS_LIB") or os.path.join(_HERE, "libbgs.so")  # BGS_LIB: A/B builds (tools/)
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbgs.so not built at {LIB_PATH}: run `python __graft_entry__.py` (build()) first")
_lib = C.CDLL(LIB_PATH)

BGS_OK, BGS_ERR_INVALID, BGS_ERR_CAPACITY, BGS_ERR_CUDA, BGS_ERR_UNSUPPORTED = 0, -1, -2, -3, -4
BGS_DEBUG_SKIP_SORT = 1
BGS_DEBUG_SORT_ONESWEEP64 = 2
BGS_DEBUG_SORT_RADIX_SPLIT = 4
BGS_DEBUG_BWD_8X4 = 8
BGS_DEBUG_SORT_ROWSPLIT = 16
BGS_DEBUG_PARITY_EXP = 64
BGS_DEBUG_SQUARE_RECT = 128


class BgsError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = _lib.bgs_status_string(status).decode()
        super().__init__(f"{what}: {msg} (status {status})")
        self.status = status


class Gaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("_pad", C.c_int32), ("means", C.c_void_p),
                ("log_scales", C.c_void_p), ("quats", C.c_void_p), ("opacity_logits", C.c_void_p),
                ("sh", C.c_void_p)]


class Camera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("proj", C.c_float * 16), ("campos", C.c_float * 3),
                ("tan_fovx", C.c_float), ("tan_fovy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("bg", C.c_float * 3), ("near_plane", C.c_float)]


class AdamHParams(C.Structure):
    _fields_ = [("lr_means", C.c_float), ("lr_log_scales", C.c_float), ("lr_quats", C.c_float),
                ("lr_opacity", C.c_float), ("lr_sh_dc", C.c_float), ("lr_sh_rest", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]

    def __init__(self, lr_means=1.6e-4, lr_log_scales=5e-3, lr_quats=1e-3, lr_opacity=0.05, lr_sh_dc=2.5e-3,
                 lr_sh_rest=1.25e-4, beta1=0.9, beta2=0.999, eps=1e-15):
        # defaults: R21 ([3DGS] learning rates; opacity 0.05, lr_means before the extent scale)
        super().__init__(lr_means, lr_log_scales, lr_quats, lr_opacity, lr_sh_dc, lr_sh_rest, beta1, beta2, eps)


class DensityParams(C.Structure):
    """bgs_density_params (include/bgs.h); defaults per DESIGN.md R31-R36 / SPEC's ledger."""
    _fields_ = [("r", C.c_float), ("alpha", C.c_float), ("beta", C.c_float), ("gamma", C.c_float),
                ("alpha_sigma", C.c_float), ("delta", C.c_float), ("k", C.c_int32), ("max_new", C.c_int32)]

    def __init__(self, r, alpha=1.0, beta=1.0, gamma=1.0, alpha_sigma=1.5, delta=None, k=8, max_new=4):
        super().__init__(r, alpha, beta, gamma, alpha_sigma, 0.1 * r if delta is None else delta, k, max_new)


class DensityReport(C.Structure):
    _fields_ = [("n_in", C.c_int64), ("n_out", C.c_int64), ("n_pairs", C.c_int64), ("n_children", C.c_int64),
                ("mu_rho", C.c_double), ("sigma_rho", C.c_double), ("rho_low", C.c_double),
                ("rho_high", C.c_double), ("mu_d", C.c_double), ("sigma_d", C.c_double), ("d_merge", C.c_double),
                ("n_sparse", C.c_int64)]


class Frame(C.Structure):
    _fields_ = [("opaque", C.c_uint64 * 128)]


class FrameViews(C.Structure):
    _fields_ = [("radius", C.c_void_p), ("depth", C.c_void_p), ("record", C.c_void_p),
                ("tiles_touched", C.c_void_p), ("offsets", C.c_void_p), ("keys_unsorted", C.c_void_p),
                ("values_unsorted", C.c_void_p), ("keys_sorted", C.c_void_p), ("values_sorted", C.c_void_p),
                ("ranges", C.c_void_p), ("grad2d", C.c_void_p), ("n", C.c_int64), ("max_keys", C.c_int64),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("sort_bits", C.c_int32), ("sort_passes", C.c_int32),
                ("sort_mode", C.c_int32), ("_pad", C.c_int32), ("cbits", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("visible", C.c_int64), ("num_keys", C.c_int64), ("evals_fwd", C.c_int64),
                ("evals_bwd", C.c_int64), ("evals_slot", C.c_int64), ("max_list", C.c_int64),
                ("blended", C.c_int64), ("evals_fwd_culled", C.c_int64), ("evals_bwd_culled", C.c_int64)]


_P = C.c_void_p
_SIGS = {
    "bgs_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32, C.c_int64]),
    "bgs_frame_init": (C.c_int, [C.POINTER(Frame), _P, C.c_size_t, C.c_int64, C.c_int32, C.c_int32, C.c_int64]),
    "bgs_preprocess": (C.c_int, [C.POINTER(Gaussians), C.POINTER(Camera), C.POINTER(Frame), _P]),
    "bgs_preprocess_batch": (C.c_int, [C.POINTER(Gaussians), C.POINTER(Camera), C.POINTER(C.POINTER(Frame)),
                                       C.c_int32, _P]),
    "bgs_sort": (C.c_int, [C.POINTER(Frame), _P]),
    "bgs_render_fwd": (C.c_int, [C.POINTER(Frame), _P, _P, _P, _P]),
    "bgs_render_bwd": (C.c_int, [C.POINTER(Gaussians), C.POINTER(Frame), _P, _P, _P, _P, _P]),
    "bgs_blend_bwd": (C.c_int, [C.POINTER(Frame), _P, _P, _P, _P]),
    "bgs_preprocess_bwd": (C.c_int, [C.POINTER(Gaussians), C.POINTER(Frame), _P, _P]),
    "bgs_preprocess_bwd_batch": (C.c_int, [C.POINTER(Gaussians), C.POINTER(C.POINTER(Frame)), C.c_int32, _P, _P]),
    "bgs_preprocess_bwd_batch_assign": (C.c_int, [C.POINTER(Gaussians), C.POINTER(C.POINTER(Frame)), C.c_int32, _P,
                                                 _P]),
    "bgs_preprocess_bwd_batch_range": (C.c_int, [C.POINTER(Gaussians), C.POINTER(C.POINTER(Frame)), C.c_int32, _P, C.c_int64,
                                                C.c_int64, _P]),
    "bgs_preprocess_bwd_batch_adam": (C.c_int, [C.POINTER(Gaussians), C.POINTER(C.POINTER(Frame)), C.c_int32, _P, _P,
                                                _P, _P, C.POINTER(AdamHParams), C.c_int64, _P]),
    "bgs_adam_step": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.POINTER(AdamHParams), C.c_int64, _P]),
    "bgs_adam_step_keep_grad": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.POINTER(AdamHParams), C.c_int64, _P]),
    "bgs_adam_step_range": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.POINTER(AdamHParams),
                                      C.c_int64, _P]),
    "bgs_adam_step_multimem": (C.c_int, [_P, _P, _P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.POINTER(AdamHParams),
                                         C.c_int64, _P]),
    "bgs_zero": (C.c_int, [_P, C.c_int64, _P]),
    "bgs_loss_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "bgs_l1_dssim_loss_grad": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_float, C.c_float, _P, _P, _P, C.c_size_t,
                                         _P]),
    "bgs_l1_loss_grad": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_float, _P, _P, _P]),
    "bgs_frame_status": (C.c_int, [C.POINTER(Frame), C.POINTER(C.c_int64)]),
    "bgs_frame_debug": (C.c_int, [C.POINTER(Frame), C.POINTER(FrameViews)]),
    "bgs_frame_stats": (C.c_int, [C.POINTER(Frame), _P, C.POINTER(Stats), _P]),
    "bgs_frame_validate": (C.c_int, [C.POINTER(Frame), _P, _P]),
    "bgs_render_fwd_plan": (C.c_int, [C.POINTER(Frame), _P]),
    "bgs_frame_set_consume": (C.c_int, [C.POINTER(Frame), C.c_int32]),
    "bgs_blend_bwd_plan": (C.c_int, [C.POINTER(Frame), _P]),
    "bgs_nonfinite": (C.c_int, [_P, C.c_int64, _P, _P]),
    "bgs_frame_set_debug": (C.c_int, [C.POINTER(Frame), C.c_int32]),
    "bgs_frame_set_seg_len": (C.c_int, [C.POINTER(Frame), C.c_int32]),
    "bgs_frame_hint_bytes": (C.c_size_t, [C.POINTER(Frame)]),
    "bgs_frame_save_hint": (C.c_int, [C.POINTER(Frame), _P, _P]),
    "bgs_frame_load_hint": (C.c_int, [C.POINTER(Frame), _P, _P]),
    "bgs_density_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "bgs_local_density": (C.c_int, [_P, C.c_int64, C.c_float, C.c_float, C.c_float, _P, _P, _P, C.c_size_t, _P]),
    "bgs_density_step_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "bgs_density_plan": (C.c_int, [_P, C.c_int64, C.POINTER(DensityParams), _P, C.c_size_t, _P]),
    "bgs_density_result": (C.c_int, [_P, C.c_int64, C.POINTER(DensityReport), C.POINTER(C.c_uint32)]),
    "bgs_density_apply": (C.c_int, [_P, _P, _P, C.c_int64, _P, C.POINTER(DensityParams), _P, _P, C.c_int64, _P, _P,
                                    _P, C.c_int64, _P]),
    "bgs_density_parents": (C.c_int, [_P, C.c_int64, C.POINTER(DensityParams), _P, _P, _P]),
    "bgs_density_round_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "bgs_density_round_plan": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.c_double, C.c_int32, _P, C.c_size_t, _P]),
    "bgs_density_round_result": (C.c_int, [_P, C.c_int64, C.POINTER(C.c_int64)]),
    "bgs_density_round_apply": (C.c_int, [_P, _P, _P, C.c_int64, _P, _P, C.c_int64, _P, C.c_float, _P, _P, C.c_int64,
                                          _P, _P, _P, _P]),
    "bgs_tile_buckets": (C.c_int, [_P, _P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P]),
    "bgs_importance_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "bgs_importance": (C.c_int, [C.POINTER(Frame), _P, _P, _P, _P, C.c_size_t, _P]),
    "bgs_importance_keep": (C.c_int, [_P, C.c_int64, C.c_float, C.c_int32, _P, _P, C.c_size_t, _P]),
    "bgs_frame_set_keep": (C.c_int, [C.POINTER(Frame), _P]),
    "bgs_status_string": (C.c_char_p, [C.c_int]),
    "bgs_last_error": (C.c_char_p, []),
    "bgs_launch_count": (C.c_uint64, []),
    "bgs_version": (C.c_int32, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def _check(st: int, what: str):
    if st != BGS_OK:
        raise BgsError(st, what)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "libbgs takes contiguous CUDA tensors"
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def camera(cam) -> Camera:
    """Marshal a gen.Camera-like object (view/proj column-major) into bgs_camera."""
    c = Camera()
    c.view[:] = [float(x) for x in cam.view]
    c.proj[:] = [float(x) for x in cam.proj]
    c.campos[:] = [float(x) for x in cam.campos]
    c.tan_fovx, c.tan_fovy = float(cam.tan_fovx), float(cam.tan_fovy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.bg[:] = [float(x) for x in cam.bg]
    c.near_plane = float(getattr(cam, "near", 0.2))
    return c


def gaussians(theta: torch.Tensor, n: int, sh_degree: int) -> Gaussians:
    """Views into theta[59n] (layout: include/bgs.h)."""
    assert theta.numel() == 59 * n and theta.dtype == torch.float32
    base = theta.data_ptr()
    return Gaussians(n, sh_degree, 0, base, base + 4 * 3 * n, base + 4 * 6 * n, base + 4 * 10 * n,
                     base + 4 * 11 * n)


# ------------------------------------------------------------------ the ABI, one call each
def bgs_workspace_bytes(n, w, h, max_keys) -> int:
    return int(_lib.bgs_workspace_bytes(n, w, h, max_keys))


def bgs_loss_workspace_bytes(w, h) -> int:
    return int(_lib.bgs_loss_workspace_bytes(w, h))


def bgs_frame_init(frame: Frame, workspace: torch.Tensor, n, w, h, max_keys):
    _check(_lib.bgs_frame_init(C.byref(frame), _ptr(workspace), workspace.numel(), n, w, h, max_keys),
           "bgs_frame_init")


def bgs_preprocess(g: Gaussians, cam: Camera, frame: Frame, stream=None):
    _check(_lib.bgs_preprocess(C.byref(g), C.byref(cam), C.byref(frame), _stream(stream)), "bgs_preprocess")


def bgs_preprocess_batch(g: Gaussians, cams, frames, stream=None):
    """a1-a3 for several views in one pass over theta: cams / frames are equal-length sequences."""
    if len(cams) != len(frames):
        raise ValueError("bgs_preprocess_batch: one camera per frame")
    carr = (Camera * len(cams))(*cams)
    farr = (C.POINTER(Frame) * len(frames))(*[C.pointer(f) for f in frames])
    _check(_lib.bgs_preprocess_batch(C.byref(g), carr, farr, len(frames), _stream(stream)), "bgs_preprocess_batch")


def bgs_sort(frame: Frame, stream=None):
    _check(_lib.bgs_sort(C.byref(frame), _stream(stream)), "bgs_sort")


def bgs_render_fwd(frame: Frame, image, final_T, n_contrib, stream=None):
    _check(_lib.bgs_render_fwd(C.byref(frame), _ptr(image), _ptr(final_T), _ptr(n_contrib), _stream(stream)),
           "bgs_render_fwd")


def bgs_render_bwd(g: Gaussians, frame: Frame, dl_dimage, final_T, n_contrib, grad, stream=None):
    _check(_lib.bgs_render_bwd(C.byref(g), C.byref(frame), _ptr(dl_dimage), _ptr(final_T), _ptr(n_contrib),
                               _ptr(grad), _stream(stream)), "bgs_render_bwd")


def bgs_blend_bwd(frame: Frame, dl_dimage, final_T, n_contrib, stream=None):
    _check(_lib.bgs_blend_bwd(C.byref(frame), _ptr(dl_dimage), _ptr(final_T), _ptr(n_contrib), _stream(stream)),
           "bgs_blend_bwd")


def bgs_preprocess_bwd(g: Gaussians, frame: Frame, grad, stream=None):
    _check(_lib.bgs_preprocess_bwd(C.byref(g), C.byref(frame), _ptr(grad), _stream(stream)), "bgs_preprocess_bwd")


def bgs_preprocess_bwd_batch(g: Gaussians, frames, grad, stream=None):
    """frames: a sequence of Frame structs (one per view of the batch)."""
    arr = (C.POINTER(Frame) * len(frames))(*[C.pointer(f) for f in frames])
    _check(_lib.bgs_preprocess_bwd_batch(C.byref(g), arr, len(frames), _ptr(grad), _stream(stream)),
           "bgs_preprocess_bwd_batch")


def bgs_preprocess_bwd_batch_assign(g: Gaussians, frames, grad, stream=None):
    """The batched chain rule with grad assigned (= the frames' sum; every element written)."""
    arr = (C.POINTER(Frame) * len(frames))(*[C.pointer(f) for f in frames])
    _check(_lib.bgs_preprocess_bwd_batch_assign(C.byref(g), arr, len(frames), _ptr(grad), _stream(stream)),
           "bgs_preprocess_bwd_batch_assign")


def bgs_preprocess_bwd_batch_range(g: Gaussians, frames, grad, begin, count, stream=None):
    """The batched chain rule for the Gaussians [begin, begin + count) only."""
    arr = (C.POINTER(Frame) * len(frames))(*[C.pointer(f) for f in frames])
    _check(_lib.bgs_preprocess_bwd_batch_range(C.byref(g), arr, len(frames), _ptr(grad), int(begin), int(count),
                                               _stream(stream)), "bgs_preprocess_bwd_batch_range")


def bgs_preprocess_bwd_batch_adam(g: Gaussians, frames, theta, grad, exp_avg, exp_avg_sq, hp: AdamHParams,
                                  step: int, stream=None):
    """a10 + a11 in one pass (one GPU): grad may be None for <= 16 frames."""
    arr = (C.POINTER(Frame) * len(frames))(*[C.pointer(f) for f in frames])
    _check(_lib.bgs_preprocess_bwd_batch_adam(C.byref(g), arr, len(frames), _ptr(theta), _ptr(grad), _ptr(exp_avg),
                                              _ptr(exp_avg_sq), C.byref(hp), step, _stream(stream)),
           "bgs_preprocess_bwd_batch_adam")


def bgs_adam_step(theta, grad, exp_avg, exp_avg_sq, n, hp: AdamHParams, step: int, stream=None):
    _check(_lib.bgs_adam_step(_ptr(theta), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), n, C.byref(hp), step,
                              _stream(stream)), "bgs_adam_step")


def bgs_adam_step_keep_grad(theta, grad, exp_avg, exp_avg_sq, n, hp: AdamHParams, step: int, stream=None):
    """bgs_adam_step without zeroing grad (for a step whose chain rule assigns grad)."""
    _check(_lib.bgs_adam_step_keep_grad(_ptr(theta), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), n, C.byref(hp),
                                        step, _stream(stream)), "bgs_adam_step_keep_grad")


def bgs_adam_step_range(theta, grad, exp_avg, exp_avg_sq, n, begin, count, hp: AdamHParams, step: int,
                        stream=None):
    _check(_lib.bgs_adam_step_range(_ptr(theta), _ptr(grad), _ptr(exp_avg), _ptr(exp_avg_sq), n, begin, count,
                                    C.byref(hp), step, _stream(stream)), "bgs_adam_step_range")


def bgs_adam_step_multimem(theta, theta_mc_ptr: int, grad_mc_ptr: int, exp_avg, exp_avg_sq, n, begin, count,
                           hp: AdamHParams, step: int, stream=None):
    """the exchange fused with Adam over NVSwitch multicast addresses
    (theta_mc_ptr / grad_mc_ptr: raw device addresses of the caller's multicast mappings)."""
    _check(_lib.bgs_adam_step_multimem(_ptr(theta), C.c_void_p(theta_mc_ptr), C.c_void_p(grad_mc_ptr), _ptr(exp_avg),
                                       _ptr(exp_avg_sq), n, begin, count, C.byref(hp), step, _stream(stream)),
           "bgs_adam_step_multimem")


def bgs_zero(t, stream=None):
    _check(_lib.bgs_zero(_ptr(t), t.numel(), _stream(stream)), "bgs_zero")


def bgs_l1_dssim_loss_grad(image, target_u8, w, h, lam, scale, dl_dimage, loss_sum, workspace, stream=None):
    """workspace: a uint8 CUDA tensor of >= bgs_loss_workspace_bytes(w, h) bytes (256-B aligned)."""
    _check(_lib.bgs_l1_dssim_loss_grad(_ptr(image), _ptr(target_u8), w, h, lam, scale, _ptr(dl_dimage),
                                       _ptr(loss_sum), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                       _stream(stream)), "bgs_l1_dssim_loss_grad")


def bgs_l1_loss_grad(image, target_u8, w, h, scale, dl_dimage, loss_sum, stream=None):
    _check(_lib.bgs_l1_loss_grad(_ptr(image), _ptr(target_u8), w, h, scale, _ptr(dl_dimage), _ptr(loss_sum),
                                 _stream(stream)), "bgs_l1_loss_grad")


def bgs_frame_status(frame: Frame) -> tuple[int, int]:
    k = C.c_int64(0)
    st = _lib.bgs_frame_status(C.byref(frame), C.byref(k))
    return st, int(k.value)


def bgs_frame_debug(frame: Frame) -> FrameViews:
    v = FrameViews()
    _check(_lib.bgs_frame_debug(C.byref(frame), C.byref(v)), "bgs_frame_debug")
    return v


def bgs_frame_stats(frame: Frame, n_contrib, stream=None) -> dict:
    s = Stats()
    _check(_lib.bgs_frame_stats(C.byref(frame), _ptr(n_contrib), C.byref(s), _stream(stream)), "bgs_frame_stats")
    return {k: int(getattr(s, k)) for k, _ in Stats._fields_}


def bgs_frame_set_consume(frame: Frame, on: bool):
    _check(_lib.bgs_frame_set_consume(C.byref(frame), 1 if on else 0), "bgs_frame_set_consume")


def bgs_render_fwd_plan(frame: Frame, stream=None):
    _check(_lib.bgs_render_fwd_plan(C.byref(frame), _stream(stream)), "bgs_render_fwd_plan")


def bgs_blend_bwd_plan(frame: Frame, stream=None):
    _check(_lib.bgs_blend_bwd_plan(C.byref(frame), _stream(stream)), "bgs_blend_bwd_plan")


VALIDATE_KEYS = ("range_errors", "member_errors", "order_errors", "count_error", "tiles_touched")


def bgs_frame_validate(frame: Frame, out: torch.Tensor, stream=None):
    """Asynchronous structural check of the frame's sorted lists into out (device int64[5])."""
    assert out.dtype == torch.int64 and out.numel() >= 5
    _check(_lib.bgs_frame_validate(C.byref(frame), _ptr(out), _stream(stream)), "bgs_frame_validate")


def validate(frame: Frame, stream=None) -> dict:
    """bgs_frame_validate, synchronised: the five counts by name (all errors 0: lists exact)."""
    out = torch.empty(5, dtype=torch.int64, device="cuda")
    bgs_frame_validate(frame, out, stream)
    return dict(zip(VALIDATE_KEYS, (int(x) for x in out.cpu())))


def bgs_nonfinite(x: torch.Tensor, out: torch.Tensor, stream=None):
    """Asynchronous: out (device int64[2]) = {NaN/Inf count, smallest such index or -1}."""
    assert x.dtype == torch.float32 and out.dtype == torch.int64 and out.numel() >= 2
    _check(_lib.bgs_nonfinite(_ptr(x), x.numel(), _ptr(out), _stream(stream)), "bgs_nonfinite")


def nonfinite(x: torch.Tensor, stream=None) -> tuple[int, int]:
    """bgs_nonfinite, synchronised: (count, first index or -1)."""
    out = torch.empty(2, dtype=torch.int64, device=x.device)
    bgs_nonfinite(x, out, stream)
    c, f = (int(v) for v in out.cpu())
    return c, (f if c else -1)


def bgs_frame_set_debug(frame: Frame, flags: int):
    _check(_lib.bgs_frame_set_debug(C.byref(frame), flags), "bgs_frame_set_debug")


def bgs_frame_set_seg_len(frame: Frame, seg_len: int):
    _check(_lib.bgs_frame_set_seg_len(C.byref(frame), seg_len), "bgs_frame_set_seg_len")


def bgs_local_density(means, r, alpha=1.0, beta=1.0, counts=None, stats=None, workspace=None, stream=None):
    """NEXT-1 / T1 (§III-C1): exact fixed-radius neighbour counts + thresholds.
    means: contiguous CUDA float32 [n, 3] (or the means segment of theta)."""
    n = means.numel() // 3
    dev = means.device
    if counts is None:
        counts = torch.empty(n, dtype=torch.int32, device=dev)
    if stats is None:
        stats = torch.empty(4, dtype=torch.float64, device=dev)
    nbytes = int(_lib.bgs_density_workspace_bytes(n))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    _check(_lib.bgs_local_density(_ptr(means), n, float(r), float(alpha), float(beta), _ptr(counts), _ptr(stats),
                                  _ptr(workspace), workspace.numel(), _stream(stream)), "bgs_local_density")
    return counts, stats


def density_control(theta, exp_avg, exp_avg_sq, n, params: DensityParams, generator=None, stream=None,
                    max_rounds=4):
    """One NEXT-1 density-control step (§III-C2-C4): plan on the device, one host
    read of the report (n_out sizes the new buffers), the method's random draws
    (N(0,1) / U(-1,1) variates, torch generator on the device), apply; then up to
    max_rounds - 1 further densification rounds (R35', "repeated iteratively until the
    desired density is achieved", l.206): the sparse points' local densities re-counted over
    the grown scene, more children for those still below rho_low.  Returns (theta',
    exp_avg', exp_avg_sq', n', report, short_knn, draws), short_knn = points with fewer than
    k neighbours within 3 r (R32), draws = [(normals, uniforms)] per round, and sets
    report.rounds / report.children_per_round (Python attributes)."""
    dev = theta.device
    nbytes = int(_lib.bgs_density_step_workspace_bytes(n))
    if nbytes == 0:
        raise BgsError(BGS_ERR_INVALID, "bgs_density_step_workspace_bytes")
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _check(_lib.bgs_density_plan(_ptr(theta), n, C.byref(params), _ptr(ws), nbytes, _stream(stream)),
           "bgs_density_plan")
    rep = DensityReport()
    short = C.c_uint32(0)

    def sync():
        torch.cuda.current_stream(dev).synchronize() if stream is None else stream.synchronize()

    sync()
    _check(_lib.bgs_density_result(_ptr(ws), n, C.byref(rep), C.byref(short)), "bgs_density_result")
    nc, n_out = int(rep.n_children), int(rep.n_out)

    def draws(count):
        z = torch.randn((max(count, 1), 3), generator=generator, device=dev)
        u = torch.rand((max(count, 1), 3), generator=generator, device=dev) * 2.0 - 1.0
        return z, u

    normals, uniforms = draws(nc)
    th2 = torch.empty(59 * n_out, dtype=torch.float32, device=dev)
    m2, v2 = torch.empty_like(th2), torch.empty_like(th2)
    _check(_lib.bgs_density_apply(_ptr(theta), _ptr(exp_avg), _ptr(exp_avg_sq), n, _ptr(ws), C.byref(params),
                                  _ptr(normals), _ptr(uniforms), nc, _ptr(th2), _ptr(m2), _ptr(v2), n_out,
                                  _stream(stream)), "bgs_density_apply")
    rounds = [(normals[:nc], uniforms[:nc])]
    per_round = [nc]
    npar = int(rep.n_sparse)
    if max_rounds > 1 and npar > 0 and params.max_new > 0:
        parents = torch.empty(npar, dtype=torch.int32, device=dev)
        sigma = torch.empty(npar, dtype=torch.float64, device=dev)
        _check(_lib.bgs_density_parents(_ptr(ws), n, C.byref(params), _ptr(parents), _ptr(sigma), _stream(stream)),
               "bgs_density_parents")
        rws = torch.empty(max(int(_lib.bgs_density_round_workspace_bytes(npar)), 256), dtype=torch.uint8, device=dev)
        for _ in range(max_rounds - 1):
            rho, _st = bgs_local_density(th2[:3 * n_out].view(n_out, 3), params.r, params.alpha, params.beta,
                                         stream=stream)
            _check(_lib.bgs_density_round_plan(_ptr(rho), n_out, _ptr(parents), npar, float(rep.rho_low),
                                               params.max_new, _ptr(rws), rws.numel(), _stream(stream)),
                   "bgs_density_round_plan")
            sync()
            kc = C.c_int64(0)
            _check(_lib.bgs_density_round_result(_ptr(rws), npar, C.byref(kc)), "bgs_density_round_result")
            kc = int(kc.value)
            if kc == 0:  # every sparse point reached rho_low
                break
            z, u = draws(kc)
            n3 = n_out + kc
            th3 = torch.empty(59 * n3, dtype=torch.float32, device=dev)
            m3, v3 = torch.empty_like(th3), torch.empty_like(th3)
            _check(_lib.bgs_density_round_apply(_ptr(th2), _ptr(m2), _ptr(v2), n_out, _ptr(parents), _ptr(sigma), npar,
                                                _ptr(rws), params.delta, _ptr(z), _ptr(u), kc, _ptr(th3), _ptr(m3),
                                                _ptr(v3), _stream(stream)), "bgs_density_round_apply")
            th2, m2, v2, n_out = th3, m3, v3, n3
            rounds.append((z[:kc], u[:kc]))
            per_round.append(kc)
    rep.rounds = len(per_round)
    rep.children_per_round = per_round
    return th2, m2, v2, n_out, rep, int(short.value), rounds


def bgs_tile_buckets(image, final_T, w, h, stream=None):
    """NEXT-3 (§IV-C1): per-tile colour buckets -> (nb, keys, counts, color_sum, opacity_sum)."""
    dev = image.device
    nt = ((w + 15) // 16) * ((h + 15) // 16)
    nb = torch.empty(nt, dtype=torch.int32, device=dev)
    keys = torch.empty(nt * 256, dtype=torch.int16, device=dev)
    counts = torch.empty(nt * 256, dtype=torch.int32, device=dev)
    csum = torch.empty(nt * 256 * 3, dtype=torch.float32, device=dev)
    osum = torch.empty(nt * 256, dtype=torch.float32, device=dev)
    _check(_lib.bgs_tile_buckets(_ptr(image), _ptr(final_T), w, h, _ptr(nb), _ptr(keys), _ptr(counts), _ptr(csum),
                                 _ptr(osum), _stream(stream)), "bgs_tile_buckets")
    return nb, keys, counts, csum, osum


def bgs_importance(frame: Frame, image, n, workspace=None, stream=None):
    """NEXT-3 (§IV-C3): (importance [n], N_g [n]) for the frame's last render."""
    dev = image.device
    nbytes = int(_lib.bgs_importance_workspace_bytes(n))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    imp = torch.empty(n, dtype=torch.float32, device=dev)
    cnt = torch.empty(n, dtype=torch.int32, device=dev)
    _check(_lib.bgs_importance(C.byref(frame), _ptr(image), _ptr(imp), _ptr(cnt), _ptr(workspace),
                               workspace.numel(), _stream(stream)), "bgs_importance")
    return imp, cnt


def bgs_importance_keep(importance, fraction, invert=False, workspace=None, stream=None):
    """R40: the keep mask (uint8 [n]) of the first ceil(fraction n) Gaussians by importance."""
    n = importance.numel()
    dev = importance.device
    nbytes = int(_lib.bgs_importance_workspace_bytes(n))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    keep = torch.empty(n, dtype=torch.uint8, device=dev)
    _check(_lib.bgs_importance_keep(_ptr(importance), n, float(fraction), int(bool(invert)), _ptr(keep),
                                    _ptr(workspace), workspace.numel(), _stream(stream)), "bgs_importance_keep")
    return keep


# device buffers a frame keeps pointers to (the keep mask): held here until replaced or
# cleared, so the caching allocator cannot reuse them while the frame may read them
_FRAME_REFS: dict = {}


def bgs_frame_set_keep(frame: Frame, keep):
    _check(_lib.bgs_frame_set_keep(C.byref(frame), None if keep is None else _ptr(keep)), "bgs_frame_set_keep")
    if keep is None:
        _FRAME_REFS.pop(C.addressof(frame), None)
    else:
        _FRAME_REFS[C.addressof(frame)] = keep


def bgs_frame_hint_bytes(frame: Frame) -> int:
    return int(_lib.bgs_frame_hint_bytes(C.byref(frame)))


def bgs_frame_save_hint(frame: Frame, dst, stream=None):
    _check(_lib.bgs_frame_save_hint(C.byref(frame), _ptr(dst), _stream(stream)), "bgs_frame_save_hint")


def bgs_frame_load_hint(frame: Frame, src, stream=None):
    _check(_lib.bgs_frame_load_hint(C.byref(frame), None if src is None else _ptr(src), _stream(stream)),
           "bgs_frame_load_hint")


def launch_count() -> int:
    return int(_lib.bgs_launch_count())


def last_error() -> str:
    return _lib.bgs_last_error().decode()


adam_step = bgs_adam_step


# ------------------------------------------------------------------ convenience wrapper
@dataclasses.dataclass
class Renderer:
    """One view's workspace (torch-allocated) + frame; forward/backward through the ABI."""
    n: int
    width: int
    height: int
    max_keys: int = 1 << 24
    device: torch.device | str = "cuda"
    debug_flags: int = 0

    def __post_init__(self):
        self.device = torch.device(self.device)
        self.frame = Frame()
        self.alloc(self.max_keys)
        hw = (self.height, self.width)
        self.image = torch.empty((3, *hw), dtype=torch.float32, device=self.device)
        self.final_T = torch.empty(hw, dtype=torch.float32, device=self.device)
        self.n_contrib = torch.empty(hw, dtype=torch.int32, device=self.device)

    def alloc(self, max_keys: int):
        self.max_keys = int(max_keys)
        nbytes = bgs_workspace_bytes(self.n, self.width, self.height, self.max_keys)
        if nbytes == 0:
            raise BgsError(BGS_ERR_INVALID, "bgs_workspace_bytes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        bgs_frame_init(self.frame, self.workspace, self.n, self.width, self.height, self.max_keys)
        if self.debug_flags:
            bgs_frame_set_debug(self.frame, self.debug_flags)

    def forward(self, theta, cam, sh_degree, stream=None, check=True):
        g = gaussians(theta, self.n, sh_degree)
        c = camera(cam)
        bgs_preprocess(g, c, self.frame, stream)
        bgs_sort(self.frame, stream)
        bgs_render_fwd(self.frame, self.image, self.final_T, self.n_contrib, stream)
        if check:
            torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
            st, k = bgs_frame_status(self.frame)
            if st == BGS_ERR_CAPACITY:  # grow and redo (R25)
                self.alloc(max(int(k * 1.25) + 1024, 2 * self.max_keys))
                return self.forward(theta, cam, sh_degree, stream, check)
            _check(st, "bgs_frame_status")
            self.num_keys = k
        return {"image": self.image, "final_T": self.final_T, "n_contrib": self.n_contrib}

    def backward(self, theta, sh_degree, dl_dimage, out, grad, stream=None):
        g = gaussians(theta, self.n, sh_degree)
        bgs_render_bwd(g, self.frame, dl_dimage, out["final_T"], out["n_contrib"], grad, stream)

    def views(self) -> FrameViews:
        return bgs_frame_debug(self.frame)
