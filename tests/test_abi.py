"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/bgs.h
declares, and host-side validation rejects bad calls without launching anything."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bgs.h")


@pytest.fixture(scope="module")
def bgs():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_14564_b200 as m

    return m


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bgs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for fn in ("bgs_preprocess", "bgs_sort", "bgs_render_fwd", "bgs_render_bwd", "bgs_adam_step"):
        assert fn in names


def test_library_exports_every_declared_symbol(bgs):
    out = subprocess.run(["nm", "-D", "--defined-only", bgs.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bgs_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert set(bgs.EXPORTED) <= exported


def test_library_is_sm100a(bgs):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bgs.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_workspace_sizing_and_validation(bgs):
    assert bgs.bgs_workspace_bytes(1000, 128, 128, 1 << 16) > 0
    assert bgs.bgs_workspace_bytes(0, 128, 128, 1 << 16) > 0  # n = 0 is valid
    assert bgs.bgs_workspace_bytes(-1, 128, 128, 1 << 16) == 0
    assert bgs.bgs_workspace_bytes(10, 0, 128, 1 << 16) == 0
    assert bgs.bgs_workspace_bytes(10, 16385, 128, 1 << 16) == 0
    assert bgs.bgs_workspace_bytes(10, 64, 64, 0) == 0
    assert bgs.bgs_workspace_bytes(10, 64, 64, 1 << 30) == 0  # max_keys < 2^30 (R25)
    # monotone in every size
    b = bgs.bgs_workspace_bytes(1000, 128, 128, 1 << 16)
    assert bgs.bgs_workspace_bytes(2000, 128, 128, 1 << 16) > b
    assert bgs.bgs_workspace_bytes(1000, 128, 128, 1 << 17) > b


def test_frame_init_validation_without_device(bgs):
    lib = bgs._lib
    f = bgs.Frame()
    need = bgs.bgs_workspace_bytes(100, 64, 48, 4096)
    fake = C.c_void_p(1 << 40)  # never dereferenced by frame_init
    assert lib.bgs_frame_init(C.byref(f), fake, need, 100, 64, 48, 4096) == bgs.BGS_OK
    assert lib.bgs_frame_init(C.byref(f), fake, need - 1, 100, 64, 48, 4096) == bgs.BGS_ERR_INVALID
    assert lib.bgs_frame_init(C.byref(f), C.c_void_p((1 << 40) + 8), need, 100, 64, 48, 4096) == bgs.BGS_ERR_INVALID
    assert lib.bgs_frame_init(C.byref(f), None, need, 100, 64, 48, 4096) == bgs.BGS_ERR_INVALID
    # a valid frame exposes its geometry through the debug view (no device access)
    assert lib.bgs_frame_init(C.byref(f), fake, need, 100, 64, 48, 4096) == bgs.BGS_OK
    v = bgs.bgs_frame_debug(f)
    assert (v.tiles_x, v.tiles_y, v.n, v.max_keys) == (4, 3, 100, 4096)
    assert v.sort_bits == 32 + 4 and v.sort_passes == 5  # 12 tiles -> bit_width(11) = 4


def test_invalid_calls_launch_nothing(bgs):
    lib = bgs._lib
    before = bgs.launch_count()
    f = bgs.Frame()  # never initialised
    assert lib.bgs_sort(C.byref(f), None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_render_fwd(C.byref(f), None, None, None, None) == bgs.BGS_ERR_INVALID
    hp = bgs.AdamHParams()
    assert lib.bgs_adam_step(None, None, None, None, -1, C.byref(hp), 1, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_adam_step(None, None, None, None, 10, C.byref(hp), 0, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_adam_step(None, None, None, None, 0, C.byref(hp), 1, None) == bgs.BGS_OK  # n = 0: no-op
    assert lib.bgs_adam_step_range(None, None, None, None, 10, 2, 8, C.byref(hp), 1, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_adam_step_range(None, None, None, None, 10, 0, 8, C.byref(hp), 1, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_adam_step_range(None, None, None, None, 10, 592, 8, C.byref(hp), 1, None) == bgs.BGS_OK  # past 59n
    assert lib.bgs_zero(None, 4, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_zero(None, 0, None) == bgs.BGS_OK
    assert bgs.bgs_loss_workspace_bytes(0, 10) == 0 and bgs.bgs_loss_workspace_bytes(64, 32) >= 9 * 64 * 32 * 4
    ws = C.c_void_p(1 << 40)
    need = bgs.bgs_loss_workspace_bytes(64, 32)
    assert lib.bgs_l1_dssim_loss_grad(None, ws, 64, 32, 0.2, 1.0, ws, ws, ws, need, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_l1_dssim_loss_grad(ws, ws, 64, 32, 0.2, 1.0, ws, ws, ws, need - 1, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_l1_dssim_loss_grad(ws, ws, 64, 32, 1.5, 1.0, ws, ws, ws, need, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_l1_dssim_loss_grad(ws, ws, 64, 32, 0.2, 1.0, ws, ws, C.c_void_p((1 << 40) + 16), need,
                                      None) == bgs.BGS_ERR_INVALID  # unaligned workspace
    # preprocess with a camera whose view is not orthonormal
    fake = C.c_void_p(1 << 40)
    need = bgs.bgs_workspace_bytes(4, 32, 32, 64)
    assert lib.bgs_frame_init(C.byref(f), fake, need, 4, 32, 32, 64) == bgs.BGS_OK
    cam = bgs.Camera()
    cam.view[:] = [2.0 if i in (0, 5, 10, 15) else 0.0 for i in range(16)]
    cam.proj[:] = [1.0 if i in (0, 5, 10, 15) else 0.0 for i in range(16)]
    cam.tan_fovx = cam.tan_fovy = 0.5
    cam.width = cam.height = 32
    cam.near_plane = 0.2
    g = bgs.Gaussians(4, 3, 0, 1 << 40, 1 << 40, 1 << 40, 1 << 40, 1 << 40)
    assert lib.bgs_preprocess(C.byref(g), C.byref(cam), C.byref(f), None) == bgs.BGS_ERR_INVALID
    g.sh_degree = 4
    cam.view[:] = [1.0 if i in (0, 5, 10, 15) else 0.0 for i in range(16)]
    assert lib.bgs_preprocess(C.byref(g), C.byref(cam), C.byref(f), None) == bgs.BGS_ERR_INVALID
    g.sh_degree = 3
    g.n = 5  # mismatch with the frame
    assert lib.bgs_preprocess(C.byref(g), C.byref(cam), C.byref(f), None) == bgs.BGS_ERR_INVALID
    # the batched preprocess: same checks per view, plus no frame twice and nframes >= 1
    g.n = 4
    f2 = bgs.Frame()
    assert lib.bgs_frame_init(C.byref(f2), C.c_void_p((1 << 40) + (1 << 30)), need, 4, 32, 32, 64) == bgs.BGS_OK
    cams = (bgs.Camera * 2)(cam, cam)
    twice = (C.POINTER(bgs.Frame) * 2)(C.pointer(f), C.pointer(f))
    both = (C.POINTER(bgs.Frame) * 2)(C.pointer(f), C.pointer(f2))
    assert lib.bgs_preprocess_batch(C.byref(g), cams, twice, 2, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_preprocess_batch(C.byref(g), cams, both, 0, None) == bgs.BGS_ERR_INVALID
    assert lib.bgs_preprocess_batch(C.byref(g), None, both, 2, None) == bgs.BGS_ERR_INVALID
    cams[1].width = 40  # view 1 does not match frame 2
    assert lib.bgs_preprocess_batch(C.byref(g), cams, both, 2, None) == bgs.BGS_ERR_INVALID
    assert bgs.launch_count() == before
    assert "invalid" in lib.bgs_status_string(bgs.BGS_ERR_INVALID).decode()
