"""Plan-ahead of the blend schedules (bgs_render_fwd_plan / bgs_blend_bwd_plan): building a
frame's forward work units with its sort on another stream, and its backward units beside
the loss, changes nothing in the results; a plan made stale by a later call is discarded."""
import numpy as np
import pytest

import gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bgs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_14564_b200 as m

    return m


def step(bgs, r, g, cam, theta, dl, grad, ahead, seg_len=None, hint=None):
    """preprocess, sort, fwd, bwd of one view; `ahead`: both plans built on a side stream"""
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    bgs.bgs_preprocess(g, bgs.camera(cam), r.frame)
    if hint is not None:
        bgs.bgs_frame_load_hint(r.frame, hint)
    bgs.bgs_sort(r.frame)
    if seg_len is not None:
        bgs.bgs_frame_set_seg_len(r.frame, seg_len)
    if ahead:
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            bgs.bgs_render_fwd_plan(r.frame)
        main.wait_stream(side)
    bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib)
    if ahead:
        side.wait_stream(main)
        with torch.cuda.stream(side):
            bgs.bgs_blend_bwd_plan(r.frame)
        main.wait_stream(side)
    bgs.bgs_blend_bwd(r.frame, dl, r.final_T, r.n_contrib)
    grad.zero_()
    bgs.bgs_preprocess_bwd(g, r.frame, grad)
    torch.cuda.synchronize()
    return r.image.clone(), r.n_contrib.clone(), grad.clone()


@pytest.mark.parametrize("seg_len", [4096, 64])
def test_plan_ahead_equals_inline(bgs, seg_len):
    s = gen.small_scene(31, 6000, 192, 128, scale_mu=0.06, depth=(2.0, 2.5))
    cam = s.cameras[0]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    dl = torch.from_numpy(gen.random_dl_dimage(3, cam.width, cam.height)).to(dev)
    grad = torch.zeros_like(theta)
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 22, device=dev)
    bgs.bgs_frame_set_seg_len(r.frame, seg_len)
    r.forward(theta, cam, s.sh_degree)  # a hint for the split schedule
    hint = torch.empty(bgs.bgs_frame_hint_bytes(r.frame), dtype=torch.uint8, device=dev)
    bgs.bgs_frame_save_hint(r.frame, hint)
    i0, n0, g0 = step(bgs, r, g, cam, theta, dl, grad, ahead=False, hint=hint)
    i1, n1, g1 = step(bgs, r, g, cam, theta, dl, grad, ahead=True, hint=hint)
    assert torch.equal(i0, i1) and torch.equal(n0, n1)
    # the backward's REDs add in hardware order: equal to float rounding
    rel = float(torch.linalg.vector_norm(g1 - g0) / torch.linalg.vector_norm(g0))
    assert rel <= 1e-5


def test_stale_plans_are_discarded(bgs):
    """A forward plan built for seg_len 4096 must not drive a forward at seg_len 64 (set
    after it), and a backward plan must not outlive the forward it was built from."""
    s = gen.small_scene(32, 6000, 192, 128, scale_mu=0.06, depth=(2.0, 2.5))
    cam = s.cameras[0]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    dl = torch.from_numpy(gen.random_dl_dimage(4, cam.width, cam.height)).to(dev)
    grad = torch.zeros_like(theta)
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 22, device=dev)
    bgs.bgs_frame_set_seg_len(r.frame, 64)
    r.forward(theta, cam, s.sh_degree)
    ref = step(bgs, r, g, cam, theta, dl, grad, ahead=False, seg_len=64)
    # plan at the default seg_len, then change it: the forward replans
    bgs.bgs_frame_set_seg_len(r.frame, 4096)
    bgs.bgs_preprocess(g, bgs.camera(cam), r.frame)
    bgs.bgs_sort(r.frame)
    bgs.bgs_render_fwd_plan(r.frame)
    bgs.bgs_frame_set_seg_len(r.frame, 64)
    bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib)
    bgs.bgs_blend_bwd_plan(r.frame)
    bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib)  # discards that backward plan
    bgs.bgs_blend_bwd(r.frame, dl, r.final_T, r.n_contrib)
    grad.zero_()
    bgs.bgs_preprocess_bwd(g, r.frame, grad)
    torch.cuda.synchronize()
    assert torch.equal(r.image, ref[0]) and torch.equal(r.n_contrib, ref[1])
    rel = float(torch.linalg.vector_norm(grad - ref[2]) / torch.linalg.vector_norm(ref[2]))
    assert rel <= 1e-5
    assert np.isfinite(grad.cpu().numpy()).all()


def test_consuming_frame_equals_default(bgs):
    """bgs_frame_set_consume: the chain rule zeroes the blend gradients it reads and the next
    preprocess skips zeroing them -- two training steps give the same gradients as the
    default frame, the slots are zero after each chain rule, and a second chain rule over
    the same backward adds nothing."""
    s = gen.small_scene(33, 5000, 160, 128, scale_mu=0.05)
    cam = s.cameras[0]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    dl = torch.from_numpy(gen.random_dl_dimage(5, cam.width, cam.height)).to(dev)
    outs = []
    for consume in (False, True):
        r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 22, device=dev)
        bgs.bgs_frame_set_consume(r.frame, consume)
        grads = []
        for it in range(2):
            grad = torch.zeros_like(theta)
            bgs.bgs_preprocess(g, bgs.camera(cam), r.frame)
            bgs.bgs_sort(r.frame)
            bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib)
            bgs.bgs_blend_bwd(r.frame, dl, r.final_T, r.n_contrib)
            bgs.bgs_preprocess_bwd_batch(g, [r.frame], grad)
            torch.cuda.synchronize()
            grads.append(grad.clone())
            v = r.views()
            g2 = torch.as_tensor(_DevPtr(v.grad2d, 12 * s.n, "<f4"), device="cuda")
            assert bool((g2 == 0).all()) == consume
            if consume and it == 1:
                again = torch.zeros_like(theta)
                bgs.bgs_preprocess_bwd_batch(g, [r.frame], again)
                torch.cuda.synchronize()
                assert not bool(again.any())
        outs.append(grads)
    for a, b in zip(*outs):
        rel = float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(a))
        assert rel <= 1e-5


class _DevPtr:
    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}
