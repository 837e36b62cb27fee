"""Workload for compute-sanitizer (tests/test_gpu_sanitizer.py): every libbgs kernel on small
inputs that still exercise the delicate synchronisation -- decoupled look-back scans and
onesweep passes (several tiles), ticket-ordered persistent blend grids, the forward's
speculative split walks and their merges (a small seg_len forces them), the backward's
checkpoint segments, the batched preprocess / chain rule, Adam, the loss kernels, the
density step with its rounds, and the importance sampling.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [tiny|garden20k]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


def scene(which):
    if which == "tiny":
        return gen.tiny()
    return gen.garden(seed=3, n=20_000, n_cams=2)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    s = scene(which)
    cam = s.cameras[0]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    W, H = cam.width, cam.height
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    # every sort path, hinted and unhinted forwards, split walks (seg_len 64)
    flags = [0, bgs.BGS_DEBUG_SORT_RADIX_SPLIT, bgs.BGS_DEBUG_SORT_ONESWEEP64, bgs.BGS_DEBUG_SORT_ROWSPLIT,
             bgs.BGS_DEBUG_BWD_8X4, bgs.BGS_DEBUG_PARITY_EXP]
    grad = torch.zeros_like(theta)
    dl = torch.full((3, H, W), 1e-3, device=dev)
    for f in flags:
        r = bgs.Renderer(s.n, W, H, max_keys=1 << 20, device=dev, debug_flags=f)
        bgs.bgs_frame_set_seg_len(r.frame, 64)
        for _ in range(2):  # the second forward is hinted (splits long walks)
            out = r.forward(theta, cam, s.sh_degree)
        r.backward(theta, s.sh_degree, dl, out, grad)
        rep = bgs.validate(r.frame)  # failure detection: the list check ...
        assert rep["member_errors"] == rep["order_errors"] == rep["range_errors"] == 0, rep
    assert bgs.nonfinite(grad)[0] == 0  # ... and the non-finite check
    # the bench's batched form: one preprocess for two views, loss, blend bwd, batched chain rule
    rs = [bgs.Renderer(s.n, W, H, max_keys=1 << 20, device=dev) for _ in range(2)]
    cams = [bgs.camera(c) for c in s.cameras[:2]] if len(s.cameras) > 1 else [bgs.camera(cam)] * 2
    for _ in range(2):
        bgs.bgs_preprocess_batch(g, cams, [x.frame for x in rs])
        for x in rs:
            bgs.bgs_sort(x.frame)
            bgs.bgs_render_fwd(x.frame, x.image, x.final_T, x.n_contrib)
    tgt = (torch.rand((3, H, W), device=dev) * 255).to(torch.uint8)
    ws = torch.empty(bgs.bgs_loss_workspace_bytes(W, H), dtype=torch.uint8, device=dev)
    loss = torch.zeros(1, device=dev)
    dl2 = torch.empty_like(rs[0].image)
    bgs.bgs_l1_dssim_loss_grad(rs[0].image, tgt, W, H, 0.2, 0.5, dl2, loss, ws)
    bgs.bgs_l1_loss_grad(rs[1].image, tgt, W, H, 1.0 / (3 * W * H), dl2, loss)
    for x in rs:
        bgs.bgs_blend_bwd(x.frame, dl2, x.final_T, x.n_contrib)
    bgs.bgs_preprocess_bwd_batch(g, [x.frame for x in rs], grad)
    m = torch.zeros_like(theta)
    v = torch.zeros_like(theta)
    bgs.adam_step(theta, grad, m, v, s.n, bgs.AdamHParams(), step=1)
    half = (59 * s.n // 2) // 4 * 4  # a 16-byte aligned shard, as the sharded update's
    bgs.bgs_adam_step_range(theta[half:], grad[half:], m[half:], v[half:], s.n, half, 59 * s.n - half,
                            bgs.AdamHParams(), 2)
    # NEXT-1: density step with rounds; NEXT-3/4: importance, keep mask, masked render
    mu = theta[: 3 * s.n].view(s.n, 3)
    from scipy.spatial import cKDTree
    pts = mu.cpu().numpy().astype(np.float64)
    r8 = float(np.median(cKDTree(pts).query(pts, k=9)[0][:, 8]))
    gen_ = torch.Generator(device=dev)
    gen_.manual_seed(1)
    bgs.density_control(theta, m, v, s.n, bgs.DensityParams(r8), gen_, max_rounds=3)
    r = rs[0]
    imp, _ = bgs.bgs_importance(r.frame, r.image, s.n)
    keep = bgs.bgs_importance_keep(imp, 0.5)
    bgs.bgs_frame_set_keep(r.frame, keep)
    r.forward(theta, cam, s.sh_degree)
    bgs.bgs_frame_set_keep(r.frame, None)
    torch.cuda.synchronize()
    print("sanitize workload done:", which, "launches", bgs.launch_count())


if __name__ == "__main__":
    main()
