"""Per-stage timing probe (not the bench): times each ABI call of one garden view in
isolation, `--reps` back-to-back launches between CUDA events, after a warm-up."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="garden")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--view", type=int, default=0)
    ap.add_argument("--only", default=None, help="comma-separated stage names")
    ap.add_argument("--step", type=int, default=0, help="run N full one-view training steps (for ncu)")
    ap.add_argument("--debug-flags", type=int, default=0, help="frame debug flags (timing experiments)")
    ap.add_argument("--views", type=int, default=1, help="--step: views per step (batched chain rule)")
    ap.add_argument("--seg-lens", default=None, help="comma-separated seg_len values: time fwd/bwd for each")
    a = ap.parse_args()
    t0 = time.time()
    s = gen.make(a.config)
    print(f"gen {time.time() - t0:.1f}s", flush=True)
    cam = s.cameras[a.view]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    grad = torch.zeros_like(theta)
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 26, device=dev, debug_flags=a.debug_flags)
    out = r.forward(theta, cam, s.sh_degree)
    dl = torch.full((3, cam.height, cam.width), 1e-6, device=dev)
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    c = bgs.camera(cam)
    stages = {
        "preprocess": lambda: bgs.bgs_preprocess(g, c, r.frame),
        "sort": lambda: bgs.bgs_sort(r.frame),
        "render_fwd": lambda: bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib),
        "blend_bwd": lambda: bgs.bgs_blend_bwd(r.frame, dl, r.final_T, r.n_contrib),
        "preprocess_bwd": lambda: bgs.bgs_preprocess_bwd(g, r.frame, grad),
    }
    if a.step:
        # one full training step of one view, repeated: preprocess, sort, fwd, L1, bwd, Adam
        m = torch.zeros_like(theta)
        v = torch.zeros_like(theta)
        tgt = torch.zeros((3, cam.height, cam.width), dtype=torch.uint8, device=dev)
        loss = torch.zeros(1, device=dev)
        hp = bgs.AdamHParams()
        vcams = [s.cameras[(a.view + 4 * j) % len(s.cameras)] for j in range(a.views)]
        rs = [r] + [bgs.Renderer(s.n, cam.width, cam.height, max_keys=r.max_keys, device=dev) for _ in vcams[1:]]
        for it in range(a.step):
            if len(rs) > 1:  # as the bench: one preprocess pass over theta for the step's views
                bgs.bgs_preprocess_batch(g, [bgs.camera(cj) for cj in vcams], [rj.frame for rj in rs])
            for rj, cj in zip(rs, vcams):
                if len(rs) == 1:
                    bgs.bgs_preprocess(g, bgs.camera(cj), rj.frame)
                bgs.bgs_sort(rj.frame)
                bgs.bgs_render_fwd(rj.frame, rj.image, rj.final_T, rj.n_contrib)
                bgs.bgs_l1_loss_grad(rj.image, tgt, cam.width, cam.height, 1.0 / (3 * cam.width * cam.height), dl,
                                     loss)
                bgs.bgs_blend_bwd(rj.frame, dl, rj.final_T, rj.n_contrib)
            bgs.bgs_preprocess_bwd_batch(g, [rj.frame for rj in rs], grad)
            bgs.bgs_adam_step(theta, grad, m, v, s.n, hp, it + 1)
        torch.cuda.synchronize()
        print("launches per step:", bgs.launch_count())
        return
    if a.seg_lens:
        for sl in [int(x) for x in a.seg_lens.split(",")]:
            bgs.bgs_frame_set_seg_len(r.frame, sl)
            bgs.bgs_frame_set_debug(r.frame, a.debug_flags)
            res = {}
            for name in ("render_fwd", "blend_bwd"):
                stages["render_fwd"]()  # records this seg_len's checkpoints
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    stages[name]()
                e1.record()
                torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1) / a.reps
            print(f"seg_len {sl:6d}: fwd {res['render_fwd']:.3f} ms  bwd {res['blend_bwd']:.3f} ms", flush=True)
        return
    if a.views > 1:
        # the batched stages as the bench runs them: one a2 launch and one a10 launch over
        # --views views (their frames rendered once first)
        vcams = [s.cameras[(a.view + 4 * j) % len(s.cameras)] for j in range(a.views)]
        rs = [r] + [bgs.Renderer(s.n, cam.width, cam.height, max_keys=r.max_keys, device=dev) for _ in vcams[1:]]
        fr = [rj.frame for rj in rs]
        bcams = [bgs.camera(cj) for cj in vcams]

        def pre_batch():
            bgs.bgs_preprocess_batch(g, bcams, fr)

        pre_batch()
        for rj in rs:
            bgs.bgs_sort(rj.frame)
            bgs.bgs_render_fwd(rj.frame, rj.image, rj.final_T, rj.n_contrib)
            bgs.bgs_blend_bwd(rj.frame, dl, rj.final_T, rj.n_contrib)
        stages["preprocess_batch"] = pre_batch
        stages["preprocess_bwd_batch"] = lambda: bgs.bgs_preprocess_bwd_batch(g, fr, grad)
    only = set(a.only.split(",")) if a.only else None
    for name, fn in stages.items():
        if only and name not in only:
            continue
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        h0 = time.perf_counter()
        for _ in range(a.reps):
            fn()
        host_us = (time.perf_counter() - h0) / a.reps * 1e6
        torch.cuda.synchronize()
        print(f"{name:16s} {ms:8.3f} ms/launch-set   host enqueue {host_us:7.1f} us", flush=True)
    st = bgs.bgs_frame_stats(r.frame, r.n_contrib)
    print(st)


if __name__ == "__main__":
    main()
