"""NEXT-4: render-only novel-view serving on the garden scene -- a2-a7
(preprocess, sort, blend forward) per view, views/s from CUDA events -- exact, and with the
per-view importance table (NEXT-3, bgs_importance) retained to skip Gaussians
(bgs_importance_keep + bgs_frame_set_keep), with PSNR against the exact
render.  Prints one JSON line (also written to --out)."""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="garden")
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fractions", default="1.0,0.9,0.75,0.5")
    ap.add_argument("--out", default=None)
    ap.add_argument("--per-view-preprocess", action="store_true",
                    help="one preprocess launch per view instead of one per 16 views")
    a = ap.parse_args()
    s = gen.make(a.config)
    cams = [s.cameras[(4 * i) % len(s.cameras)] for i in range(a.views)]
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    W, H = cams[0].width, cams[0].height
    rs = [bgs.Renderer(s.n, W, H, max_keys=1 << 26, device=dev) for _ in cams]
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    cs = [bgs.camera(c) for c in cams]

    frames = [r.frame for r in rs]

    def render_all():
        if not a.per_view_preprocess:  # the batch's views share theta: one pass over it
            bgs.bgs_preprocess_batch(g, cs, frames)
        for r, c in zip(rs, cs):
            if a.per_view_preprocess:
                bgs.bgs_preprocess(g, c, r.frame)
            bgs.bgs_sort(r.frame)
            bgs.bgs_render_fwd(r.frame, r.image, r.final_T, r.n_contrib)

    def timed():
        render_all()  # warm-up (and the frames' scheduling hints)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            render_all()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (a.reps * len(rs))

    for r, c in zip(rs, cams):  # size the key capacity (R25)
        r.forward(theta, c, s.sh_degree)
    exact_ms = timed()
    exact = [r.image.clone() for r in rs]
    # the importance table per viewpoint, from the exact render (NEXT-3)
    imps = [bgs.bgs_importance(r.frame, r.image, s.n)[0] for r in rs]
    rows = [{"fraction": 1.0, "ms_per_view": round(exact_ms, 4), "views_per_s": round(1e3 / exact_ms, 2),
             "psnr_db": None, "kept": s.n}]
    cases = [(float(x), True) for x in a.fractions.split(",")] + [(0.5, False)]
    for f, invert in cases:
        if f >= 1.0:
            continue
        # R40: invert=True keeps the highest scores; invert=False is SPEC's ascending rule
        keeps = [bgs.bgs_importance_keep(imp, f, invert=invert) for imp in imps]
        for r, k in zip(rs, keeps):
            bgs.bgs_frame_set_keep(r.frame, k)
        ms = timed()
        mse = sum(float(((r.image.clamp(0, 1) - e.clamp(0, 1)) ** 2).mean()) for r, e in zip(rs, exact)) / len(rs)
        rows.append({"fraction": f, "keep": "highest" if invert else "lowest (SPEC ascending)",
                     "ms_per_view": round(ms, 4), "views_per_s": round(1e3 / ms, 2),
                     "psnr_db": round(10 * math.log10(1.0 / max(mse, 1e-20)), 2),
                     "kept": int(keeps[0].sum().item())})
        for r in rs:
            bgs.bgs_frame_set_keep(r.frame, None)
    line = {"workload": f"{s.name}-shaped {s.n} Gaussians, {W}x{H}, render-only (a2-a7), {len(rs)} views",
            "preprocess": "one launch per view" if a.per_view_preprocess else "batched over the views",
            "keep_rule": "per-view importance I_g (R40)", "rows": rows}
    print(json.dumps(line))
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
