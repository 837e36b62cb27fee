"""Preprocess probe (not the bench): times bgs_preprocess_batch over a step's views against
one bgs_preprocess per view on the garden scene (CUDA events, after a warm-up)."""
import argparse
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
    a = ap.parse_args()
    s = gen.make(a.config)
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    g = bgs.gaussians(theta, s.n, s.sh_degree)
    cams = [s.cameras[(4 * i) % len(s.cameras)] for i in range(a.views)]
    cs = [bgs.camera(c) for c in cams]
    rs = [bgs.Renderer(s.n, c.width, c.height, max_keys=1 << 20, device=dev) for c in cams]
    frames = [r.frame for r in rs]

    def per_view():
        for c, f in zip(cs, frames):
            bgs.bgs_preprocess(g, c, f)

    def batch():
        bgs.bgs_preprocess_batch(g, cs, frames)

    for name, fn in (("per_view", per_view), ("batch", batch)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:9s} {e0.elapsed_time(e1) / a.reps:.3f} ms for {a.views} views", flush=True)


if __name__ == "__main__":
    main()
