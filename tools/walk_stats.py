"""Distribution of per-(tile, 8x4 block) walk lengths (largest n_contrib in the block) of a
garden view: the blend kernels' work-item costs (diagnostic, not the bench)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


def main():
    s = gen.make("garden")
    for view in (0, 8):
        cam = s.cameras[view]
        theta = torch.from_numpy(s.theta).cuda()
        r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 26, device="cuda")
        out = r.forward(theta, cam, s.sh_degree)
        nc = out["n_contrib"].cpu().numpy().view(np.uint32).astype(np.int64)
        H, W = nc.shape
        Hp, Wp = (H + 3) // 4 * 4, (W + 7) // 8 * 8
        pad = np.zeros((Hp, Wp), np.int64)
        pad[:H, :W] = nc
        wl = pad.reshape(Hp // 4, 4, Wp // 8, 8).max(axis=(1, 3)).ravel()
        steps = (wl + 31) // 32
        q = np.percentile(wl, [50, 90, 99, 99.9, 100])
        print(f"view {view}: items {wl.size}  walk p50/p90/p99/p99.9/max = {q}  total steps {steps.sum()}  "
              f"max steps {steps.max()}  top-10 share {np.sort(steps)[-10:].sum() / steps.sum():.4f}")
        del r, out


if __name__ == "__main__":
    main()
