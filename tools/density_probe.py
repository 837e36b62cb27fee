"""Times the NEXT-1 density-control step on the garden scene, kernel by kernel (events
around plan, result, apply); not the bench."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.spatial import cKDTree  # noqa: E402

import gen  # noqa: E402
import paper_2510_14564_b200 as bgs  # noqa: E402


def main():
    s = gen.make("garden")
    n = s.n
    mu = gen.segments(s.theta, n)["means"]
    sub = mu[gen.rng(77).choice(n, 100_000, replace=False)].astype(np.float64)
    r = float(np.median(cKDTree(sub).query(sub, k=9)[0][:, 8]) * (1e5 / n) ** (1 / 3))
    dev = torch.device("cuda")
    th = torch.from_numpy(s.theta).to(dev)
    m = torch.zeros_like(th)
    prm = bgs.DensityParams(r)
    g = torch.Generator(device=dev)
    for it in range(3):
        g.manual_seed(it)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = bgs.density_control(th, m, m, n, prm, g)
        torch.cuda.synchronize()
        rep = out[4]
        print(f"r {r:.5f}: {1e3 * (time.perf_counter() - t0):.1f} ms  n {n} -> {out[3]}  pairs {rep.n_pairs} "
              f"children {rep.n_children} rho mu {rep.mu_rho:.2f} sd {rep.sigma_rho:.2f} d_merge {rep.d_merge:.5f} "
              f"short {out[5]}", flush=True)


if __name__ == "__main__":
    main()
