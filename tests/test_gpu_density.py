"""NEXT-1 GPU parity: the T1 local densities (§III-C1) are exact integers, so the
grid kernel must equal the oracle's O(n^2) definition bit for bit; the thresholds follow."""
import numpy as np
import pytest

import gen
import oracle

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


def _fixtures():
    r = np.random.default_rng(3)
    contrast = np.concatenate([r.uniform(-0.1, 0.1, (1000, 3)), r.uniform(-1, 1, (1000, 3)) + [3.0, 0, 0]])
    s = gen.garden(seed=2, n=30000, n_cams=1)
    garden_means = gen.segments(s.theta, s.n)["means"]
    lattice = np.stack(np.meshgrid(*[np.arange(12) * 0.1] * 3), -1).reshape(-1, 3)  # exact ties at r
    return {"contrast": (contrast, 0.1), "garden30k": (garden_means, 0.05), "lattice": (lattice, 0.1),
            "single": (np.zeros((1, 3)), 1.0), "far": (r.uniform(-1e3, 1e3, (500, 3)), 3.0)}


@pytest.mark.parametrize("name", list(_fixtures()))
def test_local_density_exact(bgs, name):
    pts, rad = _fixtures()[name]
    pts = np.ascontiguousarray(pts, np.float32)
    ref = oracle.local_density(pts, rad)
    counts, stats = bgs.bgs_local_density(torch.from_numpy(pts).cuda(), rad)
    torch.cuda.synchronize()
    got = counts.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, ref)
    s = oracle.density_thresholds(ref)
    st = stats.cpu().numpy()
    np.testing.assert_allclose(st, [s["mu"], s["sigma"], s["rho_low"], s["rho_high"]], rtol=1e-12, atol=1e-12)


def test_density_on_theta_means_segment(bgs):
    # the kernel reads theta's means segment in place
    s = gen.small_scene(4, 3000, 64, 64)
    theta = torch.from_numpy(s.theta).cuda()
    counts, _ = bgs.bgs_local_density(theta[: 3 * s.n], 0.05)
    ref = oracle.local_density(gen.segments(s.theta, s.n)["means"], 0.05)
    assert np.array_equal(counts.cpu().numpy().view(np.uint32), ref)
