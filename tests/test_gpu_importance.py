"""NEXT-3 / NEXT-4 GPU parity (§IV-C1/C3): per-tile colour buckets (integer parts
bit-exact), importance scores, the keep rule, and rendering with a keep mask, all against
oracle/importance.py and the C++ oracle on the same inputs."""
import numpy as np
import pytest

import gen
import oracle
from oracle import importance as I

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


def _render(bgs, s, cam):
    dev = torch.device("cuda")
    theta = torch.from_numpy(s.theta).to(dev)
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 21, device=dev)
    out = r.forward(theta, cam, s.sh_degree)
    torch.cuda.synchronize()
    return r, theta, out


@pytest.mark.parametrize("seed,n,w,h", [(0, 2000, 64, 48), (1, 5000, 83, 57)])
def test_tile_buckets_parity(bgs, seed, n, w, h):
    s = gen.small_scene(seed, n, w, h)
    cam = s.cameras[0]
    r, _, out = _render(bgs, s, cam)
    nb, keys, counts, csum, osum = bgs.bgs_tile_buckets(out["image"], out["final_T"], w, h)
    torch.cuda.synchronize()
    img, fT = out["image"].cpu().numpy(), out["final_T"].cpu().numpy()
    ref = I.tile_buckets(img, fT)
    nb, keys = nb.cpu().numpy(), keys.cpu().numpy().view(np.uint16)
    counts, csum, osum = counts.cpu().numpy(), csum.cpu().numpy().reshape(-1, 3), osum.cpu().numpy()
    got = {}
    for t in range(len(nb)):
        ks = keys[t * 256:t * 256 + nb[t]]
        assert (np.diff(ks.astype(int)) > 0).all()  # ascending key order
        for j in range(nb[t]):
            got[(t, int(ks[j]))] = (int(counts[t * 256 + j]), csum[t * 256 + j], float(osum[t * 256 + j]))
    assert set(got) == set(ref)
    for k, (c, cs, o) in ref.items():
        assert got[k][0] == c
        np.testing.assert_allclose(got[k][1], cs, rtol=1e-5, atol=1e-5)
        assert abs(got[k][2] - o) <= 1e-5 * max(1.0, abs(o))


@pytest.mark.parametrize("seed,n,w,h", [(2, 1500, 64, 48), (3, 4000, 96, 72)])
def test_importance_and_keep_parity(bgs, seed, n, w, h):
    s = gen.small_scene(seed, n, w, h)
    cam = s.cameras[0]
    r, theta, out = _render(bgs, s, cam)
    imp, cnt = bgs.bgs_importance(r.frame, out["image"], s.n)
    torch.cuda.synchronize()
    pre = oracle.forward(s.theta, s.n, s.sh_degree, cam)["pre"]
    ref_imp, ref_cnt = I.importance(pre, out["image"].cpu().numpy(), w, h)
    imp, cnt = imp.cpu().numpy().astype(np.float64), cnt.cpu().numpy()
    # alpha >= 1/255 decisions agree except within float rounding of the threshold
    assert (cnt != ref_cnt).mean() <= 0.01
    same = cnt == ref_cnt
    np.testing.assert_allclose(imp[same], ref_imp[same], rtol=2e-4, atol=1e-6)
    assert (pre["radius"] > 0).sum() > 0.5 * s.n and (ref_cnt > 0).any()
    # the keep rule on the GPU's own scores (exact: a stable sort of float bits)
    for frac, inv in ((0.5, False), (0.3, True), (1.0, False), (0.0, False)):
        keep = bgs.bgs_importance_keep(torch.from_numpy(imp.astype(np.float32)).cuda(), frac, inv)
        # the ABI takes the fraction as a float: ceil(float(0.3) * n) can exceed ceil(0.3 n)
        ref_keep = I.keep_mask(imp.astype(np.float32), float(np.float32(frac)), inv)
        assert np.array_equal(keep.cpu().numpy().astype(bool), ref_keep)


def test_render_with_keep_mask_equals_rendering_the_kept_subset(bgs):
    s = gen.small_scene(4, 3000, 80, 56)
    cam = s.cameras[0]
    r, theta, out = _render(bgs, s, cam)
    imp, _ = bgs.bgs_importance(r.frame, out["image"], s.n)
    keep = bgs.bgs_importance_keep(imp, 0.6)
    bgs.bgs_frame_set_keep(r.frame, keep)
    out2 = r.forward(theta, cam, s.sh_degree)
    torch.cuda.synchronize()
    k = keep.cpu().numpy().astype(bool)
    seg = gen.segments(s.theta, s.n)
    sub = gen.pack(seg["means"][k], seg["log_scales"][k], seg["quats"][k], seg["opacity_logits"][k], seg["sh"][k])
    ref = oracle.forward(sub, int(k.sum()), s.sh_degree, cam)
    ok = ref["flags"] == 0
    assert np.abs(out2["image"].cpu().numpy() - ref["image"])[:, ok].max() <= 1e-4
    assert np.array_equal(out2["n_contrib"].cpu().numpy()[ok], ref["n_contrib"][ok])
    bgs.bgs_frame_set_keep(r.frame, None)  # back to all Gaussians
    out3 = r.forward(theta, cam, s.sh_degree)
    torch.cuda.synchronize()
    assert torch.equal(out3["image"], out["image"])
