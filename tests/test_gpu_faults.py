"""Failure detection and fault injection, through the C ABI.

* bgs_frame_validate proves a frame's tile lists (every tile's list = the visible Gaussians
  whose rect covers it, strictly increasing in (depth bits, index); ranges consecutive over
  [0, K); K = sum tiles_touched) on every sort path -- and reports each injected fault:
  two swapped list entries, a foreign Gaussian in a list, a shifted range boundary.
* The parity check itself is sensitive: swapping two record fields (the conic's A and C)
  or two list entries makes the image disagree with the oracle well beyond IMG_TOL.
* bgs_nonfinite counts NaN / Inf in a gradient and names the first index.
* A checkpoint written mid-run and resumed gives the uninterrupted run's parameters.
"""
import numpy as np
import pytest

import gen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4


@pytest.fixture(scope="module")
def bgs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_14564_b200 as m

    return m


class _DevPtr:
    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def dev_tensor(ptr, count, typestr):
    """Writable zero-copy view of a workspace region."""
    return torch.as_tensor(_DevPtr(ptr, count, typestr), device="cuda")


def render(bgs, s, cam, flags=0):
    theta = torch.from_numpy(s.theta).cuda()
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 21, device=torch.device("cuda"), debug_flags=flags)
    out = r.forward(theta, cam, s.sh_degree)
    torch.cuda.synchronize()
    return r, theta, out


def clean(rep):
    return rep["range_errors"] == 0 and rep["member_errors"] == 0 and rep["order_errors"] == 0 and \
        rep["count_error"] == 0


def lists(r):
    v = r.views()
    nt = v.tiles_x * v.tiles_y
    vals = dev_tensor(v.values_sorted, r.num_keys, "<i4")
    ranges = dev_tensor(v.ranges, 2 * nt, "<i4").view(nt, 2)
    depth = dev_tensor(v.depth, r.n, "<f4")
    return vals, ranges, depth


def scene():
    return gen.small_scene(21, 4000, 160, 112, scale_mu=0.05)


@pytest.mark.parametrize("path", ["direct", "onesweep64", "radix_split", "rowsplit", "square_rect"])
def test_validate_clean_on_every_sort_path(bgs, path):
    flags = {"direct": 0, "onesweep64": bgs.BGS_DEBUG_SORT_ONESWEEP64, "radix_split": bgs.BGS_DEBUG_SORT_RADIX_SPLIT,
             "rowsplit": bgs.BGS_DEBUG_SORT_ROWSPLIT, "square_rect": bgs.BGS_DEBUG_SQUARE_RECT}[path]
    for s in (scene(), gen.tiny()):
        r, _, _ = render(bgs, s, s.cameras[0], flags)
        rep = bgs.validate(r.frame)
        assert clean(rep), rep
        assert rep["tiles_touched"] == r.num_keys > 0


def test_validate_clean_at_garden_scale(bgs):
    s = gen.garden()
    cam = s.cameras[3]
    theta = torch.from_numpy(s.theta).cuda()
    r = bgs.Renderer(s.n, cam.width, cam.height, max_keys=1 << 26, device=torch.device("cuda"))
    r.forward(theta, cam, s.sh_degree)
    rep = bgs.validate(r.frame)
    assert clean(rep), rep
    assert rep["tiles_touched"] == r.num_keys > 10_000_000


def longest_tile(ranges):
    rg = ranges.cpu().numpy().astype(np.int64)
    t = int(np.argmax(rg[:, 1] - rg[:, 0]))
    return t, int(rg[t, 0]), int(rg[t, 1])


def test_swapped_entries_are_reported_and_break_parity(bgs):
    s = scene()
    cam = s.cameras[0]
    r, theta, out = render(bgs, s, cam)
    vals, ranges, depth = lists(r)
    t, a, b = longest_tile(ranges)
    assert b - a >= 8
    # swap the first two entries of different depth
    v = vals[a:b].cpu().numpy()
    d = depth.cpu().numpy()[v]
    j = int(np.nonzero(d[1:] != d[:-1])[0][0])
    x, y = vals[a + j].item(), vals[a + j + 1].item()
    vals[a + j], vals[a + j + 1] = y, x
    rep = bgs.validate(r.frame)
    assert rep["order_errors"] >= 1 and rep["member_errors"] == 0 and rep["range_errors"] == 0
    # the forward over the corrupted lists no longer matches the oracle: swap the whole list
    # order of the longest tile (front-to-back becomes back-to-front) for a visible effect
    vals[a:b] = torch.flip(vals[a:b].clone(), [0])
    bgs.bgs_render_fwd(r.frame, out["image"], out["final_T"], out["n_contrib"])
    torch.cuda.synchronize()
    ref = oracle.forward(s.theta, s.n, s.sh_degree, cam)
    assert np.abs(out["image"].cpu().numpy() - ref["image"]).max() > 100 * IMG_TOL


def test_foreign_entry_is_reported(bgs):
    s = scene()
    r, _, _ = render(bgs, s, s.cameras[0])
    vals, ranges, _ = lists(r)
    v = r.views()
    radius = dev_tensor(v.radius, s.n, "<i4").cpu().numpy()
    t, a, b = longest_tile(ranges)
    members = set(vals[a:b].cpu().numpy().tolist())
    culled = np.nonzero(radius == 0)[0]
    foreign = int(culled[0]) if len(culled) else next(i for i in range(s.n) if i not in members)
    vals[a] = foreign
    rep = bgs.validate(r.frame)
    assert rep["member_errors"] >= 1


def test_shifted_range_is_reported(bgs):
    s = scene()
    r, _, _ = render(bgs, s, s.cameras[0])
    _, ranges, _ = lists(r)
    t, a, b = longest_tile(ranges)
    ranges[t, 1] = b - 1  # the tile now ends one entry early: a gap before the next tile
    rep = bgs.validate(r.frame)
    assert rep["range_errors"] >= 1


def test_swapped_record_fields_break_parity(bgs):
    """Conic A <-> C swapped in every visible record: the parity harness must notice."""
    s = scene()
    cam = s.cameras[0]
    r, _, out = render(bgs, s, cam)
    v = r.views()
    rec = dev_tensor(v.record, 12 * s.n, "<f4").view(s.n, 12)
    rec[:, [4, 6]] = rec[:, [6, 4]].clone()
    bgs.bgs_render_fwd(r.frame, out["image"], out["final_T"], out["n_contrib"])
    torch.cuda.synchronize()
    ref = oracle.forward(s.theta, s.n, s.sh_degree, cam)
    assert np.abs(out["image"].cpu().numpy() - ref["image"]).max() > 100 * IMG_TOL
    assert clean(bgs.validate(r.frame))  # the lists themselves are still right


def test_nonfinite_counts_and_locates(bgs):
    g = torch.randn(59 * 1001 + 3, device="cuda")  # a ragged tail past the float4 body
    assert bgs.nonfinite(g) == (0, -1)
    g[4097] = float("nan")
    g[59 * 1001 + 2] = float("inf")
    g[123456 % g.numel()] = float("-inf")
    c, first = bgs.nonfinite(g)
    assert c == 3 and first == min(4097, 123456 % g.numel())
    assert bgs.nonfinite(g[:0].clone()) == (0, -1)


def test_nonfinite_gradient_from_a_poisoned_loss(bgs):
    """A NaN in dL/dimage (a broken loss) reaches the gradient through the real backward;
    the check finds it before Adam would spread it into theta."""
    s = scene()
    cam = s.cameras[0]
    r, theta, out = render(bgs, s, cam)
    grad = torch.zeros_like(theta)
    dl = torch.full((3, cam.height, cam.width), 1e-3, device="cuda")
    r.backward(theta, s.sh_degree, dl, out, grad)
    torch.cuda.synchronize()
    assert bgs.nonfinite(grad) == (0, -1)
    nc = out["n_contrib"].cpu().numpy().view(np.uint32)
    y, x = np.unravel_index(int(np.argmax(nc)), nc.shape)  # a pixel many Gaussians blend into
    dl[1, y, x] = float("nan")
    grad.zero_()
    out = r.forward(theta, cam, s.sh_degree)
    r.backward(theta, s.sh_degree, dl, out, grad)
    torch.cuda.synchronize()
    c, first = bgs.nonfinite(grad)
    assert c > 0 and 0 <= first < grad.numel()
    assert not torch.isfinite(grad[first])


def test_checkpoint_resume_matches_uninterrupted_run(bgs, tmp_path):
    from paper_2510_14564_b200 import checkpoint

    s = gen.small_scene(22, 3000, 128, 96)
    dev = torch.device("cuda")
    hp = bgs.AdamHParams()

    def train(theta, m, v, steps, start):
        r = bgs.Renderer(s.n, s.cameras[0].width, s.cameras[0].height, max_keys=1 << 21, device=dev)
        for k in range(start, start + steps):
            cam = s.cameras[k % len(s.cameras)]
            grad = torch.zeros_like(theta)
            out = r.forward(theta, cam, s.sh_degree)
            dl = torch.from_numpy(gen.random_dl_dimage(100 + k, cam.width, cam.height)).to(dev)
            r.backward(theta, s.sh_degree, dl, out, grad)
            bgs.adam_step(theta, grad, m, v, s.n, hp, step=k + 1)
        torch.cuda.synchronize()

    th_a = torch.from_numpy(s.theta).to(dev)
    m_a, v_a = torch.zeros_like(th_a), torch.zeros_like(th_a)
    train(th_a, m_a, v_a, 4, 0)
    th_b = torch.from_numpy(s.theta).to(dev)
    m_b, v_b = torch.zeros_like(th_b), torch.zeros_like(th_b)
    train(th_b, m_b, v_b, 2, 0)
    path = str(tmp_path / "ck.pt")
    checkpoint.save(path, th_b, m_b, v_b, step=2, n=s.n, sh_degree=s.sh_degree)
    del th_b, m_b, v_b
    st = checkpoint.load(path, device=dev)
    assert st["step"] == 2
    th_c, m_c, v_c = st["theta"], st["exp_avg"], st["exp_avg_sq"]
    train(th_c, m_c, v_c, 2, st["step"])
    # the backward's RED atomics sum in hardware order: equal to float rounding
    assert torch.allclose(th_c, th_a, rtol=1e-5, atol=1e-6)
    for got, want in ((m_c, m_a), (v_c, v_a)):  # per-element sums of atomics: compare in norm
        assert float(torch.linalg.vector_norm(got - want) / torch.linalg.vector_norm(want)) <= 1e-5
