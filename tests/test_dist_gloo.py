"""World-size-2 gloo test of the data-parallel host logic (paper_2510_14564_b200.dp) on CPU.

Each rank plays a GPU: it renders its share of a 4-view batch with the oracle as its
"renderer" (forward + backward, grad += over its views), the ranks all-reduce grad with
gloo, and both apply the oracle's Adam.  Checks: the all-reduced
gradient equals the single-process sum over all 4 views, and the two replicas are
bit-identical after the step.  The dp module imports no oracle code; the test supplies it.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle

WORLD = 2
N_VIEWS = 4
LR6 = [1.6e-4, 5e-3, 1e-3, 0.05, 2.5e-3, 1.25e-4]


def _scene():
    s = gen.small_scene(21, 300, 48, 40, scale_mu=0.08)
    base = s.cameras[0]
    cams = []
    for k in range(N_VIEWS):  # the same camera shifted sideways per view
        c = gen.make_camera(np.eye(3), [0.05 * k, -0.03 * k, 0.0], base.width, base.height,
                            base.width / (2 * base.tan_fovx), base.height / (2 * base.tan_fovy), bg=base.bg)
        cams.append(c)
    return s, cams


def _view_grad(s, cam, seed):
    f = oracle.forward(s.theta, s.n, s.sh_degree, cam)
    dl = gen.random_dl_dimage(seed, cam.width, cam.height, scale=1.0 / N_VIEWS)
    return oracle.backward(s.theta, s.n, s.sh_degree, cam, f, dl)["grad"]


def _worker_sharded(rank, port, out):
    """reduce-scatter -> Adam on the rank's shard -> all-gather."""
    from paper_2510_14564_b200_dp import dp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    s, cams = _scene()
    total = 59 * s.n
    shard, padded = dp.shard_layout(total, WORLD)
    grad = torch.zeros(padded, dtype=torch.float64)
    for v in dp.views_for_rank(list(range(N_VIEWS)), rank, WORLD):
        grad[:total] += torch.from_numpy(_view_grad(s, cams[v], 100 + v))
    g_shard = dp.reduce_scatter_grads(grad, rank, WORLD)
    b, e = dp.shard_range(rank, WORLD, total)
    assert g_shard.data_ptr() == grad[b:].data_ptr() and g_shard.numel() == shard
    # Adam is elementwise: the oracle's full-layout update, read on this shard only (the
    # rest of `grad` still holds this rank's partial sums and must not leak into theta)
    g_full = np.zeros(total)
    lo, hi = b, min(e, total)
    g_full[lo:hi] = grad[lo:hi].numpy()
    th_all, _, _ = oracle.adam(s.theta, g_full, np.zeros(total), np.zeros(total), s.n, LR6, step=1)
    theta = torch.zeros(padded, dtype=torch.float64)
    theta[:total] = torch.from_numpy(s.theta.astype(np.float64))
    theta[lo:hi] = torch.from_numpy(th_all[lo:hi])
    dp.all_gather_params(theta, rank, WORLD)
    out[rank] = (g_shard.numpy()[: hi - lo].copy(), theta.numpy().copy(), (lo, hi))
    dist.destroy_process_group()


def _worker(rank, port, out):
    from paper_2510_14564_b200_dp import dp  # loaded without the CUDA library (see below)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    s, cams = _scene()
    mine = dp.views_for_rank(list(range(N_VIEWS)), rank, WORLD)
    grad = torch.zeros(59 * s.n, dtype=torch.float64)
    for v in mine:
        grad += torch.from_numpy(_view_grad(s, cams[v], 100 + v))
    dp.allreduce_grads(grad, WORLD)
    th, _, _ = oracle.adam(s.theta, grad.numpy(), np.zeros(59 * s.n), np.zeros(59 * s.n), s.n, LR6, step=1)
    out[rank] = (mine, grad.numpy().copy(), th)
    dist.destroy_process_group()


def _load_dp_module():
    """Import paper_2510_14564_b200/dp.py directly: the package __init__ loads libbgs.so
    (and must fail loudly without it), but the dp helpers are pure host logic."""
    import importlib.util
    import sys
    import types

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = types.ModuleType("paper_2510_14564_b200_dp")
    spec = importlib.util.spec_from_file_location("paper_2510_14564_b200_dp.dp",
                                                  os.path.join(root, "paper_2510_14564_b200", "dp.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    pkg.dp = mod
    sys.modules["paper_2510_14564_b200_dp"] = pkg
    return mod


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _run_rank(rank, port, q):
    _load_dp_module()
    res = {}
    _worker(rank, port, res)
    mine, grad, th = res[rank]
    q.put((rank, mine, grad, th))


def _run_rank_sharded(rank, port, q):
    _load_dp_module()
    res = {}
    _worker_sharded(rank, port, res)
    q.put((rank, *res[rank]))


def test_shard_layout():
    dp = _load_dp_module()
    for total in (0, 1, 59, 59 * 3001, 59 * 5_800_000):
        for world in (1, 2, 3, 4, 8):
            shard, padded = dp.shard_layout(total, world)
            assert shard % 4 == 0 and padded == shard * world and padded >= total
            assert padded - total < world * 4 + world  # at most one alignment unit + rounding per rank
            rs = [dp.shard_range(r, world, total) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == padded
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_two_rank_sharded_update_matches_allreduce_path():
    """Sharded update == all-reduce + full Adam: gradient shards equal the single-process
    4-view sum, and both replicas end bit-identical to the full update."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank_sharded, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        rank, g_shard, theta, rng = q.get(timeout=300)
        res[rank] = (g_shard, theta, rng)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s, cams = _scene()
    ref = sum(_view_grad(s, cams[v], 100 + v) for v in range(N_VIEWS))
    th_ref, _, _ = oracle.adam(s.theta, ref, np.zeros(59 * s.n), np.zeros(59 * s.n), s.n, LR6, step=1)
    for r in range(WORLD):
        g_shard, theta, (lo, hi) = res[r]
        np.testing.assert_allclose(g_shard, ref[lo:hi], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    assert np.array_equal(res[0][1], res[1][1])  # replicas bit-identical
    np.testing.assert_allclose(res[0][1][: 59 * s.n], th_ref, rtol=1e-12, atol=1e-15)


def test_view_split_round_robin():
    dp = _load_dp_module()
    views = list(range(16))
    for world in (1, 2, 4, 8):
        parts = [dp.views_for_rank(views, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == views
        assert all(len(p) == 16 // world for p in parts)
    with pytest.raises(ValueError):
        dp.views_for_rank(views, 2, 2)


def test_two_rank_allreduce_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(WORLD):
        rank, mine, grad, th = q.get(timeout=300)
        results[rank] = (mine, grad, th)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0][0] == [0, 2] and results[1][0] == [1, 3]
    s, cams = _scene()
    ref = sum(_view_grad(s, cams[v], 100 + v) for v in range(N_VIEWS))
    for r in range(WORLD):
        g = results[r][1]
        assert np.linalg.norm(g - ref) <= 1e-12 * max(np.linalg.norm(ref), 1.0)
    assert np.array_equal(results[0][2], results[1][2])  # replicas bit-identical after Adam


def test_gaussian_chunks_cover_theta_once():
    """§8(e) 1: the chunks' segment sub-ranges tile theta[59n] exactly once."""
    dp = _load_dp_module()
    for n in (1, 7, 300, 5_800_000):
        for chunks in (1, 3, 4, 16):
            cover = np.zeros(59 * n, np.int8) if n < 10_000 else None
            total = 0
            for b, e in dp.gaussian_chunks(n, chunks):
                for lo, hi in dp.segment_slices(n, b, e):
                    assert 0 <= lo <= hi <= 59 * n
                    total += hi - lo
                    if cover is not None:
                        cover[lo:hi] += 1
            assert total == 59 * n
            if cover is not None:
                assert (cover == 1).all()


def _worker_chunked(rank, port, q):
    _load_dp_module()
    from paper_2510_14564_b200_dp import dp

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    s, cams = _scene()
    grad = torch.zeros(59 * s.n, dtype=torch.float64)
    for v in dp.views_for_rank(list(range(N_VIEWS)), rank, WORLD):
        grad += torch.from_numpy(_view_grad(s, cams[v], 100 + v))
    works = []
    for b, e in dp.gaussian_chunks(s.n, 4):  # as the chain rule finishes each chunk
        works += dp.allreduce_chunk(grad, s.n, b, e, WORLD, async_op=True)
    for w in works:
        w.wait()
    q.put((rank, grad.numpy().copy()))
    dist.destroy_process_group()


def test_two_rank_chunked_allreduce_matches_single_process():
    """The overlapped exchange (five async all-reduces per Gaussian chunk) sums the same
    gradient as one all-reduce of grad[59n]: both ranks hold the 4-view sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_chunked, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s, cams = _scene()
    ref = sum(_view_grad(s, cams[v], 100 + v) for v in range(N_VIEWS))
    for r in range(WORLD):
        assert np.linalg.norm(res[r] - ref) <= 1e-12 * max(np.linalg.norm(ref), 1.0)
    assert np.array_equal(res[0], res[1])
