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
