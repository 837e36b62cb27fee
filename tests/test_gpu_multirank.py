"""The G > 1 bench path on one GPU: two ranks over gloo pinned to cuda:0
(BGS_FORCE_DEVICE), so the view split, the reduce-scatter / all-reduce / chunked-overlap
exchange and the sharded Adam run on the real kernels.  A functional check only: gloo
stages the collectives through the host, so the timings say nothing (the ranks' kernels
never wait on one another)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("update", ["sharded", "allreduce", "overlap"])
def test_two_rank_bench_runs(update):
    env = dict(os.environ, BGS_FORCE_DEVICE="0", BGS_DIST_BACKEND="gloo")
    port = {"sharded": 29611, "allreduce": 29612, "overlap": 29613}[update]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--config", "tiny", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
           "--no-variants", "--update", update]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["steps"] == 2
    assert line["config"]["parallelism"].endswith("2")
