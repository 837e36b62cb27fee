"""compute-sanitizer over every libbgs kernel (race detection / failure
detection): memcheck (out-of-bounds and misaligned accesses), racecheck (shared-memory
hazards), synccheck (barrier misuse) on tools/sanitize_run.py -- the tiny config and a 20k
garden sample, including the look-back scans, the ticket-ordered persistent blend grids, the
forward's speculative split walks and merges, the backward's checkpoint segments, the
density rounds and the importance sampling."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("which", ["tiny", "garden20k"])
def test_compute_sanitizer_clean(tool, which):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_run.py"), which]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if "sanitize workload done" not in out and "compute-sanitizer is closed" in out:
        # the GPU pool replaced compute-sanitizer by a refusal (runs under it left GPUs needing a
        # reset); the last clean runs are profiles/r2_sanitizer.log
        pytest.skip("compute-sanitizer refused on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert "sanitize workload done" in out, out[-4000:]
    clean = ("ERROR SUMMARY: 0 errors" in out if tool != "racecheck"
             else "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out)
    assert r.returncode == 0 and clean, out[-4000:]
