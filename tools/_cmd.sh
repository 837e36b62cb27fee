timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 300 python tools/stage_probe.py --only render_fwd,blend_bwd --reps 20 2>&1 | grep -v "^{"
