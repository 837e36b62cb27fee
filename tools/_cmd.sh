timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -rs --durations=10 2>&1 | tail -15 > gpurun_out/r2v_sanitizer.log; tail -15 gpurun_out/r2v_sanitizer.log
