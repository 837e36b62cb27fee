timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sort" 2>&1 | tail -2
timeout 300 python tools/stage_probe.py --only sort --reps 20 2>&1 | grep sort
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_rs|k_scan|k_tile" -c 14 --csv python tools/stage_probe.py --only sort --reps 1 > gpurun_out/r2j_ncu.csv 2>&1
