#!/bin/bash
# FP32/ALU/MUFU pipe counts of the blend kernels for one hinted garden training step
# (lane ops per evaluation); runs on the GPU box.
OUT=gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,sm__thread_inst_executed_pipe_fma_pred_on.sum,sm__thread_inst_executed_pipe_alu_pred_on.sum,lts__t_sectors_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:"k_render_fwd|k_render_bwd" -s 2 -c 2 --csv \
    python tools/stage_probe.py --step 2 > $OUT/pipe_probe.csv 2>/dev/null
python - <<'PY'
import csv, io, re
rows = list(csv.reader(io.StringIO(open("gpurun_out/pipe_probe.csv").read()[open("gpurun_out/pipe_probe.csv").read().index('"ID"'):])))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}
out = {}
for r in rows[1:]:
    k = re.sub(r"\(.*", "", r[col["Kernel Name"]]).split("::")[-1]
    out.setdefault(k, {})[r[col["Metric Name"]]] = (r[col["Metric Unit"]], r[col["Metric Value"]])
lines = ["| kernel | metric | unit | value |", "|---|---|---|---|"]
for k, ms in out.items():
    for m, (u, v) in ms.items():
        lines.append(f"| {k} | {m} | {u} | {v} |")
open("gpurun_out/pipe_probe.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
PY
