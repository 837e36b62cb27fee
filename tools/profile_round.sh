#!/bin/bash
# Runs ON the GPU box (gpurun): the per-round ncu evidence, reduced to small files in
# gpurun_out/ (full .ncu-rep reports stay in /tmp: gpurun copies back <= 64 MiB).
#   bash tools/profile_round.sh TAG
# 1. launch list of one timed bench step (NVTX range "bench_timed"): shares per kernel
# 2. ncu --set full of two one-view training steps (tools/stage_probe.py): per-kernel
#    summary, DRAM traffic per stage, source pages of the blend kernels
TAG=${1:-r}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx --nvtx-include "bench_timed/" --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/launches_$TAG.log 2>&1
python tools/launch_shares.py $OUT/launches_$TAG.csv $OUT/launch_shares_$TAG.md \
    --title "Launch list $TAG: one bench step (16 garden views + batched chain rule + Adam)" \
    --note "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none over the NVTX range of one timed bench step. Cold-cache, serialised launches: compare SHARES, not absolutes." \
    > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -f -o /tmp/prof_$TAG \
    python tools/stage_probe.py --step 2 > $OUT/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_$TAG.ncu-rep $OUT/ncu_summary_$TAG.md --title "$TAG, one garden view (camera 0) training step" \
    --traffic $OUT/ncu_traffic_$TAG.json --stage 'render_fwd=^k_render_fwd' \
    --stage 'blend_bwd=^k_render_bwd<' --stage 'adam=^k_adam$' >> $OUT/ncu_full_$TAG.log 2>&1
# the batched preprocess over 16 views, as the bench runs it (one launch)
ncu --set full --clock-control none --import-source on -f -o /tmp/prof_pre_$TAG -k regex:k_preprocess_views -s 1 -c 1 \
    python tools/stage_probe.py --step 2 --views 16 >> $OUT/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_pre_$TAG.ncu-rep $OUT/ncu_summary_pre_$TAG.md --title "$TAG, batched a2 over 16 garden views" \
    --traffic $OUT/ncu_traffic_$TAG.json --stage 'preprocess=^k_preprocess_views$' >> $OUT/ncu_full_$TAG.log 2>&1
ncu -i /tmp/prof_pre_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_k_preprocess_views_$TAG.csv 2>&1
# the batched chain rule over 16 views, as the bench runs it (one launch)
ncu --set full --clock-control none --import-source on -f -o /tmp/prof_pb_$TAG -k regex:k_preprocess_bwd -s 1 -c 1 \
    python tools/stage_probe.py --step 2 --views 16 >> $OUT/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_pb_$TAG.ncu-rep $OUT/ncu_summary_pb_$TAG.md --title "$TAG, batched a10 over 16 garden views" \
    --traffic $OUT/ncu_traffic_$TAG.json --stage 'preprocess_bwd=^k_preprocess_bwd$' >> $OUT/ncu_full_$TAG.log 2>&1
ncu -i /tmp/prof_pb_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_k_preprocess_bwd_$TAG.csv 2>&1
# the blend kernels' hardware lane-ops and shared-memory wavefronts (bench.py's hw fractions)
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__thread_inst_executed_pipe_fma_pred_on.sum,sm__thread_inst_executed_pipe_alu_pred_on.sum,sm__sass_thread_inst_executed_ops_fadd2_fmul2_ffma2_pred_on.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum \
    --clock-control none -k regex:"k_render_fwd|render_bwd" -c 5 --csv python tools/stage_probe.py --step 2 > $OUT/ncu_hw_$TAG.csv 2>> $OUT/ncu_full_$TAG.log
python tools/ncu_hw.py $OUT/ncu_hw_$TAG.csv $OUT/ncu_hw_$TAG.json $TAG >> $OUT/ncu_full_$TAG.log 2>&1
for k in k_render_fwd k_render_bwd k_emit_direct; do
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k regex:$k -s 1 -c 1 \
      > $OUT/src_${k}_$TAG.csv 2>&1
done
ls -la $OUT
