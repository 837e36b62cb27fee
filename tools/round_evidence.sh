T=$1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for c in tandt_train db_playroom tiny; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_reference.json 2>> gpurun_out/${T}_bench.err
timeout 1500 bash tools/profile_round.sh $T > gpurun_out/${T}_profile.log 2>&1
ls -la gpurun_out | tail -30
