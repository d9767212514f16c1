mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/bench_r1_a.json 2> gpurun_out/bench_r1_a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r1_a.json
tail -5 gpurun_out/bench_r1_a.err
CMD="python bench.py --steps 6 --warmup 2 --no-e2e --no-m-sweep --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_quantize|k_apply|k_absmax|k_encode" --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_quantize" -s 4 -c 2 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu2.log
