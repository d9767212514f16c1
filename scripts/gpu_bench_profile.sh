# bench + ncu launch list + one ncu --set full capture of the step kernels (1 GPU).
mkdir -p gpurun_out
TAG=${1:-r1}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
CMD="python bench.py --steps 8 --warmup 3 --no-e2e --no-m-sweep --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_quantize|k_apply|k_absmax|k_encode" --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo "ncu list rc=$?"
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_quantize" -s 6 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
python scripts/emulated_apply.py > gpurun_out/emu_$TAG.log 2>&1 && \
ncu --set full --clock-control none --nvtx --nvtx-include "capture/" -k regex:"k_apply" -o gpurun_out/prof_emu_$TAG python scripts/emulated_apply.py > gpurun_out/ncu_emu_$TAG.log 2>&1; echo "ncu emu rc=$?"
