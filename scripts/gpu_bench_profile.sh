# ncu launch list + one ncu --set full capture of the step kernels (1 GPU), tag $1.
# Each ncu command runs only after the same command has exited 0 without ncu.
mkdir -p gpurun_out
TAG=${1:-r2}
CMD="python bench.py --steps 8 --warmup 3 --no-e2e --no-extras --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_quantize|k_apply|k_absmax|k_encode|k_round_wait|k_signal" --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_list_$TAG.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_quantize" -s 6 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
CMD0="python bench.py --steps 8 --warmup 3 --no-e2e --no-extras --no-cpu-baseline --scale-block 0"
$CMD0 > gpurun_out/plainb0_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_absmax|k_encode" -s 6 -c 2 -o gpurun_out/prof_b0_$TAG $CMD0 > gpurun_out/ncu_b0_$TAG.log 2>&1; echo "ncu b0 rc=$?"
python scripts/emulated_apply.py > gpurun_out/emu_$TAG.log 2>&1 && \
ncu --set full --clock-control none --nvtx --nvtx-include "capture/" -k regex:"k_apply" -o gpurun_out/prof_emu_$TAG python scripts/emulated_apply.py > gpurun_out/ncu_emu_$TAG.log 2>&1; echo "ncu emu rc=$?"
ls -la gpurun_out/*$TAG*
