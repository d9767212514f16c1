# k_apply: first group's loads before the round check ("early", current) vs after it ("late", the
# previous kernel, scripts/libsd_late.so), alternating on one box; N = ${N:-1}; parity tests on "early" first
mkdir -p gpurun_out
N=${N:-1}
if [ "$N" = 1 ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rounds or nonfinite or full_size_sampled or offload or cuda_graph or many_rounds or no_writes or adamw_merge" 2>&1 | tail -1
fi
run() {
  cp scripts/libsd_$1.so paper_2501_18512_b200/libsd.so
  if [ "$N" = 1 ]; then
    timeout 600 python bench.py --steps 256 --warmup 8 --no-e2e --no-cpu-baseline --no-extras $EXTRA > gpurun_out/ab_early_$1_$2.json 2>/dev/null
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --no-e2e --no-overlap $EXTRA > gpurun_out/ab_early_$1_$2.json 2>/dev/null
  fi
  python -c "
import json; j=json.loads(open('gpurun_out/ab_early_$1_$2.json').read().strip().splitlines()[-1])
print('$1 $2', 'value %.4e per_gpu %.4e ms %.4f apply %.4f quant %.4f' % (j['value'], j['value']/j['n_gpus'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac']))"
}
for rep in 1 2; do
  for lib in early late; do
    if [ "$N" = 1 ]; then EXTRA="" run $lib r$rep; else EXTRA="--gather ce" run $lib ce$rep; EXTRA="--gather pull" run $lib pull$rep; fi
  done
done
cp scripts/libsd_early.so paper_2501_18512_b200/libsd.so
