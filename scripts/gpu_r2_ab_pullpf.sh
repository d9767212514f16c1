# pull apply: L2 prefetch of the peers' code words k waves ahead (SD_PULL_PREFETCH=k) at N = ${N:-4}; copy engines as reference
mkdir -p gpurun_out
N=${N:-4}
run() {  # $1 tag, $2 gather
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --gather $2 --no-e2e --no-overlap > gpurun_out/pf_$1.json 2> gpurun_out/pf_$1.err
  python -c "
import json; j=json.loads(open('gpurun_out/pf_$1.json').read().strip().splitlines()[-1])
print('$1', 'value %.4e per_gpu %.4e ms %.4f apply %.4f quant %.4f' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac']))"
}
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "pull and (two_ranks or four)" 2>&1 | tail -1
for k in ${KS:-0 1 2 4}; do SD_PULL_PREFETCH=$k run pull_k$k pull; done
run ce ce
SD_PULL_PREFETCH=0 run pull_k0b pull
