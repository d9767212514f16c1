# pull apply with R tiles per CTA and the next tile's peer code words loaded early (SD_PULL_R=R) at N = ${N:-4}
mkdir -p gpurun_out
N=${N:-4}
run() {  # $1 tag, $2 gather
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --gather $2 --no-e2e --no-overlap > gpurun_out/pr_$1.json 2> gpurun_out/pr_$1.err
  python -c "
import json; j=json.loads(open('gpurun_out/pr_$1.json').read().strip().splitlines()[-1])
print('$1', 'value %.4e per_gpu %.4e ms %.4f apply %.4f quant %.4f' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac']))"
}
for R in 2 4; do SD_PULL_R=$R timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "pull and (four or two_ranks) and not inner" 2>&1 | tail -1 | sed "s/^/R=$R: /"; done
SD_PULL_R=1 run pull_r1 pull
SD_PULL_R=2 run pull_r2 pull
SD_PULL_R=4 run pull_r4 pull
run ce ce
SD_PULL_R=1 run pull_r1b pull
SD_PULL_R=4 run pull_r4b pull
