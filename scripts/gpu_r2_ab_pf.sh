# N GPUs: pull apply with code prefetch (SD_PULL_ITERS = 1 (k_apply), 2, 4, 8), tau 0 and tau 5
mkdir -p gpurun_out
N=${N:-2}
for TAU in 0 5; do
for R in 1 2 4 8; do
  SD_PULL_ITERS=$R python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --gather pull --tau $TAU --no-e2e --no-overlap > gpurun_out/abpf_n${N}_t${TAU}_r$R.json 2> gpurun_out/abpf_n${N}_t${TAU}_r$R.err
  python -c "
import json; j=json.loads(open('gpurun_out/abpf_n${N}_t${TAU}_r$R.json').read().strip().splitlines()[-1])
print('N=$N tau=$TAU iters=$R', 'value %.4g per_gpu %.4g ms %.4f apply %.3f quant %.3f' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac']))"
done
done
