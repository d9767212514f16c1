# 4 GPUs: bench N=4 per gather mode and signal form (128 steps, no e2e/overlap)
mkdir -p gpurun_out
run() {  # $1 tag, $2 gather, env in caller
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 128 --warmup 8 --gather $2 --no-e2e --no-overlap $EXTRA > gpurun_out/ab4_$1.json 2> gpurun_out/ab4_$1.err
  python -c "
import json; j=json.loads(open('gpurun_out/ab4_$1.json').read().strip().splitlines()[-1])
print('$1', 'value %.4g per_gpu %.4g ms %.4f apply %.3f quant %.3f ser %.4g launches %d' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac'], j['value_serialized'], j['gpu_launches']))"
}
run ce ce
SD_SIGNAL_KERNEL=0 run pull_fused pull
SD_SIGNAL_KERNEL=1 run pull_sigk pull
SD_SIGNAL_KERNEL=0 run push_fused push
SD_SIGNAL_KERNEL=1 run push_sigk push
EXTRA="--tau 0" run ce_tau0 ce
EXTRA="--tau 0" SD_SIGNAL_KERNEL=0 run pull_tau0 pull
EXTRA="--tau 0" SD_SIGNAL_KERNEL=1 run pull_sigk_tau0 pull
