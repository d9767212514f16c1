# 2 GPUs: fused last-CTA signal vs separate signal kernel, pull and push modes (bench N=2, 128 steps)
mkdir -p gpurun_out
for SK in 0 1; do
  for G in pull push; do
    SD_SIGNAL_KERNEL=$SK python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 128 --warmup 8 --gather $G --no-e2e --no-overlap > gpurun_out/ab_sig${SK}_$G.json 2> gpurun_out/ab_sig${SK}_$G.err
    python -c "
import json; j=json.loads(open('gpurun_out/ab_sig${SK}_$G.json').read().strip().splitlines()[-1])
print('signal_kernel=$SK $G', 'value %.4g ms %.4f apply %.3f quant %.3f ser %.4g launches %d' % (j['value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac'], j['value_serialized'], j['gpu_launches']))"
  done
done
