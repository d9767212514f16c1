# 2 GPUs: round-1 libsd (scripts/libsd_r1.so) vs the current one, same bench, pull and ce
mkdir -p gpurun_out
run() {  # $1 tag, $2 gather
  python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-2} --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus ${N:-2} --steps 256 --warmup 8 --gather $2 --no-e2e --no-overlap > gpurun_out/abr1_$1.json 2> gpurun_out/abr1_$1.err
  python -c "
import json; j=json.loads(open('gpurun_out/abr1_$1.json').read().strip().splitlines()[-1])
print('$1', 'value %.4g per_gpu %.4g ms %.4f apply %.3f %.4f quant %.3f launches %d' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_apply']['avg_ms'], j['kernels']['k_quantize']['frac'], j['gpu_launches']))"
}
SD_LIBSD=$PWD/scripts/libsd_r1.so run r1_pull pull
run now_pull pull
SD_LIBSD=$PWD/scripts/libsd_r1.so run r1_pull_b pull
run now_pull_b pull
SD_LIBSD=$PWD/scripts/libsd_r1.so run r1_ce ce
run now_ce ce
