# 2 GPUs: bench N=2 per gather mode (no e2e / overlap), tag $1
mkdir -p gpurun_out
TAG=${1:-r2b}
for G in ${GATHERS:-ce pull push}; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 128 --warmup 8 --gather $G --no-e2e --no-overlap ${EXTRA} > gpurun_out/bench_${TAG}_n2_$G.json 2> gpurun_out/bench_${TAG}_n2_$G.err; echo "bench $G rc=$?"; grep -v OMP_NUM\|\*\*\* gpurun_out/bench_${TAG}_n2_$G.err | tail -3
python -c "
import json; j=json.loads(open('gpurun_out/bench_${TAG}_n2_$G.json').read().strip().splitlines()[-1])
print('$G', 'value %.4g per_gpu %.4g ms %.4f apply %.3f quant %.3f ser %.4g launches %d' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac'], j['value_serialized'], j['gpu_launches']))"
done
