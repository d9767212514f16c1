# 2 GPUs: full GPU suite (junit), then bench N=2 for the copy-engine and fused-pull gathers
mkdir -p gpurun_out
TAG=${1:-r2a}
python -m pytest tests -m gpu -q -x -rs --junitxml=gpurun_out/junit_${TAG}_n2.xml > gpurun_out/pytest_${TAG}_n2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}_n2.log
for G in ce pull push; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 64 --warmup 8 --gather $G --no-e2e > gpurun_out/bench_${TAG}_n2_$G.json 2> gpurun_out/bench_${TAG}_n2_$G.err; echo "bench $G rc=$?"; tail -2 gpurun_out/bench_${TAG}_n2_$G.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_${TAG}_n2_$G.json').read().strip().splitlines()[-1])
print('$G', 'value %.4g per_gpu %.4g ms %.4f apply %.3f quant %.3f ser %s' % (j['value'], j['per_gpu_value'], j['ms_per_step'], j['kernels']['k_apply']['frac'], j['kernels']['k_quantize']['frac'], j['value_serialized']))"
done
