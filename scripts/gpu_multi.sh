# N GPUs ($1, default 2): multi-GPU tests, then bench.py under torchrun; prints value, roofline, overlap, clocks
mkdir -p gpurun_out
N=${1:-2}
nvidia-smi topo -m | head -8
python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_$N.log 2>&1; echo "pytest multi rc=$?"; tail -5 gpurun_out/pytest_multi_$N.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench rc=$?"; tail -5 gpurun_out/bench_n$N.err
python - <<PY
import json
j=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1])
print('value',j['value'],'per_gpu',j['per_gpu_value'],'ms/step',j['ms_per_step'])
print('roofline',j['roofline']['frac'],'kernels',j['kernels'])
print('overlap',json.dumps(j['overlap']))
print('clocks',j['clocks'],'e2e',j['e2e'] and j['e2e']['value'])
PY
