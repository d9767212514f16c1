# N GPUs ($1): bench.py per gather mode (GATHERS env, default ce push pull) -> gpurun_out/bench_n$N_<mode>.json
mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_push_$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_push_$N.log
for g in ${GATHERS:-ce push pull}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --gather $g --no-e2e > gpurun_out/bench_n${N}_$g.json 2> gpurun_out/bench_n${N}_$g.err; echo "bench $g rc=$?"
  python - gpurun_out/bench_n${N}_$g.json <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=j['kernels']; o=j.get('overlap') or {}
print(sys.argv[1], 'value %.3e ser %s ms %.4f q %.3f a %.3f'%(j['value'], j.get('value_serialized') and '%.3e'%j['value_serialized'], j['ms_per_step'], k['k_quantize']['frac'], k['k_apply']['frac']))
for kind,v in o.items(): print('  ', kind, 'gather %.3f exposed %.3f hidden %s'%(v['gather_alone_ms'], v['exposed_ms'], v['hidden']))
PY
done
