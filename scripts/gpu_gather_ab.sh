# N GPUs ($1): bench.py per gather mode (GATHERS env, default "ce mc"), REPS rounds -> gpurun_out/gab_n$N_<mode>.json
mkdir -p gpurun_out
N=${1:-2}
for i in $(seq ${REPS:-2}); do
for g in ${GATHERS:-ce mc}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --gather $g --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/gab_n${N}_$g.json 2> gpurun_out/gab_n${N}_$g.err; echo "bench $g rc=$?"
  python - gpurun_out/gab_n${N}_$g.json <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=j['kernels']; o=j.get('overlap') or {}
print(sys.argv[1], 'value %.4e ser %s ms %.4f q %.3f a %.3f'%(j['value'], j.get('value_serialized') and '%.4e'%j['value_serialized'], j['ms_per_step'], k['k_quantize']['frac'], k['k_apply']['frac']))
for kind,v in o.items(): print('  ', kind, 'gather %.3f exposed %.3f hidden %s GB/s %.0f'%(v['gather_alone_ms'], v['exposed_ms'], v['hidden'], v['nvlink']['GBps_per_direction']))
PY
done
done
