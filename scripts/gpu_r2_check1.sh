# 1 GPU: GPU test subset (-k $1) + bench N=1 extras record for B = 0, tag $2
mkdir -p gpurun_out
TAG=${2:-r2}
python -m pytest tests -m gpu -q -x -k "${1:-adamw}" > gpurun_out/pytest1_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest1_$TAG.log
python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench1x_$TAG.json 2> gpurun_out/bench1x_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench1x_$TAG.err
python -c "
import json; j=json.loads(open('gpurun_out/bench1x_$TAG.json').read().strip().splitlines()[-1])
print(json.dumps(j['quantize_B0'])); print(json.dumps(j['inner_adamw_fused'])); print('value', j['value'])"
