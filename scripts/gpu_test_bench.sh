# 1 GPU: GPU tests then a default bench.py run
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
j=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('value',j['value'],'ms/step',j['ms_per_step'])
print('roofline',j['roofline'])
print('kernels',j['kernels'])
print('m_sweep',json.dumps(j['m_sweep_emulated']))
print('clocks',j['clocks'],'e2e',j['e2e'] and j['e2e']['value'],'cpu',j['cpu_baseline'])
PY
