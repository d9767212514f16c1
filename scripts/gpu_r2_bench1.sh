# 1 GPU: smoke, bench N=1 (defaults and the driver's short form), reference arm; tag $1
mkdir -p gpurun_out
TAG=${1:-r2}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
python bench.py > gpurun_out/bench1_$TAG.json 2> gpurun_out/bench1_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench1_$TAG.err
python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/bench1s_$TAG.json 2> gpurun_out/bench1s_$TAG.err; echo "bench short rc=$?"; tail -3 gpurun_out/bench1s_$TAG.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench1ref_$TAG.json 2> gpurun_out/bench1ref_$TAG.err; echo "ref rc=$?"; tail -3 gpurun_out/bench1ref_$TAG.err
python - <<PY
import json
for f in ('bench1_$TAG','bench1s_$TAG','bench1ref_$TAG'):
    try:
        j=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'no json', e); continue
    print(f, 'value %.4g'%j['value'], 'ms', j.get('ms_per_step'), 'roofline', (j.get('roofline') or {}).get('frac'), 'e2e', (j.get('e2e') or {}).get('value'))
    for k in ('e2e_offloaded_state','configs','quantize_B0','cpu_baseline','clocks'):
        if j.get(k) is not None: print('  ', k, json.dumps(j[k])[:600])
PY
