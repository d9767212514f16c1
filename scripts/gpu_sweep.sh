# 1-GPU sweep of the BASELINE configs through bench.py (JSON lines -> gpurun_out/sweep_*.json)
mkdir -p gpurun_out
run() { tag=$1; shift; python bench.py "$@" > gpurun_out/sweep_$tag.json 2> gpurun_out/sweep_$tag.err; echo "$tag rc=$?"; }
run toy --workload toy --no-cpu-baseline
run 35M --workload 35M --no-cpu-baseline
run 1B_B0 --workload 1B --scale-block 0 --no-cpu-baseline --no-e2e
run 1B_B256 --workload 1B --scale-block 256 --no-cpu-baseline --no-e2e --no-m-sweep
run 4B --workload 4B --no-cpu-baseline
for f in gpurun_out/sweep_*.json; do python - $f <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=j['kernels']
print(sys.argv[1].split('_',1)[1], 'value %.3e'%j['value'], 'ms %.4f'%j['ms_per_step'], 'q %.3f a %.3f cp %.3f'%(k['k_quantize']['frac'],k['k_apply']['frac'],k['critical_path_frac']),
      'e2e', j['e2e'] and '%.3e'%j['e2e']['value'], 'l2', j['config']['l2'][:40])
if j['m_sweep_emulated']: print('   m_sweep', {m:(round(v['apply_frac'],3), '%.3e'%v['params_per_s_per_gpu']) for m,v in j['m_sweep_emulated'].items()})
PY
done
