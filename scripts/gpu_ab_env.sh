# A/B of an environment setting on the same box: "$1" (e.g. SD_QUANTIZE_TMA=1) vs default
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in default "$1"; do
    if [ "$v" = default ]; then E=""; else E="$v"; fi
    env $E python bench.py --steps 256 --no-e2e --no-cpu-baseline --no-m-sweep > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$v" <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']
print(sys.argv[1][:24], 'value %.4e ms %.4f q %.3f (%.1f us) a %.3f'%(j['value'], j['ms_per_step'], k['k_quantize']['frac'], k['k_quantize']['avg_ms']*1e3, k['k_apply']['frac']))
PY
  done
done
