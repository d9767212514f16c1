# B = 0 (two-pass quantize): default build vs each .so given, bench.py --scale-block 0
mkdir -p gpurun_out
for i in 1 2; do
  for lib in default "$@"; do
    if [ "$lib" = default ]; then unset SD_LIBSD; else export SD_LIBSD=$lib; fi
    python bench.py --scale-block 0 --steps 128 --no-e2e --no-cpu-baseline --no-m-sweep > gpurun_out/ab.json 2>/dev/null
    python - $lib <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']
print(sys.argv[1][-18:], 'value %.4e q %.3f (%.1f us) a %.3f'%(j['value'], k['k_quantize']['frac'], k['k_quantize']['avg_ms']*1e3, k['k_apply']['frac']))
PY
  done
done
