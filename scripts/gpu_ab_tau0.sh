# default build vs each .so given, at tau = 0 (serialized: the apply follows the same fragment's quantize)
# and at the default tau (pipelined), 1 GPU
mkdir -p gpurun_out
for i in 1 2; do
  for args in "--tau 0" ""; do
    for lib in default "$@"; do
      if [ "$lib" = default ]; then unset SD_LIBSD; else export SD_LIBSD=$lib; fi
      python bench.py $args --steps 256 --no-e2e --no-cpu-baseline --no-m-sweep > gpurun_out/ab.json 2>/dev/null
      python - "$lib" "$args" <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']
print(sys.argv[1][-20:], sys.argv[2] or 'pipelined', 'value %.4e q %.3f a %.3f (%.1f us)'%(j['value'], k['k_quantize']['frac'], k['k_apply']['frac'], k['k_apply']['avg_ms']*1e3))
PY
    done
  done
done
