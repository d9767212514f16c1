# A/B of libsd builds incl. the emulated M sweep: default and each .so given
mkdir -p gpurun_out
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset SD_LIBSD; else export SD_LIBSD=$lib; fi
  python bench.py --steps 256 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python - $lib <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']; ms=j['m_sweep_emulated']
print(sys.argv[1][-18:], 'value %.4e q %.3f a %.3f'%(j['value'], k['k_quantize']['frac'], k['k_apply']['frac']),
      {m:(round(v['apply_frac'],3), round(v['apply_ms']*1e3,1)) for m,v in ms.items()})
PY
done
