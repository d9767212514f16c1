# k_apply_tma variants (SD_APPLY_TMA=1 with each libsd build given) vs the direct-load k_apply
mkdir -p gpurun_out
for lib in direct default "$@"; do
  if [ "$lib" = direct ]; then unset SD_LIBSD; export SD_APPLY_TMA=0; elif [ "$lib" = default ]; then unset SD_LIBSD; export SD_APPLY_TMA=1; else export SD_LIBSD=$lib SD_APPLY_TMA=1; fi
  python bench.py --steps 128 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python - "$lib" <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']; ms=j['m_sweep_emulated']
print(sys.argv[1][-22:], 'value %.4e a %.3f'%(j['value'], k['k_apply']['frac']), 'sweep apply', {m:round(v['apply_frac'],3) for m,v in ms.items()})
PY
done
