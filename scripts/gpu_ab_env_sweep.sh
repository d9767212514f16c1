# A/B of an environment setting incl. the emulated M sweep: "$1" (e.g. SD_APPLY_TMA=1) vs default, 2 rounds
mkdir -p gpurun_out
for i in 1 2; do
  for v in default "$1"; do
    if [ "$v" = default ]; then E=""; else E="$v"; fi
    env $E python bench.py --steps 256 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$v" <<'PY'
import json,sys
j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k=j['kernels']; ms=j['m_sweep_emulated']
print(sys.argv[1][:24], 'value %.4e ms %.4f q %.3f a %.3f (%.1f us)'%(j['value'], j['ms_per_step'], k['k_quantize']['frac'], k['k_apply']['frac'], k['k_apply']['avg_ms']*1e3),
      'sweep apply', {m:(round(v['apply_frac'],3), round(v['apply_ms']*1e3,1)) for m,v in ms.items()})
PY
  done
done
