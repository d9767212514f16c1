# grid-size sweep: bench.py at several SD_BLOCKS_PER_SM caps (CTAs per SM) on 1 GPU -> gpurun_out/grid_*.json
mkdir -p gpurun_out
for k in ${KS:-8 16 32 64 100000}; do
  SD_BLOCKS_PER_SM=$k python bench.py --steps 64 --warmup 8 --no-e2e --no-cpu-baseline > gpurun_out/grid_$k.json 2>/dev/null
  python - $k <<'PY'
import json,sys
j=json.loads(open(f'gpurun_out/grid_{sys.argv[1]}.json').read().strip().splitlines()[-1])
ms=j['m_sweep_emulated']
print('bps',sys.argv[1],'value %.3e'%j['value'],'q %.3f a %.3f'%(j['kernels']['k_quantize']['frac'],j['kernels']['k_apply']['frac']),
      'sweep', {k:(round(v['quantize_frac'],3),round(v['apply_frac'],3)) for k,v in ms.items()})
PY
done
