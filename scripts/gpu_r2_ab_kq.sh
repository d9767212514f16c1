# 1 GPU: k_adamw_quantize at 2 CTAs/SM (124 regs) vs 3 CTAs/SM (80 regs, 52 B spill): bench extras
for L in default kq3; do
  if [ $L = kq3 ]; then export SD_LIBSD=$PWD/scripts/libsd_kq3.so; else unset SD_LIBSD; fi
  python bench.py --steps 32 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/abkq_$L.json 2> gpurun_out/abkq_$L.err
  python -c "
import json; j=json.loads(open('gpurun_out/abkq_$L.json').read().strip().splitlines()[-1])
f=j['inner_adamw_fused']; print('$L fused_ms %.4f frac %.3f sep %.4f' % (f['fused_ms'], f['fused_frac'], f['separate_ms']))"
done
