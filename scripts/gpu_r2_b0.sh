# staged B = 0 quantize: parity subset, the probe per staging-hint setting, bench.py at B = 0, then ncu of the two passes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "quantize or no_writes" 2>&1 | tail -5 > gpurun_out/b0_pytest.log
cat gpurun_out/b0_pytest.log
for h in ${B0_HINTS:-3 0 1 2}; do
  SD_STAGE_HINTS=$h timeout 300 python scripts/b0_probe.py 2>/dev/null | tail -1 >> gpurun_out/b0_probe.jsonl
done
timeout 300 python bench.py --scale-block 0 --steps 128 --no-e2e --no-cpu-baseline --no-m-sweep 2>/dev/null | tail -1 > gpurun_out/b0_bench.json
python - <<'PY'
import json
for l in open('gpurun_out/b0_probe.jsonl'):
    j = json.loads(l)
    print(j['hints'], 'staged %.1f us frac %.3f | reread %.1f us frac %.3f | adamw fused %.1f (reread %.1f) sep %.1f (reread %.1f)' % (
        j['quantize_ms']*1e3, j['frac_algorithmic'], j['reread']['quantize_ms']*1e3, j['reread']['frac_algorithmic'],
        j['inner_adamw_before_send']['fused_ms']*1e3, j['inner_adamw_before_send']['reread']['fused_ms']*1e3,
        j['inner_adamw_before_send']['separate_ms']*1e3, j['inner_adamw_before_send']['reread']['separate_ms']*1e3))
j = json.loads(open('gpurun_out/b0_bench.json').read())
k = j['kernels']
print('bench B=0 value %.4e q %.3f (%.1f us) a %.3f' % (j['value'], k['k_quantize']['frac'], k['k_quantize']['avg_ms']*1e3, k['k_apply']['frac']))
PY
if [ "${B0_NCU:-1}" = 1 ]; then bash scripts/gpu_r2_b0_ncu.sh; grep -E "k_absmax|k_encode" gpurun_out/b0_launches.csv | awk -F'","' '{print $5, $NF}' | tail -4; fi
