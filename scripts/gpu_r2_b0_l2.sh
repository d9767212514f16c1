# staged B = 0: MB of summaries kept in L2 between the passes (SD_STAGE_L2_MB) A/B, after the staged parity tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "quantize and (staged or B0 or 65536 or 2048 or 4096)" 2>&1 | tail -1 > gpurun_out/b0_l2_pytest.log
cat gpurun_out/b0_l2_pytest.log
for mb in ${MBS:-0 20 40 60 90}; do
  SD_STAGE_L2_MB=$mb timeout 300 python scripts/b0_probe.py 2>/dev/null | tail -1 | sed "s/^{/{\"l2mb\": $mb, /" >> gpurun_out/b0_l2_probe.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/b0_l2_probe.jsonl'):
    j = json.loads(l)
    print('l2mb', j['l2mb'], 'staged %.1f us frac %.3f | reread %.1f | adamw fused %.1f' % (
        j['quantize_ms']*1e3, j['frac_algorithmic'], j['reread']['quantize_ms']*1e3, j['inner_adamw_before_send']['fused_ms']*1e3))
PY
