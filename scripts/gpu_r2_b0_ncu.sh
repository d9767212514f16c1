# ncu of the staged B = 0 quantize: launch list of three quantizes, then a --set full capture of one pass-2 kernel
mkdir -p gpurun_out
python scripts/b0_staged_once.py || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python scripts/b0_staged_once.py > gpurun_out/b0_launches.csv 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"${B0_NCU_K:-k_encode_staged}" --launch-skip 1 --launch-count 1 -o gpurun_out/b0_staged -f python scripts/b0_staged_once.py > gpurun_out/b0_ncu.log 2>&1
tail -3 gpurun_out/b0_ncu.log
grep -E "k_absmax|k_encode" gpurun_out/b0_launches.csv | awk -F'","' '{print $5, $NF}'
