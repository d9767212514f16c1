# configs[4]: tau and fragment-size sweep of the 1B workload at N GPUs (JSON lines -> gpurun_out/msweep_N_*.json)
mkdir -p gpurun_out
N=${1:-2}
run() { tag=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 128 --no-e2e "$@" > gpurun_out/msweep_${N}_$tag.json 2> gpurun_out/msweep_${N}_$tag.err; echo "$tag rc=$?"; }
for tau in 0 1 2 5; do run tau$tau --tau $tau; done
for fs in 1 2 4 6; do run fs$fs --fragment-size $fs; done
for f in gpurun_out/msweep_${N}_*.json; do python - $f <<'PY'
import json,sys
j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=j['kernels']; o=j.get('overlap') or {}
ad=o.get('adamw') or {}; gm=o.get('gemm') or {}
print(sys.argv[1].split('msweep_')[1][:-5], 'value %.3e per_gpu %.3e ser %s ms %.4f q %.3f a %.3f'%(j['value'], j['per_gpu_value'], j.get('value_serialized') and '%.3e'%j['value_serialized'], j['ms_per_step'], k['k_quantize']['frac'], k['k_apply']['frac']),
      'gather %s exposed adamw %s gemm %s' % (ad.get('gather_alone_ms') and round(ad['gather_alone_ms'],3), ad.get('exposed_ms') is not None and round(ad['exposed_ms'],3), gm.get('exposed_ms') is not None and round(gm['exposed_ms'],3)), j['config']['gather'][:20])
PY
done
