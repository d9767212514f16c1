# 4 GPUs: the full default bench at N=4 (copy engines; overlap check + timeline), then pull and push; tag $1
mkdir -p gpurun_out
TAG=${1:-r2}
N=${N:-4}
nvidia-smi topo -m | head -6
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --timeline gpurun_out/timeline_${TAG}_n$N.json > gpurun_out/bench${N}_$TAG.json 2> gpurun_out/bench${N}_$TAG.err; echo "bench rc=$?"; grep -v "OMP\|\*\*\*" gpurun_out/bench${N}_$TAG.err | tail -6
for G in pull push; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --gather $G --no-e2e --no-overlap > gpurun_out/bench${N}_${TAG}_$G.json 2> gpurun_out/bench${N}_${TAG}_$G.err; echo "bench $G rc=$?"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 256 --warmup 8 --tau 0 --no-e2e --no-overlap > gpurun_out/bench${N}_${TAG}_tau0.json 2> gpurun_out/bench${N}_${TAG}_tau0.err; echo "bench tau0 rc=$?"
python - <<PY
import json
for f in ('bench${N}_$TAG','bench${N}_${TAG}_pull','bench${N}_${TAG}_push','bench${N}_${TAG}_tau0'):
    try:
        j=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'no json', e); continue
    k=j['kernels']
    print(f, 'value %.4g per_gpu %.4g ms %.4f apply %.3f quant %.3f ser %s' % (j['value'], j['per_gpu_value'], j['ms_per_step'], k['k_apply']['frac'], k['k_quantize']['frac'], j['value_serialized']))
    for kk in ('overlap','e2e','e2e_offloaded_state','clocks'):
        if j.get(kk) is not None: print('  ', kk, json.dumps(j[kk])[:900])
PY
