# 2 GPUs: 35M and toy bench lines (N=1, N=2), the end-to-end example on 2 GPUs (35M and 1B); tag $1
mkdir -p gpurun_out
TAG=${1:-r2}
for W in toy 35M; do
python bench.py --workload $W --steps 256 --warmup 8 --no-cpu-baseline --no-extras > gpurun_out/bench_${TAG}_${W}_n1.json 2> gpurun_out/bench_${TAG}_${W}_n1.err; echo "bench $W n1 rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload $W --steps 256 --warmup 8 --no-e2e --no-overlap > gpurun_out/bench_${TAG}_${W}_n2.json 2> gpurun_out/bench_${TAG}_${W}_n2.err; echo "bench $W n2 rc=$?"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 examples/train_streaming_diloco.py --steps 300 > gpurun_out/train_35m_2gpu_$TAG.log 2>&1; echo "train 35M rc=$?"; tail -2 gpurun_out/train_35m_2gpu_$TAG.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 examples/train_streaming_diloco.py --steps 300 --d-model 2048 --layers 24 --fragment-size 3 --H 100 --tau 5 --batch 4 --seq 1024 --amp --log-every 50 > gpurun_out/train_1b_2gpu_$TAG.log 2>&1; echo "train 1B rc=$?"; tail -3 gpurun_out/train_1b_2gpu_$TAG.log
python - <<PY
import json
for W in ('toy','35M'):
    for N in ('n1','n2'):
        try:
            j=json.loads(open('gpurun_out/bench_${TAG}_%s_%s.json'%(W,N)).read().strip().splitlines()[-1])
            print(W, N, 'value %.4g'%j['value'], 'q %.3f a %.3f'%(j['kernels']['k_quantize']['frac'], j['kernels']['k_apply']['frac']), j['schedule'][:40], (j.get('cuda_graph') or {}).get('value_eager'))
        except Exception as e: print(W, N, 'err', e)
PY
