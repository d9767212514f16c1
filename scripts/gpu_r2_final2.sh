# Final round-2 evidence on 2 GPUs (tag $1): full GPU suite with junit XML, default bench, configs[4] sweep.
mkdir -p gpurun_out
TAG=${1:-final}
SHA=$(cat .head_sha 2>/dev/null || echo unknown)
echo "head $SHA"; nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -q -rs --junitxml=gpurun_out/junit_${TAG}_n2.xml > gpurun_out/pytest_${TAG}_n2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --timeline gpurun_out/timeline_${TAG}_n2.json > gpurun_out/bench2_${TAG}.json 2> gpurun_out/bench2_${TAG}.err; echo "bench rc=$?"
if [ "${SWEEP:-0}" = 1 ]; then timeout 1200 bash scripts/gpu_sweep_multi.sh 2; fi
