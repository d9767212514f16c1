# Final round-2 evidence on 4 GPUs (tag $1): full GPU suite with junit XML, 2000-round soaks per gather mode,
# the default bench with timelines, 4B at M = 4, the configs[4] sweep.  Every step is time-bounded.
mkdir -p gpurun_out
TAG=${1:-final}
SHA=$(cat .head_sha 2>/dev/null || echo unknown)
echo "head $SHA"; nvidia-smi -L
timeout 2700 python -m pytest tests -m gpu -q -rs --junitxml=gpurun_out/junit_${TAG}_n4.xml > gpurun_out/pytest_${TAG}_n4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}_n4.log
: > gpurun_out/soak_${TAG}_n4.txt
for G in ce push pull; do
  SD_TEST_GATHER=$G SD_TEST_ROUNDS=2000 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/dist_soak_worker.py > gpurun_out/soak_${TAG}_$G.log 2>&1
  echo "$G 2000 rounds: rc=$? $(grep -c "rounds: OK" gpurun_out/soak_${TAG}_$G.log) OK line(s)" | tee -a gpurun_out/soak_${TAG}_n4.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --timeline gpurun_out/timeline_${TAG}_n4.json > gpurun_out/bench4_${TAG}.json 2> gpurun_out/bench4_${TAG}.err; echo "bench rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --workload 4B --steps 128 --no-e2e > gpurun_out/bench4_${TAG}_4B.json 2> gpurun_out/bench4_${TAG}_4B.err; echo "bench 4B rc=$?"
if [ "${SWEEP:-0}" = 1 ]; then timeout 1500 bash scripts/gpu_sweep_multi.sh 4; fi
