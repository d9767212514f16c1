# round-2 baseline on N GPUs ($1): full GPU suite with junit XML, then bench under torchrun
mkdir -p gpurun_out
N=${1:-4}
SHA=$(cat .head_sha 2>/dev/null || echo unknown)
nvidia-smi -L
python -m pytest tests -m gpu -q -rs --junitxml=gpurun_out/junit_r2base_n$N.xml > gpurun_out/pytest_r2base_n$N.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2base_n$N.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 64 --warmup 8 > gpurun_out/bench_r2base_n$N.json 2> gpurun_out/bench_r2base_n$N.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_r2base_n$N.err
