# Final round-2 evidence on 1 GPU (tag $1): GPU suite with junit XML, smoke, default bench, reference arm, 35M/toy.
mkdir -p gpurun_out
TAG=${1:-final}
SHA=$(cat .head_sha 2>/dev/null || echo unknown)
echo "head $SHA"; nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q -rs --junitxml=gpurun_out/junit_${TAG}_n1.xml > gpurun_out/pytest_${TAG}_n1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench1_${TAG}.json 2> gpurun_out/bench1_${TAG}.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench1s_${TAG}.json 2> gpurun_out/bench1s_${TAG}.err; echo "bench driver-form rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench1ref_${TAG}.json 2> gpurun_out/bench1ref_${TAG}.err; echo "ref rc=$?"
for W in toy 35M; do timeout 600 python bench.py --workload $W --no-cpu-baseline --no-extras > gpurun_out/bench1_${TAG}_$W.json 2> gpurun_out/bench1_${TAG}_$W.err; echo "bench $W rc=$?"; done
