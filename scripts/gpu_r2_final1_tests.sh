# 1-GPU suite + smoke only at the head (tag $1): junit XML
mkdir -p gpurun_out
TAG=${1:-final}
SHA=$(cat .head_sha 2>/dev/null || echo unknown)
echo "head $SHA"; nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q -rs --junitxml=gpurun_out/junit_${TAG}_n1.xml > gpurun_out/pytest_${TAG}_n1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
