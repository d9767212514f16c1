# 1-GPU: tests, bench, ncu launch list + full capture (tag $1)
mkdir -p gpurun_out
TAG=${1:-r1}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
bash scripts/gpu_bench_profile.sh $TAG
du -sh gpurun_out; ls -la gpurun_out/*.ncu-rep
