cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider -k "host or cfg1 or chunking or param_sets" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "rc=0" gpurun_out/pytest_gpu.log || exit 1
bash scripts/gpu_bench2.sh
