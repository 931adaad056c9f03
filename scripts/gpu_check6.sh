cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pool or cfg1 or chunking or host" -p no:cacheprovider > gpurun_out/pytest_pool.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pool.log
tail -15 gpurun_out/pytest_pool.log
