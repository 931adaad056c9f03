# round 2: new full-size / boundary GPU tests first, then the whole GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_nvsmi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_fullsize.py -q --timeout 600 -p no:cacheprovider \
  -k "not cfg4 and not 857 and not 953 and not 1013" > gpurun_out/r2_new_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_new_tests.log
tail -15 gpurun_out/r2_new_tests.log
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider --ignore=tests/test_gpu_fullsize.py --ignore=tests/test_gpu_boundary.py > gpurun_out/r2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest_gpu.log
tail -5 gpurun_out/r2_pytest_gpu.log
