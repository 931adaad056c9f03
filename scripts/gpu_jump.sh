cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rq_root_jump or rq_recip" -p no:cacheprovider > gpurun_out/j1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j1_pytest.log
tail -15 gpurun_out/j1_pytest.log
timeout 300 python scripts/recip_latency.py > gpurun_out/j1_lat.log 2>&1; echo "rc=$?" >> gpurun_out/j1_lat.log
cat gpurun_out/j1_lat.log | tail -9
TAG=jm2 bash scripts/gpu_jump_modes.sh
