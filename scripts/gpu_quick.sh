cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "rq_mul or r3_mul or cfg1" -p no:cacheprovider > gpurun_out/pytest_mul.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mul.log
tail -3 gpurun_out/pytest_mul.log
grep -q "rc=0" gpurun_out/pytest_mul.log || exit 1
timeout 300 python scripts/mul_bench.py --n 262144 > gpurun_out/mul_bench.log 2>&1
cat gpurun_out/mul_bench.log
