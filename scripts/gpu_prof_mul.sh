cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 > gpurun_out/mul_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_mul_kernel -c 3 \
    -o gpurun_out/prof_tc2 python scripts/mul_bench.py --n 65536 --impl tc --iters 1 > gpurun_out/ncu_tc.log 2>&1
echo "rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log
