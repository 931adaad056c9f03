cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/mul_bench.py --n 262144 > gpurun_out/mul_bench.log 2>&1 && \
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 > gpurun_out/mul_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_mul_kernel -c 3 \
    -o gpurun_out/prof_tc python scripts/mul_bench.py --n 65536 --impl tc --iters 1 > gpurun_out/ncu_tc.log 2>&1
echo "rc=$?"
cat gpurun_out/mul_bench.log
