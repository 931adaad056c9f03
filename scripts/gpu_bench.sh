cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which r3 > gpurun_out/mul_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_mul_kernel -c 1 \
    -o gpurun_out/prof_tc_r3 python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which r3 > gpurun_out/ncu_tc.log 2>&1
echo "ncu rc=$?"
