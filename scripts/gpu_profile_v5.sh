cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_v5.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which rq > gpurun_out/mul_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_mul_kernel -c 1 \
    -o gpurun_out/prof_tc_v5 python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which rq > gpurun_out/ncu_tc.log 2>&1
echo "full rc=$?"
