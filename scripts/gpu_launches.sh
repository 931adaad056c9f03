cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
python scripts/mul_bench.py --n 262144 --impl tc --iters 5 > gpurun_out/mul_$TAG.log 2>&1
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
