cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ring_mul_kernel -s 60 -c 2 \
    -o gpurun_out/prof_ringmul python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
