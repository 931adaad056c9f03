cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sample_kernel|encode_kernel|divstep" -s 4 -c 4 \
    -o gpurun_out/prof_v6 python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_v6.log 2>&1
echo "rc=$?"
