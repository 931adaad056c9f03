cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tc4_mul_kernel|sample_kernel|encode_kernel" -s 12 -c 6 \
    -o gpurun_out/prof_v5 python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_v5.log 2>&1
echo "rc=$?"
