cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_quick.sh || exit 1
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which rq > gpurun_out/mul_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_mul_kernel -c 1 \
    -o gpurun_out/prof_tc3 python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which rq > gpurun_out/ncu_tc.log 2>&1
echo "ncu rc=$?"
