cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
K=${2:-tc_mul_kernel}
python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which ${3:-rq} > gpurun_out/mulp_$TAG.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o /tmp/prof_$TAG python scripts/mul_bench.py --n 65536 --impl tc --iters 1 --which ${3:-rq} > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/details_$TAG.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/source_$TAG.csv 2>&1
ls -la gpurun_out/
