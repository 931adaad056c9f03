# ncu full capture of one warp-specialised kernel launch (mul_bench r3, impl 11)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ws}
K=${2:-tc4w_mul_kernel}
W=${3:-r3}
I=${4:-11}
python scripts/mul_bench.py --n 262144 --impl $I --iters 1 --which $W > gpurun_out/mulp_$TAG.log 2>&1 && \
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o /tmp/prof_$TAG python scripts/mul_bench.py --n 262144 --impl $I --iters 1 --which $W > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/details_$TAG.csv 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/source_$TAG.csv 2>&1
cp /tmp/prof_$TAG.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out/ | tail -5
