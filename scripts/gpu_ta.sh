# A/B of the TMEM-A fp4 variant (impl 9) against the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "tc_tmem_a" > gpurun_out/pyt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_$TAG.log
tail -3 gpurun_out/pyt_$TAG.log
for i in 0 9 10; do timeout 300 python scripts/mul_bench.py --impl $i --which r3,rqt --iters 5; done > gpurun_out/mul_$TAG.log 2>&1; cat gpurun_out/mul_$TAG.log
timeout 600 python scripts/impl_ab.py 0 9 10 > gpurun_out/ab_$TAG.log 2>&1; cat gpurun_out/ab_$TAG.log
