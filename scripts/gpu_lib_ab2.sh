# A/B of two library builds (SNTRUP_GPU_LIB): isolated ring products and the keygen step, alternating
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
OLD=paper_2106_08759_b200/libsntrup_gpu_old.so
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "r3_mul or cfg1 or param_sets or kem" > gpurun_out/pyt_$TAG.log 2>&1; tail -2 gpurun_out/pyt_$TAG.log
for r in 1 2 3; do
  echo "old:"; SNTRUP_GPU_LIB=$OLD timeout 300 python scripts/mul_bench.py --impl tc --iters 5 --which rq,rqs,r3 2>&1
  echo "new:"; timeout 300 python scripts/mul_bench.py --impl tc --iters 5 --which rq,rqs,r3 2>&1
done > gpurun_out/libab_mul_$TAG.log
cat gpurun_out/libab_mul_$TAG.log
for r in 1 2 3; do
  echo "old:"; SNTRUP_GPU_LIB=$OLD timeout 300 python scripts/impl_ab.py 0 2>&1 | tail -1
  echo "new:"; timeout 300 python scripts/impl_ab.py 0 2>&1 | tail -1
done > gpurun_out/libab_$TAG.log
cat gpurun_out/libab_$TAG.log
