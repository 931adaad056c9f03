# A/B of two builds of the library (SNTRUP_GPU_LIB): alternating processes, keygen step + ring products
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
OLD=paper_2106_08759_b200/libsntrup_gpu_old.so
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "mul or keygen_cfg or kem" > gpurun_out/pyt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_$TAG.log
tail -2 gpurun_out/pyt_$TAG.log
for r in 1 2 3; do
  echo "old:"; SNTRUP_GPU_LIB=$OLD timeout 300 python scripts/impl_ab.py 0 2>&1 | tail -1
  echo "new:"; timeout 300 python scripts/impl_ab.py 0 2>&1 | tail -1
done > gpurun_out/libab_$TAG.log
cat gpurun_out/libab_$TAG.log
echo "old:"; SNTRUP_GPU_LIB=$OLD timeout 300 python scripts/mul_bench.py --impl tc --iters 5 2>&1
echo "new:"; timeout 300 python scripts/mul_bench.py --impl tc --iters 5 2>&1
