# A/B of two library builds (SNTRUP_GPU_LIB=old vs the in-tree one): parity subset on the new one,
# then alternating processes of the bench-style keygen step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
OLD=$GRAFT_REPO_ROOT/paper_2106_08759_b200/libsntrup_gpu_base.so
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "param_sets or cfg1_every_key_bench or r3_mul or r3_recip or kem" > gpurun_out/pyt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_$TAG.log
tail -2 gpurun_out/pyt_$TAG.log
for r in 1 2 3; do
  echo "old:"; SNTRUP_GPU_LIB=$OLD timeout 300 python scripts/bench_style_ab.py 1024:32768:16 2>&1 | tail -1
  echo "new:"; timeout 300 python scripts/bench_style_ab.py 1024:32768:16 2>&1 | tail -1
done > gpurun_out/libab_$TAG.log
cat gpurun_out/libab_$TAG.log
