# round 2, session 3: A/B of the default multiplier set against u fused with level 1 (impl 7),
# twice, alternating rounds; plus isolated ring-product rates
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2; do timeout 300 python scripts/impl_ab.py 0 7 0 7 2>&1 | tail -4; done > gpurun_out/r2s3_impl_ab.log
cat gpurun_out/r2s3_impl_ab.log
timeout 300 python scripts/mul_bench.py --impl tc --iters 5 > gpurun_out/r2s3_mul_bench.log 2>&1
cat gpurun_out/r2s3_mul_bench.log
