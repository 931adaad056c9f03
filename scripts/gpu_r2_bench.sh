# round 2: bench (serialised pass, int peaks, fixed e2e) + smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
tail -2 gpurun_out/r2_smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
tail -c 3000 gpurun_out/r2_bench.log
