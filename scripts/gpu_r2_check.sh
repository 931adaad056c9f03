# round 2: split build -- whole GPU suite, smoke, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "not cfg4 and not 953 and not 1013" > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
tail -4 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
tail -2 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
tail -c 400 gpurun_out/${T}_bench.log
