# warp-specialised kernels: parity under impl 11, then microbench and keygen A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ws}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider -k "tc_ws" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -15 gpurun_out/${T}_pytest.log
timeout 300 python scripts/mul_bench.py --impl 0,11 --which r3 --n 1048576 > gpurun_out/${T}_mul.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_mul.log
cat gpurun_out/${T}_mul.log
timeout 300 python scripts/impl_ab.py 0 11 > gpurun_out/${T}_ab.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ab.log
cat gpurun_out/${T}_ab.log
