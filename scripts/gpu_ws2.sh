cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ws}
timeout 300 python scripts/mul_bench.py --impl 0,11 --which rq,r3 --n 1048576 > gpurun_out/${T}_mul.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_mul.log
cat gpurun_out/${T}_mul.log
SNTRUP_GPU_LIB=paper_2106_08759_b200/libsntrup_gpu_trace.so timeout 120 python scripts/ws_trace.py > gpurun_out/${T}_trace.log 2>&1
cat gpurun_out/${T}_trace.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python scripts/impl_ab.py 0 11 > gpurun_out/${T}_ab.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_ab.log
cat gpurun_out/${T}_ab.log
