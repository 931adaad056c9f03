# transposed int8 ring products (impl 13): parity, then isolated rates against the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "tc_transposed" > gpurun_out/tcx_pytest.log 2>&1; tail -15 gpurun_out/tcx_pytest.log
timeout 300 python scripts/mul_bench.py --impl 0,13,0,13 --which rq,rqs --iters 5 > gpurun_out/tcx_mul_bench.log 2>&1; cat gpurun_out/tcx_mul_bench.log
timeout 300 python scripts/impl_ab.py 0 13 > gpurun_out/tcx_impl_ab.log 2>&1; cat gpurun_out/tcx_impl_ab.log
