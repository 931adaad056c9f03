cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "param_sets or cfg1 or rq_recip or kem" > gpurun_out/kparts_pytest2.log 2>&1; tail -3 gpurun_out/kparts_pytest2.log
for e in 0 2 3 4 0 2 3 4; do EXP1277=$e timeout 300 python scripts/exp1277.py 1277 2>&1 | tail -1; done > gpurun_out/kparts_1277.log; cat gpurun_out/kparts_1277.log
for r in 1 2; do timeout 300 python scripts/impl_ab.py 0 14 2>&1 | tail -2; done > gpurun_out/kparts_impl_ab3.log 2>&1; cat gpurun_out/kparts_impl_ab3.log
