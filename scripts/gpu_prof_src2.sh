cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_prof_tc.sh f4d tc4_mul_kernel r3 > /dev/null 2>&1
bash scripts/gpu_prof_tc.sh i8d tc_mul_kernel rq > /dev/null 2>&1
ls gpurun_out | grep -E "f4d|i8d"
