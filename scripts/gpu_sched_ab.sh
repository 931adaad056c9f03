cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/sched_ab.py ${CFGS:-0:0:16 0:8:16 0:16:16 0:32:16 0:64:16 0:16:144 0:32:144} > gpurun_out/${OUT:-sched_ab2}.log 2>&1
cat gpurun_out/${OUT:-sched_ab2}.log
