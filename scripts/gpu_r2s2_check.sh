# session-2 check: whole GPU suite, smoke, bench, root A/B and root latency per parameter set
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2s2}
TAG=$T PROFILE=0 bash scripts/gpu_round2_final.sh
ROUNDS=10 timeout 600 python scripts/root_ab.py > gpurun_out/${T}_root_ab.log 2>&1; tail -1 gpurun_out/${T}_root_ab.log
timeout 600 python scripts/recip_latency.py > gpurun_out/${T}_recip_latency.log 2>&1; tail -1 gpurun_out/${T}_recip_latency.log
