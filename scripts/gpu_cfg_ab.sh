cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=16
timeout 600 python scripts/config_ab.py 1024:32768:$R 2048:32768:$R 2048:65536:$R 1024:65536:$R 4096:65536:$R 4096:32768:$R 2048:16384:$((R|32)) > gpurun_out/cfg_ab_kparts.log 2>&1
cat gpurun_out/cfg_ab_kparts.log
