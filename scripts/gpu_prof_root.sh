# ncu of the root inversion kernels (32 rows, B = 1): launch list and one full capture each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-root}
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python scripts/root_once.py 761 2 q > /dev/null 2>&1
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_step.csv python scripts/root_once.py 761 1 q > /dev/null 2>&1
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r3.csv python scripts/root_once.py 761 2 3 > /dev/null 2>&1
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:jump_ -c 1 -o gpurun_out/${T}_full_jump python scripts/root_once.py 761 2 q > gpurun_out/${T}_ncu.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/${T}_full_jump.ncu-rep --page raw --csv > gpurun_out/${T}_full_jump_raw.csv 2>&1
ncu -i gpurun_out/${T}_full_jump.ncu-rep --page source --csv > gpurun_out/${T}_full_jump_source.csv 2>&1
ncu -i gpurun_out/${T}_full_jump.ncu-rep --page details --csv > gpurun_out/${T}_full_jump_details.csv 2>&1
ls -la gpurun_out
ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r3_step.csv python scripts/root_once.py 761 1 3 > /dev/null 2>&1
for ps in 653 857 953 1013 1277; do
  for impl in 2 1; do
    ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_${ps}_${impl}.csv python scripts/root_once.py $ps $impl q > /dev/null 2>&1
    ncu -f --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_${ps}_${impl}_r3.csv python scripts/root_once.py $ps $impl 3 > /dev/null 2>&1
  done
done
SNTRUP_GPU_LIB=$PWD/paper_2106_08759_b200/libsntrup_gpu_jt.so python scripts/jump_trace.py > gpurun_out/${T}_jump_trace.log 2>&1
rm -f gpurun_out/*.ncu-rep
