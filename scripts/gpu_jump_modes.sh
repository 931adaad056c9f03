# jump-divstep timing split: full kernel, decisions only (mode 1), application only (mode 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-jm}
for L in libsntrup_gpu libsntrup_gpu_jm1 libsntrup_gpu_jm2; do
  for ps in 761 1277; do
    SNTRUP_GPU_LIB=$PWD/paper_2106_08759_b200/$L.so ncu -f --metrics gpu__time_duration.sum --clock-control none -k regex:jump_ --csv \
      --log-file gpurun_out/${T}_${L}_${ps}.csv python scripts/root_once.py $ps 0 q > /dev/null 2>&1
    echo "$L $ps $(grep jump_ gpurun_out/${T}_${L}_${ps}.csv | tail -1 | awk -F'","' '{print $NF}')"
  done
done
