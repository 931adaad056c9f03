# ncu --set full of the jump-divstep root kernel: default build and the two timing-split builds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-pj}
for L in libsntrup_gpu libsntrup_gpu_jm1 libsntrup_gpu_jm2; do
  SNTRUP_GPU_LIB=$PWD/paper_2106_08759_b200/$L.so timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:jump_ -c 1 \
     -o gpurun_out/${T}_$L python scripts/root_once.py 761 0 q > gpurun_out/${T}_$L.log 2>&1
  echo "$L rc=$?"
  ncu -i gpurun_out/${T}_$L.ncu-rep --page raw --csv > gpurun_out/${T}_${L}_raw.csv 2>&1
  ncu -i gpurun_out/${T}_$L.ncu-rep --page source --csv > gpurun_out/${T}_${L}_source.csv 2>&1
  rm -f gpurun_out/${T}_$L.ncu-rep
done
