# ncu --set full of the keygen step's ring-product kernels (one large launch each): stall reasons
# (instruction-fetch stalls among them), pipes, shared-memory wavefronts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-prod}
for K in "tc_mul_kernelINS_6ParamsILi761ELi4591ELi286ELi3EEELi4591ELi2ELi2ELi2ELi128ELb0ELi128ELi1E" \
         "tc_mul_kernelINS_6ParamsILi761ELi4591ELi286ELi3EEELi4591ELi2ELi2ELi1ELi128ELb0ELi128ELi1E" \
         "tc4_mul_kernelINS_6ParamsILi761ELi4591ELi286ELi3EEELi3ELi1ELi2ELb0ELi0ELb0E" \
         "tc4_mul_kernelINS_6ParamsILi761ELi4591ELi286ELi3EEELi3ELi1ELi1ELb0ELi0ELb0E" "sample_kernelINS_6ParamsILi761"; do
  N=$(echo "$K" | sed 's/INS_6ParamsILi761ELi4591ELi286ELi3EEE/_/' | tr -cd 'a-zA-Z0-9_' | cut -c1-40)
  timeout 600 ncu -f --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$K" \
     --launch-skip ${SKIP:-0} -c ${CNT:-1} -o gpurun_out/${T}_$N python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_$N.log 2>&1
  echo "$N rc=$?"
  ncu -i gpurun_out/${T}_$N.ncu-rep --page raw --csv > gpurun_out/${T}_${N}_raw.csv 2>&1
  [ "${SRC:-1}" = "1" ] && ncu -i gpurun_out/${T}_$N.ncu-rep --page source --csv > gpurun_out/${T}_${N}_source.csv 2>&1
  rm -f gpurun_out/${T}_$N.ncu-rep
done
ls -la gpurun_out | grep $T
