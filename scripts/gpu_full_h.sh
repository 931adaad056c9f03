# one full capture (source page included) of the dominant kernel's largest launch: the int8
# two-product ring-product kernel's h launch (16,384 work items) of bench.py's step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2s4b}
timeout 900 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:tc_mul_kernel.*int.1, .int.2>' --launch-skip 9 -c 1 \
    -o gpurun_out/${T}_full_tc_mul_h python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_ncu_full_h.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/${T}_ncu_full_h.log | cut -c1-300
ncu -i gpurun_out/${T}_full_tc_mul_h.ncu-rep --page raw --csv > gpurun_out/${T}_full_tc_mul_h_raw.csv 2>&1
ncu -i gpurun_out/${T}_full_tc_mul_h.ncu-rep --page source --csv > gpurun_out/${T}_full_tc_mul_h_source.csv 2>&1
ls -la gpurun_out/${T}_*
