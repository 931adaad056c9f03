# full capture (source page) of the fp4 two-product kernel's largest launch (R/3 down-sweep, bottom level)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2s4d}
timeout 900 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:tc4_mul_kernel.*int.3, .int.1, .int.2,' --launch-skip 9 -c 1 \
    -o gpurun_out/${T}_full_tc4_down python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_ncu_full_tc4.log 2>&1
echo "full rc=$?"
ncu -i gpurun_out/${T}_full_tc4_down.ncu-rep --page raw --csv > gpurun_out/${T}_full_tc4_down_raw.csv 2>&1
ncu -i gpurun_out/${T}_full_tc4_down.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${T}_full_tc4_down_source.csv 2>&1 || \
ncu -i gpurun_out/${T}_full_tc4_down.ncu-rep --page source --csv > gpurun_out/${T}_full_tc4_down_source.csv 2>&1
ls -la gpurun_out/${T}_*
