cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/plain.log 2>&1 || exit 1
MET=smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread
for k in tc_mul_kernel tc4_mul_kernel sample_kernel joint_roots_kernel encode_kernel; do
  ncu -f --metrics $MET --clock-control none -k regex:$k -c 80 \
      -o /tmp/prof6_$k python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu6_$k.log 2>&1
  echo "$k rc=$?"
  ls -la /tmp/prof6_$k.ncu-rep
  ncu -i /tmp/prof6_$k.ncu-rep --page raw --csv > gpurun_out/prof6_$k.csv
done
du -sh gpurun_out
