cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/plain20.log 2>&1 || exit 1
# launch list of the same command (per-launch device time + DRAM bytes; serialised, cold cache)
ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_v20.csv python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_launches20.log 2>&1
echo "launches rc=$?"
MET=smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for k in tc_mul_kernel tc4_mul_kernel sample_kernel divstep encode_kernel repair_kernel; do
  ncu -f --metrics $MET --clock-control none -k regex:$k -c 80 \
      -o /tmp/prof20_$k python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu20_$k.log 2>&1
  echo "$k rc=$?"
  ncu -i /tmp/prof20_$k.ncu-rep --page raw --csv > gpurun_out/prof20_$k.csv
done
du -sh gpurun_out
