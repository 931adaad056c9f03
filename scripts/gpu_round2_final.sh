# Round-2 validation and evidence: the whole GPU suite, smoke, bench, the ncu launch list of the
# same bench command, per-kernel pipe metrics, and one full capture of the dominant kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${T}_nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
tail -4 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
tail -2 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.log
tail -c 300 gpurun_out/${T}_bench.log
if [ "${PROFILE:-1}" = "1" ]; then
  python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_plain.log 2>&1
  timeout 900 ncu -f --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv \
      --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_ncu_launches.log 2>&1
  echo "launches rc=$?"
  MET=smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
  for k in tc_mul_kernel tc4_mul_kernel sample_kernel divstep encode_kernel repair_kernel; do
    timeout 600 ncu -f --metrics $MET --clock-control none -k regex:$k -c 80 \
        -o /tmp/prof_${T}_$k python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_ncu_$k.log 2>&1
    echo "$k rc=$?"
    ncu -i /tmp/prof_${T}_$k.ncu-rep --page raw --csv > gpurun_out/${T}_pipes_$k.csv
  done
  # one full capture (source page) of the dominant kernel's largest launch: the int8 two-product
  # kernel's h launch (16,384 work items; the 10th launch of that kernel in a chunk)
  timeout 900 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:tc_mul_kernel.*int.1, .int.2>' --launch-skip 9 -c 1 \
      -o gpurun_out/${T}_full_tc_mul python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/${T}_ncu_full.log 2>&1
  echo "full rc=$?"
  ncu -i gpurun_out/${T}_full_tc_mul.ncu-rep --page raw --csv > gpurun_out/${T}_full_tc_mul_raw.csv 2>&1
  ncu -i gpurun_out/${T}_full_tc_mul.ncu-rep --page details --csv > gpurun_out/${T}_full_tc_mul_details.csv 2>&1
fi
du -sh gpurun_out
