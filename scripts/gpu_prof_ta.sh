# ncu capture of the TMEM-A fp4 kernel (impl 9) vs default (impl 0) on R/3 products
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in ${IMPLS:-9 0}; do
  timeout 300 python scripts/mul_bench.py --impl $i --which r3 --iters 2 --n 65536 > /dev/null 2>&1 || echo "plain run failed"
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:tc4_mul -c 1 -o /tmp/prof_ta$i \
      python scripts/mul_bench.py --impl $i --which r3 --iters 1 --n 65536 > gpurun_out/ncu_ta$i.log 2>&1
  echo "ncu $i rc=$?"
  ncu -i /tmp/prof_ta$i.ncu-rep --page details --csv > gpurun_out/details_ta$i.csv 2>&1
  ncu -i /tmp/prof_ta$i.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/source_ta$i.csv 2>&1
  ncu -i /tmp/prof_ta$i.ncu-rep --page raw --csv > gpurun_out/raw_ta$i.csv 2>&1
done
