cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/keygen_once.py 761 65536 > /dev/null 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:sample_kernel -c 1 \
    -o /tmp/prof_samp python scripts/keygen_once.py 761 65536 > gpurun_out/ncu_samp.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_samp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/source_samp.csv 2>&1
ncu -i /tmp/prof_samp.ncu-rep --page details --csv > gpurun_out/details_samp.csv 2>&1
