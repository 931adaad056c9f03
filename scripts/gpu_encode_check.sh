# encode_kernel change check: keygen/KEM parity subset + per-launch ncu time of encode_kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "keygen or encode or pk or kem or full_sk" > gpurun_out/pyt_enc.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_enc.log
tail -2 gpurun_out/pyt_enc.log
python scripts/keygen_once.py 761 65536 > /dev/null 2>&1 || echo "plain failed"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:encode_kernel -c 4 --csv \
    python scripts/keygen_once.py 761 65536 2>/dev/null | grep encode_kernel | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
