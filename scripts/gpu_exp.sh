cd $GRAFT_REPO_ROOT
for e in 256 512 128 256 512; do
SNTRUP_JNT=$e timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/exp$e.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/exp$e.log').readlines()[0]);print('nt $e', d['value'],d['ms_per_step'], d['breakdown_ms_per_step']['root_inv'])"
done
