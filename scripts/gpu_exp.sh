cd $GRAFT_REPO_ROOT
for e in 2 4 2 4; do
SNTRUP_EXP=$e timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/exp$e.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/exp$e.log').readlines()[0]);print('exp $e', d['value'],d['ms_per_step'], d['e2e']['value'])"
done
