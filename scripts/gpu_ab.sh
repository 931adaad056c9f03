cd $GRAFT_REPO_ROOT
for r in 1 2; do
(cd abtest && timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --batch-size 512 --chunk-keys 65536 > ../gpurun_out/ab_old.log 2>&1)
python -c "
import json;d=json.loads(open('gpurun_out/ab_old.log').readlines()[0]);print('OLD', round(d['value']/1e6,3), d['breakdown_ms_per_step'])"
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --batch-size 512 --chunk-keys 65536 > gpurun_out/ab_new.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/ab_new.log').readlines()[0]);print('NEW', round(d['value']/1e6,3), d['breakdown_ms_per_step'])"
done
