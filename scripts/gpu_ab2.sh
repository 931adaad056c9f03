cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider -k "kem or rq_mul or r3_mul or cfg1" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for r in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --batch-size 512 --chunk-keys 65536 > gpurun_out/ab_new.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/ab_new.log').readlines()[0]);print('NEW', round(d['value']/1e6,3), d['breakdown_ms_per_step'])"
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras > gpurun_out/ab_new2.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/ab_new2.log').readlines()[0]);print('NEW default', round(d['value']/1e6,3), d['clocks'])"
done
