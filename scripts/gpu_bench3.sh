cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log | cut -c1-300
python -c "
import json;d=json.loads(open('gpurun_out/bench.log').readlines()[0]);print(d['value'],d['ms_per_step']);print(json.dumps(d['other_configs'], indent=1))"
