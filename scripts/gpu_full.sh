cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
grep -q "rc=0" gpurun_out/pytest_gpu.log || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
python -c "
import json;d=json.loads(open('gpurun_out/bench.log').readlines()[0]);print(d['value'],d['ms_per_step']);print(d['breakdown_ms_per_step']);print(d['e2e']['value'], d['chunk_sweep_keys_per_s']);print(json.dumps(d['other_configs']))"
