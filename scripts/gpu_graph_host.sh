cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "graph or host_output or async or workspace" > gpurun_out/gh_pytest.log 2>&1; tail -5 gpurun_out/gh_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/gh_bench.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/gh_bench.log').readlines()[0]);print(d['value'],d['ms_per_step']);print(json.dumps(d['e2e'])[:900])"
tail -c 600 gpurun_out/gh_bench.log
