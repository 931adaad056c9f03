cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider -k "small_check_policies or cfg1 or param_sets or repair or chunking" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for r in 1 2; do
for opt in "" "--ring-streams"; do for cfg in "1024 32768" "512 65536"; do set -- $cfg
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --batch-size $1 --chunk-keys $2 $opt > gpurun_out/ab3.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/ab3.log').readlines()[0]);print('B $1 chunk $2 $opt', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3))"
done; done; done
