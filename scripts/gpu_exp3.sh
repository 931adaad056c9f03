cd $GRAFT_REPO_ROOT
for r in 1 2; do for cfg in "512 65536" "1024 32768" "1024 65536"; do set -- $cfg
timeout 300 python bench.py --steps 30 --warmup 5 --no-extras --batch-size $1 --chunk-keys $2 > gpurun_out/e3.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/e3.log').readlines()[0]);print('B $1 chunk $2', round(d['value']/1e6,3), round(d['ms_per_step'],4), d['clocks'])"
done; done
