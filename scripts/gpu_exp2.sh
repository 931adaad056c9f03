cd $GRAFT_REPO_ROOT
for B in 512 1024 2048; do for C in 65536 32768; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --batch-size $B --chunk-keys $C > gpurun_out/e_${B}_${C}.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/e_${B}_${C}.log').readlines()[0]);print('B $B chunk $C', round(d['value']/1e6,3), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,3))"
done; done
