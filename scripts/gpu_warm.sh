cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 3 50 3 50 10 20; do
  python bench.py --steps 10 --warmup $w --no-extras 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); print('warmup', d['warmup'], 'value %.2f M  ms %.3f' % (d['value']/1e6, d['ms_per_step']), d['clocks'])"
done > gpurun_out/warm_ab.log 2>&1
cat gpurun_out/warm_ab.log
