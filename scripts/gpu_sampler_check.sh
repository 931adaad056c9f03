# GPU tests + plain bench + sampler ncu source page (after a sampler change).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pyt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pyt_$TAG.log
tail -2 gpurun_out/pyt_$TAG.log
python bench.py --steps 10 --warmup 3 --no-extras > gpurun_out/plain_$TAG.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/plain_$TAG.log').readlines()[0]);print(d['value'],d['ms_per_step']);print(d['breakdown_ms_per_step']);print(d['roofline']['by_kind_ms_per_step'])"
bash scripts/gpu_prof_sample.sh
