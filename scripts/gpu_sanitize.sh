cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/sanitize_small.py > gpurun_out/san_plain.log 2>&1 || { echo "plain failed"; tail -5 gpurun_out/san_plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY' gpurun_out/san_$tool.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_$tool.log | head -2)"
done
