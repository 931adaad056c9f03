# round 2, session 3: new tests, the timeline of one overlapped step, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider -k "graph or attempts_only" > gpurun_out/r2s3_pytest_new.log 2>&1; tail -3 gpurun_out/r2s3_pytest_new.log
timeout 300 python scripts/timeline.py gpurun_out/r2s3_timeline.csv > gpurun_out/r2s3_timeline.log 2>&1; head -12 gpurun_out/r2s3_timeline.log
