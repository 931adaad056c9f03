# GPU test suite against the bounds-checked build (device-side SNTRUP_CHECK asserts compiled in;
# compute-sanitizer is not available on the B200 pool).  Build it first here:
#   python -c "import paper_2106_08759_b200._build as b; b.build_checked()"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export SNTRUP_GPU_LIB=$GRAFT_REPO_ROOT/paper_2106_08759_b200/libsntrup_gpu_check.so
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_checked.log
tail -3 gpurun_out/pytest_checked.log
python scripts/sanitize_small.py > gpurun_out/san_checked.log 2>&1; echo "sanitize_small rc=$?"
grep -c "SNTRUP_CHECK failed" gpurun_out/pytest_checked.log gpurun_out/san_checked.log
