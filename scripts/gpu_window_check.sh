# window kernels after a launch-bounds change: all GPU tests + C5 line
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/win_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -1 gpurun_out/win_pytest_gpu.log
for r in 1 2; do timeout 300 python bench_suite.py --only c5 > gpurun_out/c5.log 2>&1; echo "C5 $(grep -o '"ms_per_round": [0-9.]*' gpurun_out/c5.log)"; done
