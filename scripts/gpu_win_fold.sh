cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -x -p no:cacheprovider -k "window or win_" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_suite.py --only c5 2>&1 | grep '^{'
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
