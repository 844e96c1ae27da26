# push kernel: multi-process parity (both workers), then the A/B
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_mp.log 2>&1; echo "mp tests rc=$?"; tail -5 gpurun_out/pytest_mp.log
bash scripts/gpu_push_ab.sh
