# the two 8-process time-shared tests on the box's GPUs (timed)
cd $GRAFT_REPO_ROOT
nvidia-smi -L
timeout 1800 python -m pytest tests/test_multigpu.py -k eight -v -p no:cacheprovider --durations=0 > gpurun_out/pytest_n8_shared.log 2>&1
echo "rc=$?"; tail -15 gpurun_out/pytest_n8_shared.log
