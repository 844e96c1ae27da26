# GPU test pass (any number of GPUs): every -m gpu test, logs under gpurun_out/
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
