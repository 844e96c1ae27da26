cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
timeout 60 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 90 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
TOPOS="self one_peer exp2" VTIMEOUT=60 bash scripts/gpu_variants.sh
