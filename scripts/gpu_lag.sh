cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 300 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"
grep -E "Error|error|assert|FAIL|mismatch|rel err" gpurun_out/pytest_multi.log | head -20
export BF_TIMEOUT_MS=5000
for lag in 8 16 24 32; do
  export BF_FUSED_LAG=$lag
  LIBS=" " bash scripts/gpu_var2.sh | sed "s/^/lag=$lag /"
done
