cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
for lib in variants/lib_L24B8G1.so variants/lib_L48B8G1.so; do
  BF_LIB_PATH=$lib BF_TIMEOUT_MS=8000 timeout 300 python -m pytest tests/test_multigpu.py -q -x 2>&1 | tail -1
done
bash scripts/gpu_var2.sh
