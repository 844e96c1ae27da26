cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "not eight" > gpurun_out/pf2_mp.log 2>&1; echo "mp rc=$?"; tail -1 gpurun_out/pf2_mp.log
AGENTS="4 8" TOPOS="one_peer exp2" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
