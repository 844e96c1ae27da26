# K = 4 push with the parked lag sized by the agents that wait (exchange_push.cuh):
# parity of every K with push forced for all K = 4 rounds, then bench A/B
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
BF_XFER=push_all timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -x > gpurun_out/mp_pushall_n$N.log 2>&1; echo "mp push_all rc=$?"; tail -2 gpurun_out/mp_pushall_n$N.log
AGENTS="8 $((2*N))" LIBS="variants/lib_lag24.so" bash scripts/gpu_variants_ab.sh 2>&1 | tee gpurun_out/k4lag_ab_n$N.txt
BF_XFER=push_all AGENTS="8" TOPOS=one_peer LIBS="variants/lib_lag24.so" bash scripts/gpu_variants_ab.sh 2>&1 | tee -a gpurun_out/k4lag_ab_n$N.txt
