# pull kernel reading a published agent's x_half back from its own slot (fp32 wire nar / ATC):
# parity with the default paths and with every cross-GPU call pulled, then bench A/B
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "parity and not eight" > gpurun_out/slotx_mp.log 2>&1; echo "mp default rc=$?"; tail -1 gpurun_out/slotx_mp.log
BF_XFER=pull timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "parity and not eight" > gpurun_out/slotx_mp_pull.log 2>&1; echo "mp pull rc=$?"; tail -1 gpurun_out/slotx_mp_pull.log
AGENTS="8 4" TOPOS="one_peer exp2" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
BF_XFER=pull AGENTS="8 2" TOPOS="one_peer" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
