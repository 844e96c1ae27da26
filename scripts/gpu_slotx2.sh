cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
AGENTS="8" TOPOS="one_peer" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
BF_XFER=pull AGENTS="2" TOPOS="one_peer" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
