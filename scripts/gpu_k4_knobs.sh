# K = 4 push-kernel knobs at N = 2 (reverse walk, batch length, CTAs per SM, no fence = timing only)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
L="variants/lib_norev.so variants/lib_batch6.so variants/lib_k4minb1.so variants/lib_nofence.so"
AGENTS=8 TOPOS="one_peer exp2" LIBS="$L" bash scripts/gpu_variants_ab.sh
BF_XFER=push_all AGENTS=8 TOPOS="one_peer" LIBS="$L" bash scripts/gpu_variants_ab.sh
