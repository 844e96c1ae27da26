# K = 4 push kernel after "reverse walk for K = 2 only": 1 CTA/SM variant and the
# local-store timing probe (wire copy written into the writer's own heap)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
L="variants/lib_k4minb1.so variants/lib_localstore.so"
AGENTS="8" TOPOS="one_peer exp2" LIBS="$L" bash scripts/gpu_variants_ab.sh
BF_XFER=push_all AGENTS=8 TOPOS="one_peer" LIBS="$L" bash scripts/gpu_variants_ab.sh
