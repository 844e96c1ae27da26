# final-tree bench lines at the per-GPU shape of the 8-GPU setting (K = 1) and the other agent counts
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
AGENTS="$N $((2*N)) 8" TOPOS="one_peer exp2" LIBS=" " bash scripts/gpu_variants_ab.sh
