cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
TOPOS="self one_peer" VTIMEOUT=60 bash scripts/gpu_variants.sh
