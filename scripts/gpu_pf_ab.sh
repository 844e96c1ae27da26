# push kernel: the next sub-item's x / g loads issued before the combine also at K = 2 (pf2) and K = 1 (pf1)
cd $GRAFT_REPO_ROOT
AGENTS="2 4" TOPOS="one_peer exp2" LIBS="variants/lib_pf2.so variants/lib_pf1.so" bash scripts/gpu_variants_ab.sh
