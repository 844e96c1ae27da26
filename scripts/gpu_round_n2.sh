# N = 2 round record + K = 4 push knob A/B (batch length, prefetch)
cd $GRAFT_REPO_ROOT
SUITE=c1,h,io,gt,e,c5,o bash scripts/gpu_final.sh
AGENTS=8 TOPOS="one_peer exp2" LIBS="variants/lib_batch6.so variants/lib_nopf.so" bash scripts/gpu_variants_ab.sh > gpurun_out/k4_knobs3_n2.txt 2>&1
