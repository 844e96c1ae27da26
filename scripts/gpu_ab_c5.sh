# A/B of window-kernel variants on C5 (alternating), one GPU
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for rep in 1 2; do
  for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
    BF_LIB_PATH=$lib timeout 300 python bench_suite.py --only c5 > gpurun_out/c5.log 2>&1
    echo "$(basename $lib) $(grep -o '"ms_per_round": [0-9.]*' gpurun_out/c5.log)"
  done
done
