cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for lib in paper_2111_04287_b200/libbluefog_b200.so variants/*.so; do
  echo "$(basename $lib) $(BF_LIB_PATH=$lib timeout 120 python bench_suite.py --only c1 2>&1 | grep -o '"us_per_iteration": [0-9.]*' | tr '\n' ' ')"
done; done
