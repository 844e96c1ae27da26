# C5 window round (340M bf16 x 8, one GPU) for library variants (LIBS=, default variants/*.so)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  echo "$(basename $lib) $(BF_LIB_PATH=$lib timeout 300 python bench_suite.py --only c5 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_round"],3), d["sum_p"])')"
done
done
