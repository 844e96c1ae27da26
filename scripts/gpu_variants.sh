# Tuning sweep of build variants (tile size / occupancy) on the N=1 bench config.
cd $GRAFT_REPO_ROOT
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/*.so; do
  for topo in ${TOPOS:-one_peer exp2}; do
    out=$(BF_LIB_PATH=$lib timeout ${VTIMEOUT:-300} python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
    echo "$lib $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
