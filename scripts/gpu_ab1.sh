# A/B of library variants at N=1 in one call (alternating, 3 repetitions)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3))'
for rep in 1 2 3; do
  for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
    for topo in ${TOPOS:-one_peer}; do
      echo "$(basename $lib) $topo $(BF_LIB_PATH=$lib timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1 | python -c "$summ")"
    done
  done
done
