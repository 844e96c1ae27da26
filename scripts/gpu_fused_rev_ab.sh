# N = 1: the fused kernel's reverse walk of odd epochs per operation (ATC bench line, E, H, GT, IO)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))'
for rep in 1 2; do for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_fnorev.so; do
  echo "== $(basename $lib) rep $rep"
  echo "C4 $(BF_LIB_PATH=$lib timeout 120 python bench.py --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar 2>&1 | python -c "$summ")"
  echo "C4 exp2 $(BF_LIB_PATH=$lib timeout 120 python bench.py --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology exp2 2>&1 | python -c "$summ")"
  BF_LIB_PATH=$lib timeout 300 python bench_suite.py --only e,h,gt,io --out /dev/null 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:60], round(d.get('ms', d.get('ms_per_step', d.get('ms_per_round', 0))),4), d.get('hbm_frac'))"
done; done
