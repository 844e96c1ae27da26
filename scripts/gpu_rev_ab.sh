cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for rep in 1 2 3; do for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_norev.so; do
  echo "$(basename $lib) $(BF_LIB_PATH=$lib timeout 200 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu --no-nar 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["value"],1), round(d["roofline"]["frac"],4))')"
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -x -p no:cacheprovider 2>&1 | tail -1
