# A/B of library variants across GPUs: K=1, K=4 one-peer / exp-2 (alternating, 2 reps) + multi-process tests
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 400 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 120 python -m torch.distributed.run --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stress_mp.py 1 40 2>&1 | grep "^rank" | head -2
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3))'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  for cfg in "2 one_peer" "8 one_peer" "8 exp2"; do set -- $cfg
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents $1 --steps 60 --warmup 6 --no-e2e --topology $2 2>&1 | grep '^{' | tail -1)
    echo "$(basename $lib) agents=$1 $2 $(echo "$out" | python -c "$summ" 2>/dev/null)"
  done
done
done
