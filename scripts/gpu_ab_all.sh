# A/B of library variants: N=1 bench, N=2 (K=4, K=1) benches
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3))'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/*.so; do
  echo "$(basename $lib) N=1 $(BF_LIB_PATH=$lib timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "$summ")"
  for cfg in "2 one_peer" "8 one_peer" "8 exp2"; do set -- $cfg
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents $1 --steps 60 --warmup 6 --no-e2e --topology $2 2>&1 | grep '^{' | tail -1)
    echo "$(basename $lib) N=2 agents=$1 $2 $(echo "$out" | python -c "$summ" 2>/dev/null)"
  done
done
done
