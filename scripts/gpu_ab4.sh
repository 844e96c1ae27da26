# A/B of library variants on 4 GPUs: K=1 (agents=4), K=2 (agents=8) one-peer / exp-2
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3))'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  for cfg in "4 one_peer" "8 one_peer" "8 exp2"; do set -- $cfg
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --agents $1 --steps 60 --warmup 6 --no-e2e --topology $2 2>&1 | grep '^{' | tail -1)
    echo "$(basename $lib) N=4 agents=$1 $2 $(echo "$out" | python -c "$summ" 2>/dev/null)"
  done
done
done
