cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_nopf.so; do
  for cfg in "2 one_peer push" "4 one_peer push" "8 exp2 push" "8 one_peer push_all"; do set -- $cfg
    out=$(BF_XFER=$3 BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents $1 --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology $2 2>&1)
    echo "$(basename $lib) $3 agents=$1 $2 $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done
done
done
