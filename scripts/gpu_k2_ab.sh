cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_b8.so variants/lib_l8.so variants/lib_s2.so variants/lib_s8.so; do
  for topo in one_peer exp2; do
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --agents 8 --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology $topo 2>&1)
    echo "$(basename $lib) K=2 $topo $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done
done
done
