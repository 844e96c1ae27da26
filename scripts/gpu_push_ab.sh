# A/B of the cross-GPU transfer: push (default) vs pull, N = #GPUs, K = 1 and 2
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["frac"],3), round(r.get("frac_per_round_bound",0),3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for agents in $N $((2*N)) 8; do
 for topo in one_peer exp2; do
  for xf in push pull; do
   out=$(BF_XFER=$xf timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-cpu --agents $agents --topology $topo 2>&1)
   echo "N=$N agents=$agents $topo $xf: $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done
 done
done
