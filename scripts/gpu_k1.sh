# K = 1 (one agent per GPU, the N = 8 configuration's per-GPU shape) at N = 2 and 4
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
N=$(nvidia-smi -L | wc -l)
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["achieved"],1), round(r["frac"],3), round(r["frac_per_round_bound"],3), [(round(b["ms"],3), round(b["t_roof_ms"],3)) for b in r["by_round"]])'
for n in 2 4; do
  [ $n -le $N ] || continue
  for topo in one_peer exp2; do
    out=$(timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $n --agents $n --steps 60 --warmup 6 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
    echo "N=$n K=1 $topo $(echo "$out" | python -c "$summ" 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
