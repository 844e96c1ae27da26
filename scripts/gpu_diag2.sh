# Diagnostics: HBM efficiency of the fused kernel per local-agent count K, and N=2 with no exchange
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["achieved"],1), round(r["frac"],3), d["clocks"]["sm_mhz"])'
for ag in 8 8 4 2 1; do
  for topo in one_peer; do
    out=$(timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo --agents $ag --count $((25600000*8/ag)) 2>&1 | tail -1)
    echo "N=1 agents=$ag count=$((25600000*8/ag)) $topo $(echo "$out" | python -c "$summ" 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
out=$(timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --topology self 2>&1 | grep '^{' | tail -1)
echo "N=$N self $(echo "$out" | python -c "$summ" 2>/dev/null || echo "$out" | tail -c 300)"
