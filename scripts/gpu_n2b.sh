# N=2 bench with per-round detail for the fused kernel at several chunk sizes
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
for ct in ${CTS:-1024 256 64}; do
  for topo in ${TOPOS:-one_peer exp2}; do
    out=$(BF_CHUNK_TILES=$ct timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 60 --warmup 6 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
    echo "N=$N ct=$ct $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3), [(round(b["ms"],3), round(b["t_roof_ms"],3)) for b in r["by_round"]])' 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
