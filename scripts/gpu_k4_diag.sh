# K = 4 local-streaming diagnostics: the fused kernel with 4 agents on one GPU (no
# cross-GPU protocol), and the push kernel with / without its release fence (timing only)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for agents in 4 8; do for topo in one_peer exp2; do
  out=$(CUDA_VISIBLE_DEVICES=0 timeout 120 python bench.py --agents $agents --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology $topo 2>&1)
  echo "N=1 agents=$agents $topo $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
done; done
BF_XFER=push_all AGENTS=8 TOPOS="one_peer exp2" LIBS="variants/lib_nofence.so" bash scripts/gpu_variants_ab.sh
AGENTS=4 TOPOS="one_peer" LIBS="variants/lib_nofence.so" bash scripts/gpu_variants_ab.sh
