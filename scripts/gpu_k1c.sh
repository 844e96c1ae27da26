cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3))'
for rep in 1 2; do
for lib in variants/lib_lb3.so variants/lib_lb2.so; do
for grid in 0 296 222; do
  out=$(BF_LIB_PATH=$lib BF_FUSED_GRID=$grid timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents 2 --steps 60 --warmup 6 --no-e2e --topology one_peer 2>&1 | grep '^{' | tail -1)
  echo "$(basename $lib) grid=$grid K=1 $(echo "$out" | python -c "$summ" 2>/dev/null || echo "$out" | tail -c 200)"
done
done
done
