cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "parity and (2-4 or 2-2)" 2>&1 | tail -1
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do for xf in push pull; do
    out=$(BF_XFER=$xf timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents 8 --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology one_peer 2>&1)
    echo "$xf agents=8 one_peer $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
done; done
