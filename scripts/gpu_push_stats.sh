# push kernel with NSIG signal warps: parity, stats, A/B of variants, NVLink hardware counters
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 600 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
echo "--- stats K=1"
BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py one_peer 2 2>&1 | grep -E "^rank|Error" | sort | head
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_sig2.so variants/lib_sig8.so variants/lib_batch8.so variants/lib_lag24.so variants/lib_batch2.so; do
  for cfg in "2 one_peer" "4 one_peer" "4 exp2"; do set -- $cfg
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents $1 --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology $2 2>&1)
    echo "$(basename $lib) agents=$1 $2 $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done
done
done
echo "--- NVLink counters"
for xf in push pull; do
BF_XFER=$xf timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29542 scripts/nvlink_bytes.py one_peer 2 200 2>&1 | grep "^{" | tee -a gpurun_out/nvlink_bytes.jsonl
done
nvidia-smi nvlink -gt d 2>&1 | head -20
