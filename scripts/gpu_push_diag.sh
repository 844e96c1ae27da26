# window kernels (NV-deep loads) check + C5 at N=1; push-kernel diagnostics and A/B at N=2
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -x -p no:cacheprovider -k "window" 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench_suite.py --only c5 --out gpurun_out/c5_n1.jsonl 2>&1 | tail -2
echo "--- stats K=1"
BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py one_peer 2 2>&1 | grep -E "^rank|Error" | sort | head
echo "--- stats K=2"
BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py one_peer 4 2>&1 | grep -E "^rank|Error" | sort | head
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_lag8.so variants/lib_lag24.so variants/lib_batch2.so variants/lib_batch8.so; do
  for agents in 2 4; do
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents $agents --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology one_peer 2>&1)
    echo "$(basename $lib) agents=$agents $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done
done
done
out=$(BF_XFER=pull timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --agents 2 --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology self 2>&1)
echo "self (W=I) agents=2: $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
