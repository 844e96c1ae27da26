# 4-GPU record: all GPU tests, bench N=4 (8 agents and 4 agents), C1 latency, H
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_n$N.log
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])], "nar", round(d.get("neighbor_allreduce",{}).get("gbs_per_gpu",0),1), round(d.get("neighbor_allreduce",{}).get("frac_of_nvlink_770",0),3))'
for agents in 8 $N; do for topo in one_peer exp2; do
  out=$(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $N --agents $agents --topology $topo --steps 50 --warmup 5 --no-e2e 2>&1)
  echo "$out" | grep '^{' | tail -1 > gpurun_out/bench_n${N}_a${agents}_${topo}.json
  echo "N=$N agents=$agents $topo: $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 bench_suite.py --only c1,h,gt,e,c5 --out gpurun_out/suite_n$N.jsonl 2>&1 | grep '^{'
