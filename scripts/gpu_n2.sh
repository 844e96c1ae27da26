# 2-GPU round trip: single-GPU parity, IPC multi-process parity, bench A/B at N=1 and N=2.
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
timeout 500 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
BF_TIMEOUT_MS=8000 timeout 400 python -m pytest tests/test_multigpu.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"; tail -3 gpurun_out/pytest_multi.log
for K in ${KERNELS:-fused chunk}; do
  for topo in ${TOPOS:-one_peer exp2}; do
    out=$(BF_EXCH=$K timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
    echo "N=1 $K $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["achieved"],1), round(r["frac"],3), round(r["frac_per_round_bound"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
    out=$(BF_EXCH=$K timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
    echo "N=$N $K $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["achieved"],1), round(r["frac"],3), round(r["frac_per_round_bound"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
