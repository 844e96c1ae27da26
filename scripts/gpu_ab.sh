# A/B of the exchange kernels at N=1 and N=2 (run with gpurun --gpus 2)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
run_bench() {   # $1 label
  for topo in ${TOPOS:-one_peer exp2}; do
    out=$(timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
    echo "N=1 $1 $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d["roofline"]["bound"], round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
    if [ $N -ge 2 ]; then
      out=$(timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
      echo "N=$N $1 $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d["roofline"]["bound"], round(d["roofline"]["frac"],3), round(d["roofline"]["achieved"],1))' 2>/dev/null || echo "$out" | tail -c 300)"
    fi
  done
}
for K in ${KERNELS:-chunk}; do
  export BF_EXCH=$K
  timeout 200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -p no:cacheprovider > gpurun_out/pytest_$K.log 2>&1; echo "parity $K rc=$?"; tail -2 gpurun_out/pytest_$K.log
  if [ $N -ge 2 ]; then
    BF_TIMEOUT_MS=8000 timeout 300 python -m pytest tests/test_multigpu.py -q -x --timeout 200 -k "2-1 or 2-2" > gpurun_out/pytest_multi_$K.log 2>&1; echo "multi $K rc=$?"; tail -2 gpurun_out/pytest_multi_$K.log
  fi
  if [ "$K" = "chunk" ]; then
    for ct in ${CTS:-128}; do BF_CHUNK_TILES=$ct run_bench "chunk$ct"; done
  else
    run_bench $K
  fi
done
