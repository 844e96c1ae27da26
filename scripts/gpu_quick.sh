# Quick round trip on one GPU: smoke, single-GPU parity tests, bench A/B of exchange kernels.
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
timeout 60 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 90 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for K in ${KERNELS:-fused chunk}; do
  for topo in ${TOPOS:-one_peer exp2}; do
    for wire in ${WIRES:-fp32}; do
      out=$(BF_EXCH=$K timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo --wire $wire 2>&1 | tail -1)
      echo "N=1 $K $topo $wire $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), d["roofline"]["bound"], round(d["roofline"]["achieved"],1), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
    done
  done
done
