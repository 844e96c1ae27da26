cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
timeout 60 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x --timeout 90 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for topo in one_peer exp2; do
  out=$(timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
  echo "N=1 $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
done
for ct in 64 128; do
  out=$(BF_CHUNK_TILES=$ct timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1)
  echo "N=1 ct=$ct $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
done
timeout 1200 python bench_suite.py --only h,c5,c2,c1 --out gpurun_out/suite2_n1.jsonl > gpurun_out/suite2_n1.log 2>&1; echo "suite rc=$?"; tail -12 gpurun_out/suite2_n1.log | cut -c1-400
