cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_H0.so variants/lib_H2.so; do
 for rep in 1 2; do
  for topo in one_peer exp2; do
    out=$(BF_LIB_PATH=$lib timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
    echo "$lib $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 300)"
  done
 done
done
timeout 1200 python bench_suite.py --only h,c5,c2,c1 --out gpurun_out/suite2_n1.jsonl > gpurun_out/suite2_n1.log 2>&1; echo "suite rc=$?"; tail -12 gpurun_out/suite2_n1.log | cut -c1-400
