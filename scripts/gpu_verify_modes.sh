# after restricting the push kernel's reverse walk to ATC and its prefetch to MODE <= 2:
# bench lines (ATC) and the suite's E / GT / H / IO lines, previous library as variants/lib_prev.so
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
q='import sys,json
for l in sys.stdin:
    d=json.loads(l); v=d.get("ms", d.get("ms_per_step", d.get("ms_per_round", 0))); print("   ", d["config"][:50], round(v,4))'
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_prev.so; do
  echo "== $(basename $lib)"
  AGENTS="8 $((2*N))" LIBS=" " bash scripts/gpu_variants_ab.sh 2>/dev/null | head -0
  for agents in 8 $((2*N)); do
    echo " agents=$agents"
    BF_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only e,gt,h,io --agents $agents --out /dev/null 2>&1 | grep '^{' | python -c "$q"
  done
done
AGENTS="8 $((2*N))" TOPOS="one_peer exp2" LIBS="variants/lib_prev.so" bash scripts/gpu_variants_ab.sh
