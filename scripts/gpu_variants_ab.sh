# A/B of library variants on N = #GPUs: bench.py C4 lines for every library in LIBS
# (default: the built library + variants/*.so, each built with
#   python -m paper_2111_04287_b200.build -D<MACRO>=<value> --out=$PWD/variants/lib_<name>.so)
# over the agent counts AGENTS and topologies TOPOS, two repetitions, alternating.
# BF_XFER=push|pull|push_all selects the cross-GPU path.  Records of this script:
# profiles/r02_push_pull_ab_n2.txt, r02_push_prefetch_ab_n2.txt, r02_push_k2_variants_n4.txt.
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
summ='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac"],3), [round(b["ms"],3) for b in r.get("by_round",[])])'
for rep in 1 2; do
for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  for agents in ${AGENTS:-$N 8}; do for topo in ${TOPOS:-one_peer exp2}; do
    out=$(BF_LIB_PATH=$lib timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --agents $agents --steps 60 --warmup 6 --no-e2e --no-cpu --no-nar --topology $topo 2>&1)
    echo "$(basename $lib) ${BF_XFER:-push} N=$N agents=$agents $topo $(echo "$out" | python -c "$summ" 2>&1 | tail -1)"
  done; done
done
done
