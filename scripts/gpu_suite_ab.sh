# A/B of library variants on bench_suite lines (ONLY=e,gt,h ... AGENTS="8 4"), two repetitions,
# N = box GPUs (variants: python -m paper_2111_04287_b200.build -D<MACRO>=<v> --out=$PWD/variants/lib_<name>.so).
# Records: profiles/r02c_fused_reverse_ab_n1.txt, r02c_ed_ab_n2.txt, r02c_push_modes_ab_n2.txt, r02c_hawc_rows_ab_n2.txt
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
q='import sys,json
for l in sys.stdin:
    d=json.loads(l); v=d.get("ms", d.get("ms_per_step", d.get("ms_per_round", 0))); print("   ", d["config"][:50], round(v,4))'
for rep in 1 2; do for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  for agents in ${AGENTS:-8}; do
    echo "$(basename $lib) agents=$agents"
    if [ $N -gt 1 ]; then
      BF_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only ${ONLY:-e,gt,h} --agents $agents --out /dev/null 2>&1 | grep '^{' | python -c "$q"
    else
      BF_LIB_PATH=$lib timeout 300 python bench_suite.py --only ${ONLY:-e,gt,h} --agents $agents --out /dev/null 2>&1 | grep '^{' | python -c "$q"
    fi
  done
done; done
