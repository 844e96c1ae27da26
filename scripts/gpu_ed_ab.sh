# Exact-Diffusion / GT steps across GPUs: push-kernel reverse walk and prefetch A/B, K = 4 and K = 2
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
q='import sys,json
for l in sys.stdin:
    d=json.loads(l); v=d.get("ms", d.get("ms_per_step", d.get("ms_per_round", 0))); print("   ", d["config"][:40], round(v,4))'
for rep in 1 2; do for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_pnorev.so variants/lib_nopf.so; do
  for agents in 8 $((2*N)); do
    echo "$(basename $lib) agents=$agents"
    BF_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only e,gt --agents $agents --out /dev/null 2>&1 | grep '^{' | python -c "$q"
  done
done; done
