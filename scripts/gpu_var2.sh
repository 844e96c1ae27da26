# N-GPU bench of library variants (BF_LIB_PATH) with per-round detail
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
for lib in paper_2111_04287_b200/libbluefog_b200.so ${LIBS:-variants/*.so}; do
  for topo in ${TOPOS:-one_peer exp2}; do
    out=$(BF_LIB_PATH=$lib timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 60 --warmup 6 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
    echo "N=$N $(basename $lib) $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["frac_per_round_bound"],3), [(round(b["ms"],3), round(b["t_roof_ms"],3)) for b in r["by_round"]], d["clocks"]["sm_mhz"])' 2>/dev/null || echo "$out" | tail -c 300)"
  done
done
