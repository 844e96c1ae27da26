cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
N=$(nvidia-smi -L | wc -l)
for lib in paper_2111_04287_b200/libbluefog_b200.so variants/lib_M3.so variants/lib_T8192M1.so; do
 for ct in 256 1024; do
  for topo in one_peer exp2; do
    out=$(BF_LIB_PATH=$lib BF_CHUNK_TILES=$ct timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1)
    echo "N=1 $lib ct=$ct $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 200)"
    out=$(BF_LIB_PATH=$lib BF_CHUNK_TILES=$ct timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --topology $topo 2>&1 | grep '^{' | tail -1)
    echo "N=$N $lib ct=$ct $topo $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))' 2>/dev/null || echo "$out" | tail -c 200)"
  done
 done
done
