cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "parity" 2>&1 | tail -1
for ag in 4 8; do for nv in 1 0; do
BF_NVLS=$nv timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29546 bench_suite.py --only h --agents $ag 2>&1 | grep '^{' | python -c '
import json,sys
for l in sys.stdin:
    d=json.loads(l); print("NVLS='$nv' agents='$ag'", d["config"], round(d["ms"],3), d["path"][:40])'
done; done
