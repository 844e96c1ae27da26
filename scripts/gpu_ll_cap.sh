cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for cap in 32768 1048576; do
BF_LL_CAP=$cap timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29547 bench_suite.py --only c3 --agents 2 --max-bytes 16777216 2>&1 | grep '^{' | python -c '
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    print("cap='$cap'", d["dtype"], d["topology"], d["bytes_per_agent"], round(d["us"],1))'
done
