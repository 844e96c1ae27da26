cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
for topo in one_peer; do
BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py $topo 2 2>&1 | grep -E "^rank|Error" | sort | head
done
