cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for xf in push_all pull; do
echo "--- $xf K=4 one_peer"
BF_XFER=$xf BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py one_peer 8 2>&1 | grep -E "^rank 0|Error" | sort | head
done
