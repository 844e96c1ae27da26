# BF_STATS per-CTA timings of the cross-GPU kernels at N = 2: K = 4 one-peer (pull rounds 0/1,
# push round 2), K = 4 with push forced, K = 1 push
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for cfg in "default 8 one_peer" "push_all 8 one_peer" "default 2 one_peer" "default 8 exp2"; do set -- $cfg
  echo "--- BF_XFER=$1 agents=$2 $3"
  BF_XFER=$1 BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/stats_probe.py $3 $2 2>&1 | grep -E "^rank|Error" | sort
done
