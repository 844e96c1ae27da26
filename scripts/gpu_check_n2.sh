cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for k in 1 2 4; do timeout 120 python -m torch.distributed.run --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29519 scripts/debug_mp.py $k 1048576 2>&1 | grep "^rank" | grep "wire" | awk '{print $1,$2,$3,$4,$5,$6,$7,$8,$9,$10}'; done
timeout 300 python -m pytest tests/test_multigpu.py -q -x 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
export BF_TIMEOUT_MS=5000
LIBS=" " bash scripts/gpu_var2.sh
