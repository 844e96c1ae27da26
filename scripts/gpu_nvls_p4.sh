cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
for nv in 1 0; do
BF_NVLS=$nv timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29546 bench_suite.py --only h --agents 4 2>&1 | grep '^{' | sed "s/^/NVLS=$nv /"
done
python scripts/host_overhead.py 2>&1 | tail -3
