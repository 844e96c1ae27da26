cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_mp_ll.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/pytest_mp_ll.log
for ll in 1 0; do
BF_LL=$ll timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only c1,c2 2>&1 | grep '^{' | sed "s/^/LL=$ll /"
done
