cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider -k "multiprocess_parity" > gpurun_out/pytest_mp_nvls.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/pytest_mp_nvls.log; grep -h "NVLS" gpurun_out/pytest_mp_nvls.log | head
for nv in 1 0; do
BF_NVLS=$nv timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29546 bench_suite.py --only h,c1,c2 2>&1 | grep '^{' | sed "s/^/NVLS=$nv /"
done
