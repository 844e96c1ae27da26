# multi-GPU parity tests + the C3 sweep at N = box GPUs (full log)
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_mp_n$N.log 2>&1; echo "mp pytest rc=$?"; tail -3 gpurun_out/pytest_mp_n$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only c3 --out gpurun_out/suite_c3_n$N.jsonl > gpurun_out/suite_c3_n$N.log 2>&1
echo "c3 rc=$?"; grep -v '^{' gpurun_out/suite_c3_n$N.log | grep -i error | head -5; wc -l gpurun_out/suite_c3_n$N.jsonl
