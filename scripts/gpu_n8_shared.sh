# The 8-process flow (one agent per process, the 8-GPU setting) on a box with fewer GPUs:
# processes time-share the GPUs (p on GPU p mod G, gloo bootstrap).  Parity worker + the bench
# line's flow (its timings are not measurements).
cd $GRAFT_REPO_ROOT
G=$(nvidia-smi -L | wc -l)
export BF_TIMEOUT_MS=20000
BF_TEST_SHARE_GPUS=$G BF_TEST_K=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29571 tests/mp_worker.py > gpurun_out/mp8_shared.log 2>&1
echo "mp_worker 8 procs on $G GPUs rc=$? ALL OK count: $(grep -c 'ALL OK' gpurun_out/mp8_shared.log)"
grep -E "FAIL|Error|error" gpurun_out/mp8_shared.log | head -20
BF_BENCH_SHARE_GPUS=$G timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 8 --steps 6 --warmup 3 > gpurun_out/bench8_shared.json 2> gpurun_out/bench8_shared.err
echo "bench 8 procs rc=$?"; tail -c 1500 gpurun_out/bench8_shared.json; tail -5 gpurun_out/bench8_shared.err
