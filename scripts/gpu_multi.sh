# Multi-GPU round trip (run with gpurun --gpus N): IPC parity tests, then the bench at N.
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m | head -8
export BF_TIMEOUT_MS=8000
timeout 900 python -m pytest tests/test_multigpu.py -q -ra -x > gpurun_out/pytest_multi_n$N.log 2>&1; echo "pytest multi rc=$?"
tail -25 gpurun_out/pytest_multi_n$N.log
for extra in "" "--topology exp2"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
     --master-port 29511 bench.py --gpus $N --steps 30 --warmup 5 $extra > gpurun_out/bench_n$N$(echo $extra | tr -d ' -').log 2>&1
  echo "bench n=$N $extra rc=$?"
  tail -2 gpurun_out/bench_n$N$(echo $extra | tr -d ' -').log
done
