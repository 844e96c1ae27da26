# Full check on an N-GPU box: smoke, all GPU tests, bench at 1..N GPUs (both topologies)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
N=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 60 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -ra --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest -m gpu rc=$?"; tail -12 gpurun_out/pytest_gpu_n$N.log
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench n=1 rc=$?"; tail -1 gpurun_out/bench_n1.json
timeout 300 python bench.py --topology exp2 --no-cpu > gpurun_out/bench_n1_exp2.json 2>/dev/null; tail -1 gpurun_out/bench_n1_exp2.json | cut -c1-400
for n in 2 4; do
  if [ $N -ge $n ]; then
    for topo in one_peer exp2; do
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $n --topology $topo > gpurun_out/bench_n${n}_$topo.json 2> gpurun_out/bench_n${n}_$topo.err
      echo "bench n=$n $topo rc=$?"; grep '^{' gpurun_out/bench_n${n}_$topo.json | tail -1 | cut -c1-600
    done
  fi
done
