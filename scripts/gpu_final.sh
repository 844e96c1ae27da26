# round record on N GPUs: GPU tests, default bench line, suite
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_n$N.log
if [ $N -gt 1 ]; then
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $N > gpurun_out/bench_final_n$N.json 2> gpurun_out/bench_final_n$N.err
else
  timeout 300 python bench.py > gpurun_out/bench_final_n$N.json 2> gpurun_out/bench_final_n$N.err
fi
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_final_n$N.json
if [ $N -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 bench_suite.py --only ${SUITE:-c1,h,io,gt,e,c5,o} --out gpurun_out/suite_final_n$N.jsonl 2>&1 | grep '^{'
else
  timeout 900 python bench_suite.py --only ${SUITE:-c1,c3,h,io,gt,e,c5,o,c2} --out gpurun_out/suite_final_n$N.jsonl 2>&1 | grep '^{'
fi
