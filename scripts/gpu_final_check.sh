# Round-close check: smoke, all GPU tests, bench N=1 (and N=2 when present)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -3 gpurun_out/final_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench n1 rc=$?"; tail -1 gpurun_out/final_bench_n1.json
N=$(nvidia-smi -L | wc -l)
if [ $N -ge 2 ]; then
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/final_bench_n2.json 2> gpurun_out/final_bench_n2.err; echo "bench n2 rc=$?"; tail -1 gpurun_out/final_bench_n2.json
fi
