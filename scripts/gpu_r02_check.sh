# round-2 check on N GPUs: all GPU tests, NVLink hardware counters, bench N lines
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
echo "--- NVLink counters"
for cfg in "one_peer $N" "exp2 $N" "one_peer 8"; do set -- $cfg
for xf in push pull; do
BF_XFER=$xf timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 scripts/nvlink_bytes.py $1 $2 200 2>&1 | grep "^{" | tee -a gpurun_out/nvlink_bytes.jsonl
done; done
echo "--- bench"
for agents in $N 8; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $N --agents $agents --steps 50 --warmup 5 > gpurun_out/bench_n${N}_a${agents}.json 2> gpurun_out/bench_n${N}_a${agents}.err; echo "bench agents=$agents rc=$?"; tail -c 1500 gpurun_out/bench_n${N}_a${agents}.json
done
