# C3 sweep incl. the registered-input (bf_alloc) lines, on the box's GPUs
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
if [ $N -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29546 bench_suite.py --only c3 --out gpurun_out/c3_reg_n$N.jsonl > gpurun_out/c3_reg_n$N.log 2>&1
else
  timeout 900 python bench_suite.py --only c3 --out gpurun_out/c3_reg_n$N.jsonl > gpurun_out/c3_reg_n$N.log 2>&1
fi
echo "rc=$?"; grep '"bytes_per_agent": 1073741824' gpurun_out/c3_reg_n$N.jsonl | cut -c1-330; tail -3 gpurun_out/c3_reg_n$N.log | cut -c1-300
