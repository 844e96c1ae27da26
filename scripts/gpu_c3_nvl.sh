# C3 sweep at N GPUs with the full log, then the NVLink byte capture (rank 0 under ncu)
cd $GRAFT_REPO_ROOT
N=$(nvidia-smi -L | wc -l)
export BF_TIMEOUT_MS=8000
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29545 bench_suite.py --only c3 --out gpurun_out/suite_c3_n$N.jsonl > gpurun_out/suite_c3_n$N.log 2>&1
echo "c3 rc=$?"; grep -v '^{' gpurun_out/suite_c3_n$N.log | tail -30
bash scripts/gpu_ncu_nvlink.sh
