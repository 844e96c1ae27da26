# suite lines (fresh allocations per config) on the box's GPUs + the bench line
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
if [ $N -gt 1 ]; then
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 bench_suite.py --only ${SUITE:-c1,h,io,gt,e,c5,o} --out gpurun_out/suite_fresh_n$N.jsonl 2>&1 | grep '^{' | cut -c1-160
else
  timeout 900 python bench_suite.py --only ${SUITE:-c1,c3,h,io,gt,e,c5,o,c2} --out gpurun_out/suite_fresh_n$N.jsonl 2>&1 | grep '^{' | grep -v "C3 neighbor" | cut -c1-160
fi
