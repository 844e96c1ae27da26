# Round record on a 4-GPU box: scaling record, suites at N = 2 / 4, one-agent-per-GPU shape
cd $GRAFT_REPO_ROOT
bash scripts/gpu_scale.sh
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2953$n bench_suite.py --only c1,c3,h,c5,o,e --out gpurun_out/suite_n$n.jsonl > gpurun_out/suite_n$n.log 2>&1
  echo "suite n=$n rc=$?"
done
bash scripts/gpu_k1.sh | tee gpurun_out/k1.txt
