# Round record on a 4-GPU box: scaling record (smoke, all GPU tests, bench N = 1..4), suites at
# N = 1 / 2 / 4, one-agent-per-GPU shape, multi-process stress
cd $GRAFT_REPO_ROOT
bash scripts/gpu_scale.sh
export BF_TIMEOUT_MS=8000
N=$(nvidia-smi -L | wc -l)
timeout 1200 python bench_suite.py --out gpurun_out/suite_n1.jsonl > gpurun_out/suite_n1.log 2>&1
echo "suite n=1 rc=$?"
for n in 2 4; do
  [ $n -le $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2953$n bench_suite.py --only c1,c3,h,c5,o,e --out gpurun_out/suite_n$n.jsonl > gpurun_out/suite_n$n.log 2>&1
  echo "suite n=$n rc=$?"
done
bash scripts/gpu_k1.sh | tee gpurun_out/k1.txt
if [ $N -ge 4 ]; then
  for k in 1 2; do
    timeout 500 python -m torch.distributed.run --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29561 scripts/stress_mp.py $k 60 2>&1 | grep -E "^rank" | tee -a gpurun_out/stress.txt
  done
fi
