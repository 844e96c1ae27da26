# Scaling record: smoke, GPU tests (all), bench at N = 1 .. #GPUs for both topologies (full JSON lines)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/bench_scale.jsonl
: > $OUT
timeout 60 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -ra --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_n$N.log 2>&1; echo "pytest -m gpu rc=$?"; tail -4 gpurun_out/pytest_gpu_n$N.log
fi
for n in 1 2 4 8; do
  [ $n -le $N ] || continue
  for topo in one_peer exp2; do
    if [ $n = 1 ]; then
      extra=""; [ $topo = exp2 ] && extra="--no-cpu"
      timeout 300 python bench.py --topology $topo $extra > gpurun_out/b.json 2> gpurun_out/b.err
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $n --topology $topo > gpurun_out/b.json 2> gpurun_out/b.err
    fi
    echo "bench n=$n $topo rc=$?"
    grep '^{' gpurun_out/b.json | tail -1 | tee -a $OUT | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(" ", round(d["ms_per_step"],4), "ms", round(d["value"],1), d["unit"], r["bound"], round(r["frac"],3), "per-round", round(r["frac_per_round_bound"],3), "e2e", round(d.get("e2e",{}).get("value",0),1), d["clocks"])' 2>/dev/null || tail -3 gpurun_out/b.err
  done
done
