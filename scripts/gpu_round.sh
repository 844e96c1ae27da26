# parity (1 GPU + multi-process), N=1 bench + C3 sweep, N=#GPUs bench
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 400 python -m pytest tests/test_multigpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
export BF_TIMEOUT_MS=5000
summ='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), r["bound"], round(r["frac"],3), round(r.get("frac_per_round_bound",0),3), [(round(b["ms"],3), round(b["t_roof_ms"],3)) for b in r.get("by_round",[])])'
for topo in one_peer exp2; do
  echo "N=1 $topo $(timeout 60 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --topology $topo 2>&1 | tail -1 | python -c "$summ")"
done
timeout 600 python bench_suite.py --only ${SUITE:-c3} --out gpurun_out/suite_round.jsonl > gpurun_out/suite_round.log 2>&1; echo "suite rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/suite_round.jsonl'):
    d=json.loads(l)
    if d.get('config','').startswith('C3') and d['bytes_per_agent'] in (1<<20, 1<<26, 1<<30):
        print('C3', d['dtype'], d['topology'], d['bytes_per_agent'], round(d['us'],1), 'us', round(d['hbm_frac'],3))
    elif not d.get('config','').startswith('C3'):
        print({k:(round(v,4) if isinstance(v,float) else v) for k,v in d.items()})
PY
N=$(nvidia-smi -L | wc -l)
if [ $N -ge 2 ]; then LIBS=" " bash scripts/gpu_var2.sh; fi
