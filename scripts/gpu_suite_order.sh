# Exact-Diffusion / GT lines with and without the C5 window round before them (N = 1)
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
q='import sys,json
for l in sys.stdin:
    d=json.loads(l); v=d.get("ms", d.get("ms_per_step", d.get("ms_per_round", 0))); print(d["config"][:50], round(v,4))'
echo "-- e,gt"; timeout 300 python bench_suite.py --only e,gt --out /dev/null 2>&1 | grep '^{' | python -c "$q"
echo "-- c5,e,gt"; timeout 300 python bench_suite.py --only c5,e,gt --out /dev/null 2>&1 | grep '^{' | python -c "$q"
nvidia-smi --query-gpu=clocks.sm,clocks.mem,temperature.gpu,power.draw,clocks_event_reasons.active --format=csv
echo "-- c3,e,gt"; timeout 300 python bench_suite.py --only c3,e,gt --out /dev/null 2>&1 | grep '^{' | grep -v "C3 neighbor" | python -c "$q"
echo "-- h,e"; timeout 300 python bench_suite.py --only h,e --out /dev/null 2>&1 | grep '^{' | python -c "$q"
