# N = 1 round record of the final tree: smoke, GPU tests, bench line, full suite, ncu launch
# list of the bench command + --set full of the fused ATC kernel
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_n1.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_n1.log
SUITE=c1,c3,h,io,gt,e,c5,o,c2 bash scripts/gpu_final.sh
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-nar"
timeout 120 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02c_launches_fused.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_fused_kernel -s 3 -c 1 \
    -o gpurun_out/r02c_prof_fused -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu bench rc=$?"
