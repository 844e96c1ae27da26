# ncu evidence for the default (local-agent fused) exchange kernel at N=1, bench C4 config
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 120 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_fused.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_fused_kernel -s 3 -c 1 \
    -o gpurun_out/prof_fused -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
