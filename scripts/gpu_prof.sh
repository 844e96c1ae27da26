cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=3000
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
timeout 120 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 2 -c 1 \
    -o gpurun_out/prof_v4 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
