cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
bash scripts/gpu_variants.sh
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 2 -c 1 \
    -o gpurun_out/prof_v3 -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
