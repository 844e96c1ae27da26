# r02 ncu evidence (1 GPU): bench launch list + --set full of the fused ATC kernel,
# window kernels (C5-shaped round), gradient-tracking kernels
cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=8000
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-nar"
timeout 120 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02_launches_fused.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_fused_kernel -s 3 -c 1 \
    -o gpurun_out/r02_prof_fused -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu bench rc=$?"
timeout 120 python scripts/prof_win.py > gpurun_out/plain_win.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_win.csv python scripts/prof_win.py > gpurun_out/ncu_wl.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"win_(push|collect)_kernel" -s 2 -c 2 -o gpurun_out/r02_prof_win -f python scripts/prof_win.py > gpurun_out/ncu_win.log 2>&1
echo "ncu win rc=$?"
timeout 120 python scripts/prof_gt.py > gpurun_out/plain_gt.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:exchange_fused_kernel -s 2 -c 2 -o gpurun_out/r02_prof_gt -f python scripts/prof_gt.py > gpurun_out/ncu_gt.log 2>&1
echo "ncu gt rc=$?"
