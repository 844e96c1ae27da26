# GPU round trip: smoke, GPU tests, bench, then (only after a clean plain run) ncu.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
export BF_TIMEOUT_MS=5000
timeout 120 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -ra ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:exchange_kernel -s 2 -c 1 \
      -o gpurun_out/prof_exchange -f $CMD > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"
  tail -3 gpurun_out/ncu_full.log
fi
