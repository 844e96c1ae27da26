cd $GRAFT_REPO_ROOT
export BF_TIMEOUT_MS=5000
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu"
timeout 120 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_chunk.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exchange_chunk_kernel -s 2 -c 1 \
    -o gpurun_out/prof_chunk -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full.log
timeout 1500 python bench_suite.py --out gpurun_out/suite_n1.jsonl > gpurun_out/suite_n1.log 2>&1; echo "suite rc=$?"; tail -40 gpurun_out/suite_n1.log | cut -c1-300
